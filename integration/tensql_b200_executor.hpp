// tensql_b200_executor.hpp — the reference-side binding a tensql maintainer
// adds to run lowered plans on a B200 through the C ABI (include/tqp_b200.h).
// It has the surface of tensql::Executor (proj/include/tensql/exec/executor.hpp:43-59):
//
//   tensql::OperatorPlan op = tensql::plan_operators(tensql::optimize(plan, cat), cat);
//   tqp_integration::B200Executor ex(std::move(op));          // was: Executor(op, backend)
//   tensql::EncodedTable out = ex.execute(tables);            // same TableSet in, same table out
//
// Errors are rethrown as the reference's exception types with its messages.
// Header-only; compile against /root/reference/proj/include and link
// libtqp_b200.so.
#pragma once

#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "tensql/exec/executor.hpp"
#include "tensql/exec/operator_plan.hpp"
#include "tqp_b200.h"

namespace tqp_integration {

inline void rethrow(const tqp_status& st) {
  switch (st.code) {
    case TQP_OK: return;
    case TQP_ERR_KERNEL: throw tensql::KernelError(st.msg);
    case TQP_ERR_EXEC: throw tensql::ExecError(st.msg);
    case TQP_ERR_PLAN: throw tensql::PlanError(st.msg);
    case TQP_ERR_ENCODING: throw tensql::EncodingError(st.msg);
    default: throw std::runtime_error(st.msg);
  }
}

inline int dtype_of(tensql::DType t) {
  switch (t) {
    case tensql::DType::Bool: return TQP_BOOL;
    case tensql::DType::Int32: return TQP_I32;
    case tensql::DType::Int64: return TQP_I64;
    case tensql::DType::Float64: return TQP_F64;
  }
  return TQP_I64;
}

inline int logical_of(tensql::LogicalType t) { return static_cast<int>(t); }  // same enum order

inline const void* host_data(const tensql::Tensor& t) {
  switch (t.dtype()) {
    case tensql::DType::Bool: return t.data<uint8_t>().data();
    case tensql::DType::Int32: return t.data<int32_t>().data();
    case tensql::DType::Int64: return t.data<int64_t>().data();
    case tensql::DType::Float64: return t.data<double>().data();
  }
  return nullptr;
}

// One process-wide device context (cuda:0 unless TQP_DEVICE is set).
inline tqp_ctx* context() {
  static tqp_ctx* ctx = [] {
    tqp_status st{};
    const char* d = std::getenv("TQP_DEVICE");
    tqp_ctx* c = tqp_init(d ? std::atoi(d) : 0, &st);
    rethrow(st);
    return c;
  }();
  return ctx;
}

// OperatorPlan (operator_plan.hpp:73-92) -> tqp_plan, instruction by
// instruction; op names are the reference's instr_op_name strings.
inline tqp_plan* to_tqp_plan(const tensql::OperatorPlan& op) {
  tqp_status st{};
  tqp_plan* p = tqp_plan_create(op.num_slots, &st);
  rethrow(st);
  for (const auto& step : op.steps) {
    tqp_plan_begin_step(p, step.id.c_str(), step.kind.c_str(), &st);
    rethrow(st);
    for (const auto& in : step.instrs) {
      tqp_instr_desc d{};
      d.op = tensql::instr_op_name(in.op);
      d.inputs = in.inputs.data();
      d.num_inputs = static_cast<int>(in.inputs.size());
      d.output = in.output;
      d.cmp = static_cast<int>(in.cmp);
      d.arith = static_cast<int>(in.arith);
      d.logic = static_cast<int>(in.logic);
      d.side = static_cast<int>(in.side);
      d.reduce = static_cast<int>(in.reduce);
      d.anchor = static_cast<int>(in.anchor);
      d.cast_to = dtype_of(in.cast_to);
      d.pattern = in.pattern.data();
      d.pattern_len = static_cast<int64_t>(in.pattern.size());
      d.table = in.table.c_str();
      d.column = in.column.c_str();
      d.param = in.param;
      if (in.op == tensql::InstrOp::ConstTensor) {
        d.const_dtype = dtype_of(in.constant.dtype());
        d.const_rows = in.constant.rows();
        d.const_cols = in.constant.cols();
        d.const_data = host_data(in.constant);
      }
      tqp_plan_add_instr(p, &d, &st);
      rethrow(st);
    }
    tqp_plan_set_step_outputs(p, step.output_slots.data(), static_cast<int>(step.output_slots.size()), &st);
    rethrow(st);
  }
  for (const auto& o : op.outputs) {
    tqp_plan_add_output(p, o.name.c_str(), logical_of(o.type), o.slot, &st);
    rethrow(st);
  }
  for (const auto& [name, schema] : op.input_tables) {
    for (const auto& c : schema) {
      tqp_plan_add_input_column(p, name.c_str(), c.name.c_str(), logical_of(c.type), &st);
      rethrow(st);
    }
  }
  return p;
}

// EncodedTable (columnar.hpp:41-54) -> device table (uploads every column).
inline tqp_table* upload(const tensql::EncodedTable& t) {
  tqp_status st{};
  tqp_table* tab = tqp_table_create(context(), &st);
  rethrow(st);
  for (const auto& c : t.columns()) {
    tqp_tensor* x;
    if (c.logical == tensql::LogicalType::Utf8) {
      x = tqp_tensor_from_host_utf8_i32(context(), c.tensor.rows(), c.tensor.cols(), c.tensor.data<int32_t>().data(), &st);
    } else {
      x = tqp_tensor_from_host(context(), dtype_of(c.tensor.dtype()), c.tensor.rows(), c.tensor.cols(), host_data(c.tensor),
                               &st);
    }
    rethrow(st);
    tqp_table_add_column(tab, c.name.c_str(), logical_of(c.logical), x, &st);
    tqp_tensor_free(x);
    rethrow(st);
  }
  return tab;
}

inline tensql::Tensor download(const tqp_tensor* t) {
  tqp_status st{};
  const int64_t rows = tqp_tensor_rows(t), cols = tqp_tensor_cols(t);
  const size_t n = static_cast<size_t>(rows * cols);
  switch (tqp_tensor_dtype(t)) {
    case TQP_BOOL: {
      std::vector<uint8_t> v(n);
      tqp_tensor_to_host(context(), t, v.data(), &st);
      rethrow(st);
      return tensql::Tensor::from_matrix(rows, cols, std::move(v));
    }
    case TQP_I32:
    case TQP_STR8: {
      std::vector<int32_t> v(n);
      tqp_tensor_to_host_utf8_i32(context(), t, v.data(), &st);
      rethrow(st);
      return tensql::Tensor::from_matrix(rows, cols, std::move(v));
    }
    case TQP_I64: {
      std::vector<int64_t> v(n);
      tqp_tensor_to_host(context(), t, v.data(), &st);
      rethrow(st);
      return tensql::Tensor::from_matrix(rows, cols, std::move(v));
    }
    default: {
      std::vector<double> v(n);
      tqp_tensor_to_host(context(), t, v.data(), &st);
      rethrow(st);
      return tensql::Tensor::from_matrix(rows, cols, std::move(v));
    }
  }
}

class B200Executor {
 public:
  explicit B200Executor(tensql::OperatorPlan plan, bool fuse = true) : plan_(std::move(plan)) {
    tqp_status st{};
    tqp_plan* p = to_tqp_plan(plan_);
    ex_ = tqp_executor_create(context(), p, fuse ? TQP_EXEC_FUSE : TQP_EXEC_NO_FUSE, &st);
    tqp_plan_free(p);
    rethrow(st);
  }
  B200Executor(const B200Executor&) = delete;
  B200Executor& operator=(const B200Executor&) = delete;
  ~B200Executor() { tqp_executor_free(ex_); }

  const tensql::OperatorPlan& plan() const { return plan_; }
  std::string_view backend_name() const { return "b200"; }
  std::string explain() const { return tqp_executor_explain(ex_); }
  // fused units that handed their steps to the exact per-instruction path
  // (their data left the fused contract) over this executor's runs
  long long fallbacks() const { return static_cast<long long>(tqp_executor_fallbacks(ex_)); }

  // Executor::execute (executor.cpp:346): uploads the tables, runs on device
  // and returns the result as an EncodedTable.
  tensql::EncodedTable execute(const tensql::TableSet& tables) const {
    std::vector<std::unique_ptr<tqp_table, void (*)(tqp_table*)>> owned;
    std::vector<const char*> names;
    std::vector<tqp_table*> tabs;
    for (const auto& [name, t] : tables) {
      owned.emplace_back(upload(t), tqp_table_free);
      names.push_back(name.c_str());
      tabs.push_back(owned.back().get());
    }
    return run(names, tabs);
  }

  // Same, over tables already resident on the device.
  tensql::EncodedTable execute_device(const std::vector<const char*>& names, const std::vector<tqp_table*>& tabs) const {
    return run(names, tabs);
  }

 private:
  tensql::EncodedTable run(const std::vector<const char*>& names, const std::vector<tqp_table*>& tabs) const {
    tqp_status st{};
    tqp_result* r = tqp_executor_execute(ex_, names.data(), tabs.data(), static_cast<int>(tabs.size()), &st);
    rethrow(st);
    std::vector<tensql::EncodedColumn> cols;
    const int n = tqp_result_num_columns(r);
    for (int i = 0; i < n; ++i) {
      cols.push_back({tqp_result_column_name(r, i), static_cast<tensql::LogicalType>(tqp_result_column_type(r, i)),
                      download(tqp_result_column(r, i))});
    }
    tqp_result_free(r);
    return tensql::EncodedTable(std::move(cols));
  }

  tensql::OperatorPlan plan_;
  tqp_executor* ex_ = nullptr;
};

}  // namespace tqp_integration
