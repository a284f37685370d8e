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

#include <algorithm>
#include <cctype>
#include <cstdlib>
#include <map>
#include <memory>
#include <set>
#include <thread>
#include <stdexcept>
#include <string>
#include <vector>

#include "tensql/exec/executor.hpp"
#include "tensql/exec/operator_plan.hpp"
#include "tqp_b200.h"

#include <cuda_runtime_api.h>
#include <nlohmann/json.hpp>

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

// Columns the plan loads, lower-case "table.column" (LoadColumn instructions,
// executor.cpp:214-221). The executor binds every column of the plan's input
// schema (executor.cpp:355-371); the others are declared without data.
inline std::set<std::string> loaded_columns(const tensql::OperatorPlan& op) {
  auto lower = [](std::string x) {
    for (auto& ch : x) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    return x;
  };
  std::set<std::string> out;
  for (const auto& step : op.steps)
    for (const auto& in : step.instrs)
      if (in.op == tensql::InstrOp::LoadColumn) out.insert(lower(in.table) + "." + lower(in.column));
  return out;
}

// EncodedTable (columnar.hpp:41-54) -> device table on `ctx`: rows [lo, hi)
// of the columns in `wanted` (all when null) are copied, Utf8 narrowed to one
// byte per UTF-8 byte on the host; every other column is declared (name, type,
// rows) without data.
inline tqp_table* upload(const tensql::EncodedTable& t, tqp_ctx* ctx = nullptr, const std::string& table = "",
                         const std::set<std::string>* wanted = nullptr, int64_t lo = 0, int64_t hi = -1) {
  if (!ctx) ctx = context();
  tqp_status st{};
  tqp_table* tab = tqp_table_create(ctx, &st);
  rethrow(st);
  std::string tl = table;
  for (auto& ch : tl) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  for (const auto& c : t.columns()) {
    const int64_t rows = c.tensor.rows(), cols = c.tensor.cols();
    const int64_t a = std::min(lo, rows), b = hi < 0 ? rows : std::min(hi, rows);
    std::string cl = c.name;
    for (auto& ch : cl) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    if (wanted && !wanted->count(tl + "." + cl)) {
      tqp_table_declare_column(tab, c.name.c_str(), logical_of(c.logical), b - a, &st);
      rethrow(st);
      continue;
    }
    tqp_tensor* x;
    if (c.logical == tensql::LogicalType::Utf8) {
      x = tqp_tensor_from_host_utf8_i32(ctx, b - a, cols, c.tensor.data<int32_t>().data() + a * cols, &st);
    } else {
      const size_t esz = c.tensor.dtype() == tensql::DType::Bool ? 1 : c.tensor.dtype() == tensql::DType::Int32 ? 4 : 8;
      x = tqp_tensor_from_host(ctx, dtype_of(c.tensor.dtype()), b - a, cols,
                               static_cast<const char*>(host_data(c.tensor)) + a * cols * esz, &st);
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
  explicit B200Executor(tensql::OperatorPlan plan, bool fuse = true) : B200Executor(std::move(plan), 1, fuse) {}
  // num_gpus ranks (devices 0..num_gpus-1, wrapping when fewer exist), one
  // host thread per rank: every table is cut into num_gpus row ranges and the
  // plan runs through tqp_executor_execute_sharded (build sides exchanged,
  // partials merged; plans that do not shard run on the gathered tables).
  B200Executor(tensql::OperatorPlan plan, int num_gpus, bool fuse = true)
      : plan_(std::move(plan)), loads_(loaded_columns(plan_)), n_(std::max(1, num_gpus)) {
    tqp_status st{};
    tqp_plan* p = to_tqp_plan(plan_);
    int ndev = 1;
    if (n_ > 1 && (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1)) ndev = 1;
    for (int r = 0; r < n_; ++r) {
      tqp_ctx* ctx = r == 0 ? context() : tqp_init(r % ndev, &st);
      if (st.code) {
        tqp_plan_free(p);
        rethrow(st);
      }
      if (r) owned_ctx_.push_back(ctx);
      ctx_.push_back(ctx);
      ex_.push_back(tqp_executor_create(ctx, p, fuse ? TQP_EXEC_FUSE : TQP_EXEC_NO_FUSE, &st));
      if (st.code) {
        tqp_plan_free(p);
        rethrow(st);
      }
    }
    tqp_plan_free(p);
    if (n_ > 1) {
      comm_.assign(n_, nullptr);
      tqp_comm_init_local(n_, comm_.data(), &st);
      rethrow(st);
    }
  }
  B200Executor(const B200Executor&) = delete;
  B200Executor& operator=(const B200Executor&) = delete;
  ~B200Executor() {
    for (auto& [ptr, keep] : pinned_) cudaHostUnregister(const_cast<void*>(ptr));
    for (auto* c : comm_) tqp_comm_free(c);
    for (auto* e : ex_) tqp_executor_free(e);
    for (auto* c : owned_ctx_) tqp_shutdown(c);
  }

  const tensql::OperatorPlan& plan() const { return plan_; }
  std::string_view backend_name() const { return "b200"; }
  int num_gpus() const { return n_; }
  std::string explain() const { return tqp_executor_explain(ex_[0]); }
  // fused units that handed their steps to the exact per-instruction path
  // (their data left the fused contract) over this executor's runs
  long long fallbacks() const {
    long long f = 0;
    for (auto* e : ex_) f += static_cast<long long>(tqp_executor_fallbacks(e));
    return f;
  }

  // Executor::execute (executor.cpp:346): uploads the columns the plan loads
  // (the rest of its input schema is declared without data), runs on the
  // device(s) and returns the result as an EncodedTable.
  tensql::EncodedTable execute(const tensql::TableSet& tables) const {
    pin(tables);
    if (n_ == 1) {
      Uploaded u(tables, ctx_[0], &loads_, 0, 1);
      return run(u.names, u.tabs);
    }
    return run_sharded(tables);
  }

  // Executor::profile_execute (executor.hpp:51, executor.cpp:348-352): the
  // same, filling the reference's ProfileTrace (operators and per-instruction
  // kernels, synchronised after each; on rank 0 for a sharded executor).
  tensql::EncodedTable profile_execute(const tensql::TableSet& tables, tensql::ProfileTrace& trace) const {
    trace = tensql::ProfileTrace{};
    trace.backend = "b200";
    pin(tables);
    if (n_ > 1) return run_sharded(tables);
    Uploaded u(tables, ctx_[0], &loads_, 0, 1);
    tqp_status st{};
    char* json = nullptr;
    tqp_result* r = tqp_executor_profile(ex_[0], u.names.data(), u.tabs.data(), static_cast<int>(u.tabs.size()), &json, &st);
    rethrow(st);
    if (json) {
      for (const auto& e : nlohmann::json::parse(json)) {
        const int64_t ts = static_cast<int64_t>(e.at("ts").get<double>() * 1000.0);
        const int64_t dur = static_cast<int64_t>(e.at("dur").get<double>() * 1000.0);
        const auto& a = e.at("args");
        if (e.at("cat") == "operator") {
          trace.operators.push_back({e.at("name").get<std::string>(), "", ts, dur, a.value("rows", int64_t{0}),
                                     a.value("bytes", int64_t{0})});
        } else {
          trace.kernels.push_back({a.value("operator", std::string()), e.at("name").get<std::string>(), ts, dur,
                                   a.value("rows", int64_t{0}), a.value("bytes", int64_t{0})});
        }
      }
      tqp_free_str(json);
    }
    // operator kinds from the plan (the trace names operators by step id)
    for (auto& op : trace.operators)
      for (const auto& step : plan_.steps)
        if (step.id == op.id) op.kind = step.kind;
    return collect(r);
  }

  // Same, over tables already resident on the device (single GPU).
  tensql::EncodedTable execute_device(const std::vector<const char*>& names, const std::vector<tqp_table*>& tabs) const {
    return run(names, tabs);
  }

 private:
  struct Uploaded {
    std::vector<std::unique_ptr<tqp_table, void (*)(tqp_table*)>> owned;
    std::vector<const char*> names;
    std::vector<tqp_table*> tabs;
    Uploaded(const tensql::TableSet& tables, tqp_ctx* ctx, const std::set<std::string>* wanted, int rank, int n) {
      for (const auto& [name, t] : tables) {
        const int64_t rows = t.row_count();
        owned.emplace_back(upload(t, ctx, name, wanted, rows * rank / n, rows * (rank + 1) / n), tqp_table_free);
        names.push_back(name.c_str());
        tabs.push_back(owned.back().get());
      }
    }
  };

  // The reference's host tensors are immutable shared buffers
  // (tensor.hpp:107-121): the numeric columns the plan loads are page-locked
  // in place once (cudaHostRegister) and kept registered - and alive, through
  // a copy of the tensor - for this executor's lifetime, so every later
  // execute() uploads them by DMA at full PCIe speed instead of through the
  // driver's pageable staging. Utf8 columns are narrowed on the host first.
  void pin(const tensql::TableSet& tables) const {
    for (const auto& [name, t] : tables) {
      std::string tl = name;
      for (auto& ch : tl) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
      for (const auto& c : t.columns()) {
        if (c.logical == tensql::LogicalType::Utf8) continue;
        std::string cl = c.name;
        for (auto& ch : cl) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
        if (!loads_.count(tl + "." + cl)) continue;
        const void* ptr = host_data(c.tensor);
        const size_t esz = c.tensor.dtype() == tensql::DType::Bool ? 1 : c.tensor.dtype() == tensql::DType::Int32 ? 4 : 8;
        const size_t bytes = static_cast<size_t>(c.tensor.rows() * c.tensor.cols()) * esz;
        if (!ptr || bytes < (size_t(1) << 20) || pinned_.count(ptr)) continue;
        if (cudaHostRegister(const_cast<void*>(ptr), bytes, cudaHostRegisterReadOnly) == cudaSuccess) {
          pinned_.emplace(ptr, c.tensor);
        } else {
          cudaGetLastError();  // not registrable (already pinned, ...): the copy stages as before
        }
      }
    }
  }

  tensql::EncodedTable run(const std::vector<const char*>& names, const std::vector<tqp_table*>& tabs) const {
    tqp_status st{};
    tqp_result* r = tqp_executor_execute(ex_[0], names.data(), tabs.data(), static_cast<int>(tabs.size()), &st);
    rethrow(st);
    return collect(r);
  }

  tensql::EncodedTable run_sharded(const tensql::TableSet& tables) const {
    std::vector<tqp_result*> res(n_, nullptr);
    std::vector<tqp_status> sts(n_);
    std::vector<std::thread> th;
    for (int r = 0; r < n_; ++r) {
      th.emplace_back([&, r] {
        try {
          Uploaded u(tables, ctx_[r], &loads_, r, n_);
          std::vector<int> kinds(u.tabs.size(), TQP_SHARD_ROWS);
          res[r] = tqp_executor_execute_sharded(ex_[r], comm_[r], u.names.data(), u.tabs.data(), kinds.data(),
                                                static_cast<int>(u.tabs.size()), &sts[r]);
        } catch (const std::exception& e) {
          sts[r].code = TQP_ERR_ARG;
          std::snprintf(sts[r].msg, sizeof(sts[r].msg), "%s", e.what());
        }
      });
    }
    for (auto& t : th) t.join();
    for (int r = 1; r < n_; ++r)
      if (res[r]) tqp_result_free(res[r]);
    for (int r = 0; r < n_; ++r)
      if (sts[r].code) {
        if (res[0]) tqp_result_free(res[0]);
        rethrow(sts[r]);
      }
    return collect(res[0]);
  }

  static tensql::EncodedTable collect(tqp_result* r) {
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
  std::set<std::string> loads_;
  int n_ = 1;
  std::vector<tqp_ctx*> ctx_, owned_ctx_;
  std::vector<tqp_executor*> ex_;
  std::vector<tqp_comm*> comm_;
  mutable std::map<const void*, tensql::Tensor> pinned_;  // registered host column -> the tensor keeping it alive
};

}  // namespace tqp_integration
