// JSON dumps of reference objects (test infrastructure; links the reference
// library built by oracle/Makefile). Formats:
//   tensor  {"dtype": "int64", "rows": n, "cols": m, "data": [...]}
//   table   {"rows": n, "columns": [{"name", "type", "tensor"}]}
//   opplan  the reference's OperatorPlan (operator_plan.hpp:53-92) field by
//           field; the B200 executor consumes exactly this
//           (paper_2209_04579_b200/tqp.py: plan_from_opplan_json).
#pragma once

#include <cmath>
#include <nlohmann/json.hpp>
#include <string>

#include "tensql/columnar.hpp"
#include "tensql/exec/operator_plan.hpp"

namespace tqp_oracle {

using nlohmann::json;
using namespace tensql;

inline json f64_json(double v) {
  if (std::isnan(v)) return "nan";
  if (std::isinf(v)) return v > 0 ? "inf" : "-inf";
  return v;
}

inline json tensor_to_json(const Tensor& t) {
  json j;
  j["dtype"] = dtype_name(t.dtype());
  j["rows"] = t.rows();
  j["cols"] = t.cols();
  json d = json::array();
  switch (t.dtype()) {
    case DType::Bool:
      for (auto v : t.data<uint8_t>()) d.push_back(static_cast<int>(v));
      break;
    case DType::Int32:
      for (auto v : t.data<int32_t>()) d.push_back(v);
      break;
    case DType::Int64:
      for (auto v : t.data<int64_t>()) d.push_back(v);
      break;
    case DType::Float64:
      for (auto v : t.data<double>()) d.push_back(f64_json(v));
      break;
  }
  j["data"] = std::move(d);
  return j;
}

inline json table_to_json(const EncodedTable& t) {
  json j;
  j["rows"] = t.row_count();
  json cols = json::array();
  for (const auto& c : t.columns()) {
    cols.push_back({{"name", c.name}, {"type", logical_type_name(c.logical)},
                    {"tensor", tensor_to_json(c.tensor)}});
  }
  j["columns"] = std::move(cols);
  return j;
}

inline json instr_to_json(const Instr& in) {
  json j;
  j["op"] = instr_op_name(in.op);
  j["inputs"] = in.inputs;
  j["output"] = in.output;
  switch (in.op) {
    case InstrOp::Compare:
    case InstrOp::StringCompare: j["cmp"] = compare_op_name(in.cmp); break;
    case InstrOp::Arith: j["arith"] = arith_op_name(in.arith); break;
    case InstrOp::Logical: j["logic"] = logical_op_name(in.logic); break;
    case InstrOp::SearchSorted: j["side"] = in.side == SearchSide::LEFT ? "left" : "right"; break;
    case InstrOp::SegmentedReduce: j["reduce"] = reduce_op_name(in.reduce); break;
    case InstrOp::SubstringMatch:
      j["anchor"] = match_anchor_name(in.anchor);
      j["pattern"] = in.pattern;
      break;
    case InstrOp::Cast: j["cast_to"] = dtype_name(in.cast_to); break;
    case InstrOp::LoadColumn:
      j["table"] = in.table;
      j["column"] = in.column;
      break;
    case InstrOp::ConstTensor: j["constant"] = tensor_to_json(in.constant); break;
    default: break;
  }
  j["param"] = in.param;
  return j;
}

inline json opplan_to_json(const OperatorPlan& p) {
  json j;
  j["num_slots"] = p.num_slots;
  json steps = json::array();
  for (const auto& s : p.steps) {
    json instrs = json::array();
    for (const auto& in : s.instrs) instrs.push_back(instr_to_json(in));
    steps.push_back({{"id", s.id}, {"kind", s.kind}, {"instrs", instrs},
                     {"output_slots", s.output_slots}});
  }
  j["steps"] = std::move(steps);
  json outs = json::array();
  for (const auto& o : p.outputs) {
    outs.push_back({{"name", o.name}, {"type", logical_type_name(o.type)}, {"slot", o.slot}});
  }
  j["outputs"] = std::move(outs);
  json tabs = json::array();
  for (const auto& [name, schema] : p.input_tables) {
    json cols = json::array();
    for (const auto& c : schema) cols.push_back({{"name", c.name}, {"type", logical_type_name(c.type)}});
    tabs.push_back({{"name", name}, {"schema", cols}});
  }
  j["input_tables"] = std::move(tabs);
  return j;
}

}  // namespace tqp_oracle
