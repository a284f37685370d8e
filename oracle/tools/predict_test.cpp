// tqp_predict_test - PREDICT on the device: the reference
// lowers PREDICT(model, x...) to tensor instructions (operator_plan.cpp:
// 521-577: PackCols, MatMul, Compare, Cast, ExpF64, Gather - the Hummingbird
// GEMM tree of ml_model.cpp:154-231 for decision trees, X.w + b [-> sigmoid]
// for linear / logistic models); the B200 executor runs them (MatMul on the
// FP64 tensor cores). Models: the ml_test.cpp fixtures (depth-1 tree,
// constant tree, linear, logistic) and seeded random trees up to depth 8 over
// up to 6 features; tables with NaN / -0.0 / tie-with-threshold features.
// Every query must match tensql::Executor (fp64 within 1e-9; trees exact).
// Test infrastructure (links the oracle); run by tests/test_predict_gpu.py.
//
//   tqp_predict_test [--seed 1] [--rows 20000]
#include <cmath>
#include <cstdio>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "tensql/exec/executor.hpp"
#include "tensql/ml/model.hpp"
#include "tensql/optimizer.hpp"
#include "tensql/sql.hpp"
#include "tensql_b200_executor.hpp"

using namespace tensql;

namespace {

using Rng = std::mt19937_64;

bool close(double a, double b) {
  if (std::isnan(a) || std::isnan(b)) return std::isnan(a) && std::isnan(b);
  if (a == b) return true;
  double m = std::max({1.0, std::fabs(a), std::fabs(b)});
  return std::fabs(a - b) <= 1e-9 * m;
}

std::string diff(const EncodedTable& a, const EncodedTable& b) {
  if (a.columns().size() != b.columns().size()) return "column count differs";
  if (a.row_count() != b.row_count())
    return "row count " + std::to_string(a.row_count()) + " vs " + std::to_string(b.row_count());
  auto ra = decode_table(a), rb = decode_table(b);
  for (size_t i = 0; i < ra.size(); ++i)
    for (size_t c = 0; c < ra[i].size(); ++c) {
      const Cell &x = ra[i][c], &y = rb[i][c];
      bool ok = x.index() == y.index() &&
                (std::holds_alternative<double>(x) ? close(std::get<double>(x), std::get<double>(y)) : x == y);
      if (!ok)
        return "cell mismatch at row " + std::to_string(i) + " column " + a.columns()[c].name + ": " +
               cell_to_text(x, a.columns()[c].logical) + " vs " + cell_to_text(y, b.columns()[c].logical);
    }
  return "";
}

ModelSpec depth1_tree() {  // ml_test.cpp:17-30
  ModelSpec s;
  s.kind = ModelKind::DecisionTree;
  s.nodes.resize(3);
  s.nodes[0].feature = 0;
  s.nodes[0].threshold = 5.0;
  s.nodes[0].left = 1;
  s.nodes[0].right = 2;
  s.nodes[1].is_leaf = true;
  s.nodes[1].leaf_value = 10.0;
  s.nodes[2].is_leaf = true;
  s.nodes[2].leaf_value = 20.0;
  return s;
}

// random full-ish tree: internal nodes split on a random feature at a random
// threshold (sometimes a value the table holds exactly: strict < ties)
ModelSpec random_tree(Rng& r, int features, int depth) {
  ModelSpec s;
  s.kind = ModelKind::DecisionTree;
  std::function<int(int)> grow = [&](int d) -> int {
    const int id = static_cast<int>(s.nodes.size());
    s.nodes.emplace_back();
    if (d == 0 || (d < depth && r() % 5 == 0)) {
      s.nodes[id].is_leaf = true;
      s.nodes[id].leaf_value = static_cast<double>(static_cast<int64_t>(r() % 20001) - 10000) / 8.0;
      return id;
    }
    s.nodes[id].feature = static_cast<int>(r() % features);
    s.nodes[id].threshold = static_cast<double>(static_cast<int64_t>(r() % 2001) - 1000) / 10.0;
    const int l = grow(d - 1);
    const int rr = grow(d - 1);
    s.nodes[id].left = l;
    s.nodes[id].right = rr;
    return id;
  };
  grow(depth);
  return s;
}

int failures = 0, compared = 0;

void check(const std::string& name, const std::string& sql, const Catalog& cat, const TableSet& tables) {
  OperatorPlan op;
  try {
    op = plan_operators(optimize(sql::parse_and_plan(sql, cat), cat), cat);
  } catch (const std::exception& e) {
    std::printf("FAIL %s: planning: %s\n", name.c_str(), e.what());
    ++failures;
    return;
  }
  std::string want_err;
  EncodedTable want;
  try {
    ParallelBackend par;
    want = Executor(op, par).execute(tables);
  } catch (const std::exception& e) {
    want_err = e.what();
  }
  for (bool fuse : {true, false}) {
    std::string got_err;
    EncodedTable got;
    try {
      tqp_integration::B200Executor ex(op, fuse);
      got = ex.execute(tables);
    } catch (const std::exception& e) {
      got_err = e.what();
    }
    const std::string d = !want_err.empty() || !got_err.empty()
                              ? (want_err == got_err ? "" : "error '" + got_err + "' vs '" + want_err + "'")
                              : diff(got, want);
    ++compared;
    if (!d.empty()) {
      ++failures;
      std::printf("FAIL %s [%s]: %s\n", name.c_str(), fuse ? "fused" : "per-instruction", d.c_str());
    }
  }
}

}  // namespace

int main(int argc, char** argv) {
  std::map<std::string, std::string> fl;
  for (int i = 1; i + 1 < argc; i += 2) fl[argv[i]] = argv[i + 1];
  const uint64_t seed = fl.count("--seed") ? std::stoull(fl["--seed"]) : 1;
  const int64_t rows = fl.count("--rows") ? std::stoll(fl["--rows"]) : 20000;
  Rng r(seed);
  const int F = 6;
  TableSchema schema{{"rowid", LogicalType::Int64}};
  for (int f = 0; f < F; ++f) schema.push_back({"f" + std::to_string(f), LogicalType::Float64});
  std::vector<Row> cells;
  for (int64_t i = 0; i < rows; ++i) {
    Row row{i};
    for (int f = 0; f < F; ++f) {
      double v = static_cast<double>(static_cast<int64_t>(r() % 2001) - 1000) / 10.0;
      if (r() % 200 == 0) v = -0.0;
      if (r() % 500 == 0) v = std::nan("");
      row.emplace_back(v);
    }
    cells.push_back(std::move(row));
  }
  TableSet tables{{"t", encode_table(schema, cells)}};
  auto args = [](int n) {
    std::string a;
    for (int f = 0; f < n; ++f) a += ", f" + std::to_string(f);
    return a;
  };
  std::vector<std::pair<std::string, std::pair<ModelSpec, int>>> models;
  models.push_back({"depth1", {depth1_tree(), 1}});
  {
    ModelSpec leaf;
    leaf.kind = ModelKind::DecisionTree;
    leaf.nodes.resize(1);
    leaf.nodes[0].is_leaf = true;
    leaf.nodes[0].leaf_value = 3.5;
    models.push_back({"constant", {leaf, 0}});
  }
  models.push_back({"linear", {load_model_json_text(R"({"kind":"linear","weights":[2.0,-0.5,0.25],"bias":1.0})"), 3}});
  models.push_back(
      {"logistic", {load_model_json_text(R"({"kind":"logistic","weights":[0.01,-0.02,0.03,0.005],"bias":-0.1})"), 4}});
  for (int d = 1; d <= 8; ++d) {
    const int nf = 1 + static_cast<int>(r() % F);
    models.push_back({"tree_d" + std::to_string(d), {random_tree(r, nf, d), nf}});
  }
  for (const auto& [name, mf] : models) {
    Catalog cat;
    cat.add_table("t", schema);
    cat.register_model("m", mf.first);
    const int nargs = mf.first.feature_count();  // the model's arity (highest feature index + 1)
    const std::string call = nargs ? "PREDICT(m" + args(nargs) + ")" : "PREDICT(m)";
    check(name + ": project", "SELECT rowid, " + call + " AS p FROM t", cat, tables);
    check(name + ": sum + count", "SELECT SUM(" + call + ") AS s, COUNT(*) AS n FROM t WHERE f0 > 0", cat, tables);
    check(name + ": filter", "SELECT rowid FROM t WHERE " + call + " > 10", cat, tables);
  }
  std::printf("predict: %zu models, %d comparisons, %d failure(s)\n", models.size(), compared, failures);
  return failures ? 1 : 0;
}
