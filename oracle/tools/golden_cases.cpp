// golden_cases — runs the UNMODIFIED reference (oracle/_ref/libtensql.a) on
// seeded inputs and dumps inputs + outputs (or the reference's error text)
// as JSON fixtures for tests/golden/. Test infrastructure only.
//
//   golden_cases kernels OUT.json   per-kernel cases (kernels.hpp:28-78 +
//                                   executor plumbing); includes the known
//                                   answers of tests/kernels_test.cpp
//   golden_cases plans OUT.json     lowered OperatorPlans + tables + results,
//                                   restating the fixtures of
//                                   tests/executor_test.cpp
#include <cmath>
#include <fstream>
#include <functional>
#include <iostream>
#include <random>

#include "dump.hpp"
#include "tensql/exec/executor.hpp"
#include "tensql/optimizer.hpp"
#include "tensql/sql.hpp"

using namespace tensql;
using namespace tqp_oracle;
using Rng = std::mt19937_64;

namespace {

Tensor i64(std::vector<int64_t> v) { return Tensor::from_vector(std::move(v)); }
Tensor f64(std::vector<double> v) { return Tensor::from_vector(std::move(v)); }
Tensor b8(std::vector<uint8_t> v) { return Tensor::from_vector(std::move(v)); }

std::vector<int64_t> rand_i64(Rng& r, size_t n, int64_t lo, int64_t hi) {
  std::uniform_int_distribution<int64_t> d(lo, hi);
  std::vector<int64_t> v(n);
  for (auto& x : v) x = d(r);
  return v;
}
std::vector<double> rand_f64(Rng& r, size_t n, double lo, double hi) {
  std::uniform_real_distribution<double> d(lo, hi);
  std::vector<double> v(n);
  for (auto& x : v) x = d(r);
  return v;
}
std::vector<uint8_t> rand_mask(Rng& r, size_t n) {
  std::bernoulli_distribution d(0.5);
  std::vector<uint8_t> v(n);
  for (auto& x : v) x = d(r);
  return v;
}
std::string rand_ascii(Rng& r, size_t max_len) {
  std::uniform_int_distribution<size_t> len(0, max_len);
  std::uniform_int_distribution<int> ch(32, 126);
  std::string s(len(r), ' ');
  for (auto& c : s) c = static_cast<char>(ch(r));
  return s;
}

json cases = json::array();

void add_case(const std::string& kernel, json args, const std::function<Tensor()>& run) {
  json c = {{"kernel", kernel}, {"args", args}};
  try {
    c["out"] = tensor_to_json(run());
  } catch (const std::exception& e) {
    c["error"] = e.what();
  }
  cases.push_back(c);
}

const KernelBackend& ref() { return reference_backend(); }

void kernel_cases() {
  auto T = [](const Tensor& t) { return tensor_to_json(t); };
  Rng rng(2024);
  const char* cmp_names[] = {"eq", "ne", "lt", "le", "gt", "ge"};
  const char* ar_names[] = {"add", "sub", "mul", "div"};
  // --- known answers from kernels_test.cpp (re-run through the reference)
  struct KA {
    std::string k;
    std::vector<Tensor> t;
    std::string op;
  };
  auto run_named = [&](const std::string& k, std::vector<Tensor> t, json extra) {
    json args = extra;
    json ts = json::array();
    for (auto& x : t) ts.push_back(T(x));
    args["tensors"] = ts;
    add_case(k, args, [&]() -> Tensor {
      if (k == "compare") return compare(ref(), t[0], t[1], static_cast<CompareOp>(extra["op"].get<int>()));
      if (k == "arith") return arith(ref(), t[0], t[1], static_cast<ArithOp>(extra["op"].get<int>()));
      if (k == "logical") return logical(ref(), t[0], t[1], static_cast<LogicalOp>(extra["op"].get<int>()));
      if (k == "not") return logical_not(ref(), t[0]);
      if (k == "select_where") return select_where(ref(), t[0], t[1], t[2]);
      if (k == "prefix_sum_exclusive") return prefix_sum_exclusive(ref(), t[0]);
      if (k == "compact") return compact(ref(), t[0], t[1]);
      if (k == "argsort_stable") return argsort_stable(ref(), t[0]);
      if (k == "gather") return gather(ref(), t[0], t[1]);
      if (k == "searchsorted")
        return searchsorted(ref(), t[0], t[1], extra["side"].get<int>() ? SearchSide::RIGHT : SearchSide::LEFT);
      if (k == "expand_segments") return expand_segments(ref(), t[0], t[1]);
      if (k == "segment_starts") return segment_starts(ref(), t[0]);
      if (k == "segmented_reduce")
        return segmented_reduce(ref(), t[0], t[1], extra["num"].get<int64_t>(),
                                static_cast<ReduceOp>(extra["op"].get<int>()));
      if (k == "matmul") return matmul(ref(), t[0], t[1]);
      if (k == "substring_match")
        return substring_match(ref(), t[0], extra["pattern"].get<std::string>(),
                               static_cast<MatchAnchor>(extra["anchor"].get<int>()));
      throw std::runtime_error("unknown kernel " + k);
    });
  };
  // compare
  run_named("compare", {i64({1, 5, 3}), Tensor::scalar<int64_t>(4)}, {{"op", 2}});
  run_named("compare", {i64({2, 2}), i64({2, 3})}, {{"op", 0}});
  run_named("compare", {i64({1}), f64({1.0})}, {{"op", 0}});
  run_named("compare", {i64({1, 2}), i64({1, 2, 3})}, {{"op", 0}});
  for (int t = 0; t < 12; ++t) {
    size_t n = 1 + rng() % 300;
    int op = static_cast<int>(rng() % 6);
    if (t % 3 == 0) {
      run_named("compare", {f64(rand_f64(rng, n, -3, 3)), Tensor::scalar<double>(0.5)}, {{"op", op}});
    } else if (t % 3 == 1) {
      run_named("compare", {i64(rand_i64(rng, n, -5, 5)), i64(rand_i64(rng, n, -5, 5))}, {{"op", op}});
    } else {
      auto m = Tensor::from_matrix<int64_t>(static_cast<int64_t>(n), 3, rand_i64(rng, n * 3, 0, 3));
      run_named("compare", {m, Tensor::from_matrix<int64_t>(1, 3, {1, 2, 0})}, {{"op", op}});
    }
  }
  (void)cmp_names;
  (void)ar_names;
  // arith
  run_named("arith", {f64({1.0, 2.0}), f64({3.0, 4.0})}, {{"op", 2}});
  run_named("arith", {f64({1.0}), f64({0.0})}, {{"op", 3}});
  run_named("arith", {f64({1.0, 2.0, 3.0}), f64({1.0, 0.0, 0.0})}, {{"op", 3}});
  run_named("arith", {i64({1}), i64({2})}, {{"op", 3}});
  run_named("arith", {i64({INT64_MAX}), i64({1})}, {{"op", 0}});
  run_named("arith", {i64({5, INT64_MIN, 3}), i64({1, 1, 2})}, {{"op", 1}});
  run_named("arith", {i64({5, 1LL << 40, 3}), i64({1, 1LL << 40, 2})}, {{"op", 2}});
  run_named("arith", {b8({1}), b8({0})}, {{"op", 0}});
  for (int t = 0; t < 12; ++t) {
    size_t n = 1 + rng() % 300;
    int op = static_cast<int>(rng() % 4);
    run_named("arith", {f64(rand_f64(rng, n, -100, 100)), f64(rand_f64(rng, n, 0.5, 9))}, {{"op", op}});
    if (op < 3) run_named("arith", {i64(rand_i64(rng, n, -1000, 1000)), Tensor::scalar<int64_t>(7)}, {{"op", op}});
    if (op < 3) {
      std::vector<int32_t> a(n), b(n);
      for (size_t i = 0; i < n; ++i) {
        a[i] = static_cast<int32_t>(rng() % 100000) - 50000;
        b[i] = static_cast<int32_t>(rng() % 100000);
      }
      run_named("arith", {Tensor::from_vector(a), Tensor::from_vector(b)}, {{"op", op}});
    }
  }
  // logical / not / select_where
  run_named("logical", {b8({1, 0}), b8({1, 1})}, {{"op", 0}});
  run_named("logical", {i64({1}), i64({1})}, {{"op", 0}});
  for (int t = 0; t < 4; ++t) {
    size_t n = 1 + rng() % 200;
    run_named("logical", {b8(rand_mask(rng, n)), b8(rand_mask(rng, n))}, {{"op", t % 2}});
    run_named("not", {b8(rand_mask(rng, n))}, json::object());
  }
  run_named("select_where", {b8({1, 0}), i64({1, 1}), i64({0, 0})}, json::object());
  run_named("select_where", {b8({1, 0}), Tensor::scalar(1.0), Tensor::scalar(0.0)}, json::object());
  run_named("select_where", {b8({1}), i64({1}), f64({1.0})}, json::object());
  run_named("select_where", {b8({1, 0, 1}), Tensor::from_matrix<int32_t>(3, 2, {1, 2, 3, 4, 5, 6}),
                             Tensor::from_matrix<int32_t>(1, 2, {9, 9})},
            json::object());
  for (int t = 0; t < 4; ++t) {
    size_t n = 1 + rng() % 200;
    run_named("select_where", {b8(rand_mask(rng, n)), f64(rand_f64(rng, n, -1, 1)), Tensor::scalar(0.0)},
              json::object());
  }
  // prefix sum
  run_named("prefix_sum_exclusive", {i64({1, 1, 0, 1})}, json::object());
  run_named("prefix_sum_exclusive", {i64({})}, json::object());
  run_named("prefix_sum_exclusive", {i64({INT64_MAX, 1})}, json::object());
  run_named("prefix_sum_exclusive", {i64({5, INT64_MAX - 10, 5, 1, 3})}, json::object());
  for (int t = 0; t < 6; ++t) run_named("prefix_sum_exclusive", {i64(rand_i64(rng, rng() % 1500, -50, 100))}, json::object());
  // compact
  run_named("compact", {i64({10, 20, 30}), b8({1, 0, 1})}, json::object());
  run_named("compact", {i64({4, 5, 6}), b8({0, 0, 0})}, json::object());
  run_named("compact", {Tensor::from_matrix<int32_t>(3, 2, {1, 2, 3, 4, 5, 6}), b8({1, 0, 1})}, json::object());
  run_named("compact", {Tensor::from_matrix<int32_t>(3, 2, {1, 2, 3, 4, 5, 6}), b8({1, 0})}, json::object());
  for (int t = 0; t < 8; ++t) {
    size_t n = rng() % 1500;
    run_named("compact", {f64(rand_f64(rng, n, -100, 100)), b8(rand_mask(rng, n))}, json::object());
  }
  // argsort
  run_named("argsort_stable", {i64({3, 1, 3, 1})}, json::object());
  run_named("argsort_stable", {i64({5, 4, 3, 2})}, json::object());
  run_named("argsort_stable", {f64({1.0, std::nan("")})}, json::object());
  run_named("argsort_stable", {f64({0.0, -0.0, 0.0, -1.5, -0.0})}, json::object());
  for (int t = 0; t < 8; ++t) {
    size_t n = rng() % 1500;
    run_named("argsort_stable", {i64(rand_i64(rng, n, -20, 20))}, json::object());
    run_named("argsort_stable", {f64(rand_f64(rng, n, -1e6, 1e6))}, json::object());
  }
  run_named("argsort_stable", {i64(rand_i64(rng, 1000, INT64_MIN / 2, INT64_MAX / 2))}, json::object());
  // gather
  run_named("gather", {i64({10, 20, 30}), i64({2, 0})}, json::object());
  run_named("gather", {f64({1.0, 2.0, 3.0}), i64({1, 3})}, json::object());
  run_named("gather", {f64({1.0, 2.0, 3.0}), i64({-1})}, json::object());
  run_named("gather", {f64({1.0, 2.0, 3.0}), i64({})}, json::object());
  run_named("gather", {Tensor::from_matrix<int32_t>(3, 2, {1, 2, 3, 4, 5, 6}), i64({2, 2, 0})}, json::object());
  for (int t = 0; t < 4; ++t) {
    size_t n = 1 + rng() % 500;
    run_named("gather", {f64(rand_f64(rng, n, -5, 5)), i64(rand_i64(rng, rng() % 800, 0, n - 1))}, json::object());
  }
  // searchsorted
  run_named("searchsorted", {i64({1, 3, 5}), i64({3})}, {{"side", 0}});
  run_named("searchsorted", {i64({1, 3, 5}), i64({3})}, {{"side", 1}});
  run_named("searchsorted", {i64({1, 3, 5}), i64({0, 9})}, {{"side", 0}});
  run_named("searchsorted", {i64({1, 3}), f64({1.0})}, {{"side", 0}});
  run_named("searchsorted", {i64({3, 1}), i64({2})}, {{"side", 0}});
  for (int t = 0; t < 6; ++t) {
    auto s = rand_i64(rng, rng() % 400, -20, 20);
    std::sort(s.begin(), s.end());
    run_named("searchsorted", {i64(s), i64(rand_i64(rng, rng() % 300, -25, 25))}, {{"side", t % 2}});
  }
  // expand
  run_named("expand_segments", {i64({1}), i64({2})}, json::object());
  run_named("expand_segments", {i64({5, 0}), i64({0, 3})}, json::object());
  run_named("expand_segments", {i64({7, 8}), i64({0, 0})}, json::object());
  run_named("expand_segments", {i64({0}), i64({-1})}, json::object());
  for (int t = 0; t < 4; ++t) {
    size_t k = rng() % 200;
    run_named("expand_segments", {i64(rand_i64(rng, k, 0, 1000)), i64(rand_i64(rng, k, 0, 8))}, json::object());
  }
  // segment starts
  run_named("segment_starts", {i64({1, 1, 2, 2, 2, 5})}, json::object());
  run_named("segment_starts", {Tensor::from_matrix<int64_t>(3, 2, {1, 1, 1, 2, 1, 2})}, json::object());
  for (int t = 0; t < 3; ++t) {
    auto s = rand_i64(rng, rng() % 500, 0, 30);
    std::sort(s.begin(), s.end());
    run_named("segment_starts", {i64(s)}, json::object());
  }
  // segmented reduce
  run_named("segmented_reduce", {i64({1, 2, 3, 4}), i64({0, 0, 1, 1})}, {{"num", 2}, {"op", 0}});
  run_named("segmented_reduce", {f64({1, 1, 1, 1, 1}), i64({0, 0, 0, 0, 0})}, {{"num", 1}, {"op", 1}});
  run_named("segmented_reduce", {i64({5, 1, 9}), i64({0, 0, 0})}, {{"num", 1}, {"op", 2}});
  run_named("segmented_reduce", {i64({5, 1, 9}), i64({0, 0, 0})}, {{"num", 1}, {"op", 3}});
  run_named("segmented_reduce", {i64({4}), i64({1})}, {{"num", 3}, {"op", 0}});
  run_named("segmented_reduce", {i64({4}), i64({1})}, {{"num", 3}, {"op", 2}});
  run_named("segmented_reduce", {i64({1, 2}), i64({1, 0})}, {{"num", 2}, {"op", 0}});
  run_named("segmented_reduce", {i64({1}), i64({5})}, {{"num", 2}, {"op", 0}});
  run_named("segmented_reduce", {i64({INT64_MAX, 1, -1}), i64({0, 0, 0})}, {{"num", 1}, {"op", 0}});
  run_named("segmented_reduce", {i64({1, INT64_MAX, -5, 1}), i64({0, 1, 1, 1})}, {{"num", 2}, {"op", 0}});
  run_named("segmented_reduce", {f64({0.0, -0.0, 3.0}), i64({0, 0, 0})}, {{"num", 1}, {"op", 2}});
  run_named("segmented_reduce", {f64({-0.0, 0.0, 3.0}), i64({0, 0, 0})}, {{"num", 1}, {"op", 2}});
  run_named("segmented_reduce", {f64({2.0, std::nan(""), 3.0}), i64({0, 0, 1})}, {{"num", 2}, {"op", 3}});
  run_named("segmented_reduce", {b8({1, 0}), i64({0, 0})}, {{"num", 1}, {"op", 0}});
  for (int t = 0; t < 8; ++t) {
    size_t n = rng() % 2500;
    int64_t segs = 1 + static_cast<int64_t>(rng() % 12);
    auto ids = rand_i64(rng, n, 0, segs - 1);
    std::sort(ids.begin(), ids.end());
    int op = static_cast<int>(rng() % 4);
    run_named("segmented_reduce", {i64(rand_i64(rng, n, -1000, 1000)), i64(ids)}, {{"num", segs}, {"op", op}});
    run_named("segmented_reduce", {f64(rand_f64(rng, n, -100, 100)), i64(ids)}, {{"num", segs}, {"op", op}});
  }
  // matmul
  run_named("matmul", {Tensor::from_matrix<double>(1, 2, {1, 2}), Tensor::from_matrix<double>(2, 1, {3, 4})},
            json::object());
  run_named("matmul", {Tensor::from_matrix<double>(3, 2, {1, 2, 3, 4, 5, 6}),
                       Tensor::from_matrix<double>(3, 2, {1, 2, 3, 4, 5, 6})},
            json::object());
  // substring match
  run_named("substring_match", {encode_string_rows({"PROMO BRUSHED", "STANDARD"})},
            {{"pattern", "PROMO"}, {"anchor", 0}});
  run_named("substring_match", {encode_string_rows({"PROMO", "PLAIN"})}, {{"pattern", "OM"}, {"anchor", 2}});
  run_named("substring_match", {encode_string_rows({"PROMO", "PLAIN"})}, {{"pattern", "PROMOTION"}, {"anchor", 2}});
  run_named("substring_match", {encode_string_rows({"", "x"})}, {{"pattern", ""}, {"anchor", 2}});
  run_named("substring_match", {encode_string_rows({"", "x"})}, {{"pattern", ""}, {"anchor", 3}});
  for (int t = 0; t < 6; ++t) {
    std::vector<std::string> strs(1 + rng() % 60);
    for (auto& s : strs) s = rand_ascii(rng, 12);
    std::string pat = rand_ascii(rng, 2);
    run_named("substring_match", {encode_string_rows(strs)}, {{"pattern", pat}, {"anchor", t % 4}});
  }
}

// ---- plan-level cases ---------------------------------------------------------
json plan_cases = json::array();

void add_plan_case(const std::string& name, const PlanPtr& plan, const Catalog& cat, const TableSet& tables,
                   bool optimized = false) {
  json c = {{"name", name}};
  PlanPtr p = optimized ? optimize(plan, cat) : plan;
  OperatorPlan op = plan_operators(p, cat);
  c["opplan"] = opplan_to_json(op);
  json tj = json::object();
  for (const auto& [n, t] : tables) tj[n] = table_to_json(t);
  c["tables"] = tj;
  try {
    Executor ex(op, reference_backend());
    c["result"] = table_to_json(ex.execute(tables));
    ParallelBackend par(4);
    Executor exp(op, par);
    c["result_par"] = table_to_json(exp.execute(tables));
  } catch (const std::exception& e) {
    c["error"] = e.what();
  }
  plan_cases.push_back(c);
}

TableSchema lineitem5() {
  return {{"l_partkey", LogicalType::Int64},
          {"l_quantity", LogicalType::Int64},
          {"l_extendedprice", LogicalType::Float64},
          {"l_discount", LogicalType::Float64},
          {"l_shipdate", LogicalType::Date}};
}

void plan_cases_all(const std::string& qdir) {
  auto read = [&](const std::string& f) {
    std::ifstream in(qdir + "/" + f);
    std::stringstream ss;
    ss << in.rdbuf();
    return ss.str();
  };
  Catalog tpch;
  tpch.add_table("lineitem", lineitem5());
  tpch.add_table("part", {{"p_partkey", LogicalType::Int64}, {"p_type", LogicalType::Utf8}});
  // Q6 fixture (fixtures.hpp:46-60): revenue 2155.0
  std::vector<Row> q6rows = {
      {int64_t{1}, int64_t{10}, 1000.0, 0.05, std::string("1994-03-15")},
      {int64_t{2}, int64_t{30}, 2000.0, 0.06, std::string("1994-06-01")},
      {int64_t{3}, int64_t{23}, 1500.0, 0.07, std::string("1994-12-31")},
      {int64_t{4}, int64_t{5}, 800.0, 0.04, std::string("1994-05-20")},
      {int64_t{5}, int64_t{5}, 800.0, 0.06, std::string("1995-01-01")},
      {int64_t{6}, int64_t{1}, 40000.0, 0.05, std::string("1994-01-01")},
  };
  TableSet q6t{{"lineitem", encode_table(lineitem5(), q6rows)}};
  std::string q6 = read("q6.sql"), q14 = read("q14.sql");
  add_plan_case("q6_fixture", sql::parse_and_plan(q6, tpch), tpch, q6t);
  add_plan_case("q6_fixture_opt", sql::parse_and_plan(q6, tpch), tpch, q6t, true);
  // Q14 fixture (executor_test.cpp:71-98)
  std::vector<Row> li{
      {int64_t{1}, int64_t{5}, 1000.0, 0.10, std::string("1995-09-10")},
      {int64_t{2}, int64_t{7}, 2000.0, 0.00, std::string("1995-09-20")},
      {int64_t{3}, int64_t{9}, 3000.0, 0.50, std::string("1995-10-01")},
      {int64_t{1}, int64_t{2}, 500.0, 0.20, std::string("1995-09-30")},
  };
  std::vector<Row> pa{{int64_t{1}, std::string("PROMO BRUSHED TIN")},
                      {int64_t{2}, std::string("STANDARD POLISHED COPPER")},
                      {int64_t{3}, std::string("PROMO PLATED BRASS")}};
  TableSet q14t{{"lineitem", encode_table(lineitem5(), li)},
                {"part", encode_table({{"p_partkey", LogicalType::Int64}, {"p_type", LogicalType::Utf8}}, pa)}};
  add_plan_case("q14_fixture", sql::parse_and_plan(q14, tpch), tpch, q14t);
  add_plan_case("q14_fixture_opt", sql::parse_and_plan(q14, tpch), tpch, q14t, true);
  // filter edge cases (executor_test.cpp:100-114)
  add_plan_case("filter_all", sql::parse_and_plan("SELECT l_partkey FROM lineitem WHERE 1 < 2", tpch), tpch, q6t);
  add_plan_case("filter_none", sql::parse_and_plan("SELECT l_partkey FROM lineitem WHERE 2 < 1", tpch), tpch, q6t);
  add_plan_case("filter_empty_input", sql::parse_and_plan("SELECT l_partkey FROM lineitem WHERE 1 < 2", tpch), tpch,
                TableSet{{"lineitem", encode_table(lineitem5(), {})}});
  // join order (executor_test.cpp:116-153)
  {
    Catalog c;
    c.add_table("l", {{"lk", LogicalType::Int64}, {"lv", LogicalType::Int64}});
    c.add_table("r", {{"rk", LogicalType::Int64}, {"rv", LogicalType::Int64}});
    PlanPtr plan = make_join(make_scan("l"), make_scan("r"), "lk", "rk");
    TableSchema ls{{"lk", LogicalType::Int64}, {"lv", LogicalType::Int64}};
    TableSchema rs{{"rk", LogicalType::Int64}, {"rv", LogicalType::Int64}};
    auto mk = [](TableSchema s, std::vector<std::pair<int64_t, int64_t>> rows) {
      std::vector<Row> out;
      for (auto [a, b] : rows) out.push_back({a, b});
      return encode_table(s, out);
    };
    TableSet t{{"l", mk(ls, {{2, 100}, {1, 101}, {2, 102}, {9, 103}})}, {"r", mk(rs, {{2, 201}, {1, 202}, {2, 203}, {1, 204}})}};
    add_plan_case("join_order", plan, c, t);
    add_plan_case("join_empty_right", plan, c, TableSet{{"l", t.at("l")}, {"r", mk(rs, {})}});
    add_plan_case("join_disjoint", plan, c, TableSet{{"l", mk(ls, {{1, 1}})}, {"r", mk(rs, {{2, 2}})}});
  }
  // zipf join (executor_test.cpp:155-179)
  {
    Catalog c;
    c.add_table("l", {{"k", LogicalType::Int64}, {"lv", LogicalType::Int64}});
    c.add_table("r", {{"k", LogicalType::Int64}, {"rv", LogicalType::Int64}});
    PlanPtr plan = make_join(make_scan("l"), make_scan("r"), "k", "k");
    Rng rng(77);
    for (int trial = 0; trial < 3; ++trial) {
      auto zipf = [&](size_t n, int64_t domain) {
        std::vector<double> w(domain);
        for (size_t i = 0; i < w.size(); ++i) w[i] = 1.0 / std::pow(double(i + 1), 1.2);
        std::discrete_distribution<int64_t> d(w.begin(), w.end());
        std::vector<int64_t> v(n);
        for (auto& x : v) x = d(rng) + 1;
        return v;
      };
      auto lk = zipf(80, 8), rk = zipf(60, 8);
      std::vector<Row> lr, rr;
      for (size_t i = 0; i < lk.size(); ++i) lr.push_back({lk[i], int64_t(i)});
      for (size_t i = 0; i < rk.size(); ++i) rr.push_back({rk[i], int64_t(1000 + i)});
      TableSet t{{"l", encode_table({{"k", LogicalType::Int64}, {"lv", LogicalType::Int64}}, lr)},
                 {"r", encode_table({{"k", LogicalType::Int64}, {"rv", LogicalType::Int64}}, rr)}};
      add_plan_case("join_zipf_" + std::to_string(trial), plan, c, t);
    }
  }
  // multi-key string group-by, 5 aggregates (executor_test.cpp:181-214)
  {
    Catalog c;
    TableSchema s{{"g", LogicalType::Utf8}, {"h", LogicalType::Int64}, {"x", LogicalType::Float64}, {"n", LogicalType::Int64}};
    c.add_table("t", s);
    PlanPtr plan = make_aggregate(make_scan("t"), {"g", "h"},
                                  {{"s", AggFn::Sum, col("x")},
                                   {"c", AggFn::Count, col("n")},
                                   {"a", AggFn::Avg, col("x")},
                                   {"lo", AggFn::Min, col("n")},
                                   {"hi", AggFn::Max, col("n")}});
    Rng rng(99);
    const char* groups[] = {"alpha", "beta", "gamma", "a", "ab", "\xc3\xa9"};
    for (int trial = 0; trial < 3; ++trial) {
      std::vector<Row> rows;
      size_t n = 20 + rng() % 120;
      for (size_t i = 0; i < n; ++i) {
        rows.push_back({std::string(groups[rng() % 6]), static_cast<int64_t>(rng() % 3), rand_f64(rng, 1, -50, 50)[0],
                        static_cast<int64_t>(rng() % 1000)});
      }
      add_plan_case("groupby_strings_" + std::to_string(trial), plan, c, TableSet{{"t", encode_table(s, rows)}});
    }
  }
  // zero-row aggregates (executor_test.cpp:216-238)
  {
    Catalog c;
    c.add_table("t", {{"x", LogicalType::Float64}});
    TableSet t{{"t", encode_table({{"x", LogicalType::Float64}}, {})}};
    add_plan_case("agg_zero_rows",
                  make_aggregate(make_scan("t"), {}, {{"s", AggFn::Sum, col("x")}, {"n", AggFn::Count, col("x")}}), c, t);
    add_plan_case("agg_zero_rows_min", make_aggregate(make_scan("t"), {}, {{"v", AggFn::Min, col("x")}}), c, t);
    add_plan_case("agg_zero_rows_avg", make_aggregate(make_scan("t"), {}, {{"v", AggFn::Avg, col("x")}}), c, t);
    add_plan_case("agg_zero_rows_keyed", make_aggregate(make_scan("t"), {"x"}, {{"v", AggFn::Min, col("x")}}), c, t);
  }
  // sort: multi-key, mixed directions, strings (executor_test.cpp:240-265)
  {
    Catalog c;
    TableSchema s{{"a", LogicalType::Int64}, {"s", LogicalType::Utf8}, {"x", LogicalType::Float64}, {"id", LogicalType::Int64}};
    c.add_table("t", s);
    Rng rng(123);
    int k = 0;
    for (auto dirs : std::vector<std::pair<bool, bool>>{{true, true}, {false, true}, {true, false}, {false, false}}) {
      PlanPtr plan = make_sort(make_scan("t"), {{"a", dirs.first}, {"s", dirs.second}});
      std::vector<Row> rows;
      const char* words[] = {"pear", "fig", "fig", "apple", "", "p\xc3\xa9" "che"};
      for (int i = 0; i < 60; ++i) {
        rows.push_back({static_cast<int64_t>(rng() % 4), std::string(words[rng() % 6]), rand_f64(rng, 1, -5, 5)[0],
                        static_cast<int64_t>(i)});
      }
      add_plan_case("sort_mixed_" + std::to_string(k++), plan, c, TableSet{{"t", encode_table(s, rows)}});
    }
    // fp64 sort keys with ties
    std::vector<Row> rows;
    for (int i = 0; i < 50; ++i) {
      rows.push_back({int64_t(i % 3), std::string("w"), double(int(rng() % 5)) - 2.0, int64_t(i)});
    }
    add_plan_case("sort_f64_desc", make_sort(make_scan("t"), {{"x", false}, {"a", true}}), c,
                  TableSet{{"t", encode_table(s, rows)}});
  }
  // limit (executor_test.cpp:267-283)
  for (int64_t kk : {0, 3, 100}) add_plan_case("limit_" + std::to_string(kk), make_limit(make_scan("lineitem"), kk), tpch, q6t);
  // string predicates + CASE (executor_test.cpp:285-316)
  {
    Catalog c;
    TableSchema s{{"s", LogicalType::Utf8}, {"x", LogicalType::Float64}};
    c.add_table("t", s);
    std::vector<Row> rows{{std::string("PROMO TIN"), 1.0}, {std::string("STANDARD"), 2.0}, {std::string("PROMO"), 3.0},
                          {std::string(""), 4.0}, {std::string("abc PROMO"), 5.0}};
    TableSet t{{"t", encode_table(s, rows)}};
    int k = 0;
    for (const char* q : {"SELECT x FROM t WHERE s LIKE 'PROMO%'", "SELECT x FROM t WHERE s LIKE '%PROMO'",
                          "SELECT x FROM t WHERE s LIKE '%PROMO%'", "SELECT x FROM t WHERE s LIKE 'PROMO'",
                          "SELECT x FROM t WHERE s LIKE '%'", "SELECT x FROM t WHERE s = 'PROMO'",
                          "SELECT x FROM t WHERE s <> ''", "SELECT x FROM t WHERE s < 'PROMO'",
                          "SELECT x FROM t WHERE s >= 'PROMO'",
                          "SELECT CASE WHEN s LIKE 'PROMO%' THEN s ELSE 'other things' END AS tag FROM t",
                          "SELECT CASE WHEN x > 2.5 THEN 'big' ELSE s END AS tag FROM t",
                          "SELECT x FROM t WHERE NOT (x > 2.5 AND s LIKE 'PROMO%')",
                          "SELECT s, SUM(x) AS sx, MIN(x) AS mn, MAX(x) AS mx FROM t GROUP BY s"}) {
      add_plan_case("strings_" + std::to_string(k++), sql::parse_and_plan(q, c), c, t);
    }
  }
  // runtime error carries the operator id (executor_test.cpp:374-388)
  {
    Catalog c;
    c.add_table("t", {{"x", LogicalType::Float64}});
    TableSet t{{"t", encode_table({{"x", LogicalType::Float64}}, {{1.0}, {0.0}})}};
    add_plan_case("div_zero_error", sql::parse_and_plan("SELECT 1.0 / x AS inv FROM t", c), c, t);
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::cerr << "usage: golden_cases kernels|plans OUT.json [QDIR]\n";
    return 2;
  }
  std::string mode = argv[1];
  std::ofstream out(argv[2]);
  if (mode == "kernels") {
    kernel_cases();
    out << json({{"generator", "oracle/tools/golden_cases.cpp (reference libtensql, ref backend)"}, {"cases", cases}}).dump()
        << "\n";
  } else {
    plan_cases_all(argc > 3 ? argv[3] : "oracle/_ref/queries");
    out << json({{"generator", "oracle/tools/golden_cases.cpp (reference libtensql)"}, {"cases", plan_cases}}).dump()
        << "\n";
  }
  return 0;
}
