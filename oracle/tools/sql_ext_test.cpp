// tqp_sql_ext_test - checks integration/tensql_sql_ext.hpp (ORDER BY and
// n-way joins over the unmodified reference frontend) with the reference
// executor itself: queries/q3.sql planned by the extension returns exactly
// what the committed plan JSON (queries/q3.json) returns; ORDER BY over one-
// and two-table statements equals the reference plan with make_sort added by
// hand; statements the reference accepts plan to the identical plan; errors
// carry the reference's SqlError type. CPU only (run by tests/test_sql_ext.py).
//
//   tqp_sql_ext_test [--sf 0.05] [--qdir DIR]
#include <cmath>
#include <cstdio>
#include <fstream>
#include <map>
#include <sstream>

#include "tensql/exec/executor.hpp"
#include "tensql/optimizer.hpp"
#include "tensql/plan_json.hpp"
#include "tensql/sql.hpp"
#include "tensql_sql_ext.hpp"
#include "tpch_tables.hpp"

using namespace tensql;

namespace {

std::string read_file(const std::string& p) {
  std::ifstream in(p);
  if (!in) throw std::runtime_error("cannot open " + p);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

bool close(double a, double b) {
  if (std::isnan(a) || std::isnan(b)) return std::isnan(a) && std::isnan(b);
  double m = std::max({1.0, std::fabs(a), std::fabs(b)});
  return std::fabs(a - b) <= 1e-9 * m;
}

std::string diff(const EncodedTable& a, const EncodedTable& b) {
  if (a.columns().size() != b.columns().size()) return "column count differs";
  for (size_t c = 0; c < a.columns().size(); ++c)
    if (a.columns()[c].logical != b.columns()[c].logical) return "column type differs at " + std::to_string(c);
  if (a.row_count() != b.row_count())
    return "row count " + std::to_string(a.row_count()) + " vs " + std::to_string(b.row_count());
  auto ra = decode_table(a), rb = decode_table(b);
  for (size_t i = 0; i < ra.size(); ++i)
    for (size_t c = 0; c < ra[i].size(); ++c) {
      const Cell &x = ra[i][c], &y = rb[i][c];
      bool ok = x.index() == y.index() &&
                (std::holds_alternative<double>(x) ? close(std::get<double>(x), std::get<double>(y)) : x == y);
      if (!ok) return "cell mismatch at row " + std::to_string(i) + " column " + a.columns()[c].name;
    }
  return "";
}

int failures = 0;

EncodedTable run(const PlanPtr& p, const Catalog& cat, const TableSet& t) {
  ParallelBackend par;
  return Executor(plan_operators(optimize(p, cat), cat), par).execute(t);
}

void expect_same(const std::string& name, const PlanPtr& got, const PlanPtr& want, const Catalog& cat, const TableSet& t) {
  std::string d;
  size_t rows = 0;
  try {
    EncodedTable a = run(got, cat, t), b = run(want, cat, t);
    d = diff(a, b);
    rows = a.row_count();
  } catch (const std::exception& e) {
    d = std::string("exception: ") + e.what();
  }
  std::printf("%s %s (%zu rows)%s%s\n", d.empty() ? "PASS" : "FAIL", name.c_str(), rows, d.empty() ? "" : ": ", d.c_str());
  if (!d.empty()) ++failures;
}

void expect_error(const std::string& sql, const std::string& fragment, const Catalog& cat) {
  std::string msg = "(no error)";
  try {
    tqp_sqlx::parse_and_plan(sql, cat);
  } catch (const sql::SqlError& e) {
    msg = e.what();
  } catch (const std::exception& e) {
    msg = std::string("wrong exception type: ") + e.what();
  }
  const bool ok = msg.find(fragment) != std::string::npos;
  std::printf("%s error '%s' -> %s\n", ok ? "PASS" : "FAIL", sql.c_str(), msg.c_str());
  if (!ok) ++failures;
}

}  // namespace

int main(int argc, char** argv) {
  std::map<std::string, std::string> fl;
  for (int i = 1; i + 1 < argc; i += 2) fl[argv[i]] = argv[i + 1];
  const double sf = fl.count("--sf") ? std::stod(fl["--sf"]) : 0.05;
  std::string exe = argv[0];
  const std::string qdir = fl.count("--qdir") ? fl["--qdir"] : exe.substr(0, exe.rfind('/')) + "/queries";
  try {
    Catalog cat = tqp_oracle::tpch_catalog();
    TableSet t = tqp_oracle::tpch_tables(sf, 7);
    // Q3 as SQL (three tables, ORDER BY, LIMIT) == the committed plan JSON
    expect_same("q3.sql == q3.json", tqp_sqlx::parse_and_plan(read_file(qdir + "/q3.sql"), cat),
                plan_from_json(read_file(qdir + "/q3.json")), cat, t);
    // comma form of the same chain, WHERE equalities as join keys
    expect_same("q3 comma join",
                tqp_sqlx::parse_and_plan(
                    "SELECT l_orderkey, SUM(l_extendedprice * (1 - l_discount)) AS revenue, o_orderdate, o_shippriority "
                    "FROM customer, orders, lineitem WHERE c_mktsegment = 'BUILDING' AND c_custkey = o_custkey AND "
                    "l_orderkey = o_orderkey AND o_orderdate < DATE '1995-03-15' AND l_shipdate > DATE '1995-03-15' "
                    "GROUP BY l_orderkey, o_orderdate, o_shippriority ORDER BY revenue DESC, o_orderdate LIMIT 10",
                    cat),
                plan_from_json(read_file(qdir + "/q3.json")), cat, t);
    // statements the reference accepts: the identical plan
    for (const std::string q : {"q1", "q6", "q14"}) {
      const std::string s = read_file(qdir + "/" + q + ".sql");
      const bool same = plan_to_json(tqp_sqlx::parse_and_plan(s, cat)) == plan_to_json(sql::parse_and_plan(s, cat));
      std::printf("%s %s plans as the reference frontend\n", same ? "PASS" : "FAIL", q.c_str());
      if (!same) ++failures;
    }
    // ORDER BY over one and two tables == the reference plan + make_sort / make_limit
    const std::string q1 = read_file(qdir + "/q1.sql");
    expect_same("q1 ORDER BY l_returnflag DESC, l_linestatus",
                tqp_sqlx::parse_and_plan(q1 + " ORDER BY l_returnflag DESC, l_linestatus", cat),
                make_sort(sql::parse_and_plan(q1, cat), {{"l_returnflag", false}, {"l_linestatus", true}}), cat, t);
    const std::string j2 =
        "SELECT o_orderkey, o_orderdate, c_mktsegment FROM orders JOIN customer ON o_custkey = c_custkey WHERE "
        "o_orderkey < 2000";
    expect_same("2-table ORDER BY .. LIMIT",
                tqp_sqlx::parse_and_plan(j2 + " ORDER BY c_mktsegment, o_orderdate DESC LIMIT 25", cat),
                make_limit(make_sort(sql::parse_and_plan(j2, cat), {{"c_mktsegment", true}, {"o_orderdate", false}}), 25),
                cat, t);
    expect_same("LIMIT without ORDER BY", tqp_sqlx::parse_and_plan("SELECT l_orderkey FROM lineitem LIMIT 7", cat),
                sql::parse_and_plan("SELECT l_orderkey FROM lineitem LIMIT 7", cat), cat, t);
    // lineitem probes (orders JOIN customer), grouped by a customer column
    const PlanPtr three = tqp_sqlx::parse_and_plan(
        "SELECT c_mktsegment, SUM(l_extendedprice * (1 - l_discount)) AS rev, COUNT(*) AS n "
        "FROM customer JOIN orders ON o_custkey = c_custkey JOIN lineitem ON l_orderkey = o_orderkey "
        "WHERE o_orderdate < DATE '1995-03-15' GROUP BY c_mktsegment ORDER BY rev DESC",
        cat);
    const PlanPtr hand = make_sort(
        make_project(
            make_aggregate(
                make_join(make_scan("lineitem"),
                          make_join(make_filter(make_scan("orders"),
                                                make_compare(CompareOp::LT, col("o_orderdate"), lit_date("1995-03-15"))),
                                    make_scan("customer"), "o_custkey", "c_custkey"),
                          "l_orderkey", "o_orderkey"),
                {"c_mktsegment"},
                {{"rev", AggFn::Sum,
                  make_arith(ArithOp::MUL, col("l_extendedprice"), make_arith(ArithOp::SUB, lit_f64(1.0), col("l_discount")))},
                 {"n", AggFn::Count, lit_i64(1)}}),
            {{"c_mktsegment", col("c_mktsegment")}, {"rev", col("rev")}, {"n", col("n")}}),
        {{"rev", false}});
    expect_same("3-table GROUP BY c_mktsegment ORDER BY rev DESC", three, hand, cat, t);
    expect_error("SELECT l_orderkey FROM lineitem ORDER BY nope", "ORDER BY column 'nope'", cat);
    expect_error("SELECT l_orderkey FROM customer, orders, lineitem WHERE l_orderkey = o_orderkey",
                 "needs an equality with an earlier table", cat);
    expect_error("SELECT l_orderkey FROM lineitem ORDER l_orderkey", "expected BY after ORDER", cat);
    expect_error("SELECT c_custkey, SUM(o_totalprice) FROM customer, orders, lineitem WHERE c_custkey = o_custkey AND "
                 "l_orderkey = o_orderkey GROUP BY c_custkey",
                 "unknown column 'o_totalprice'", cat);
  } catch (const std::exception& e) {
    std::printf("FAIL: %s\n", e.what());
    return 1;
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
