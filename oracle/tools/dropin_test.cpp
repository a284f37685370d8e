// tqp_dropin_test — the drop-in proof: the reference's own SQL frontend,
// optimizer and lowering (unchanged, oracle/_ref/libtensql.a) produce an
// OperatorPlan; integration/tensql_b200_executor.hpp runs it on the B200 and
// the result is compared with tensql::Executor on the same TableSet.
// Test infrastructure (links the oracle); run by tests/test_dropin_gpu.py.
//
//   tqp_dropin_test [--sf 0.01] [--qdir DIR]
#include <cmath>
#include <cstdio>
#include <fstream>
#include <map>
#include <sstream>

#include "tensql/exec/executor.hpp"
#include "tensql/optimizer.hpp"
#include "tensql/plan_json.hpp"
#include "tensql/sql.hpp"
#include "tensql_b200_executor.hpp"
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

// tables_diff_ordered (tests/support/table_compare.hpp:37-64)
std::string diff(const EncodedTable& a, const EncodedTable& b) {
  if (a.columns().size() != b.columns().size()) return "column count differs";
  if (a.row_count() != b.row_count())
    return "row count " + std::to_string(a.row_count()) + " vs " + std::to_string(b.row_count());
  auto ra = decode_table(a), rb = decode_table(b);
  for (size_t i = 0; i < ra.size(); ++i) {
    for (size_t c = 0; c < ra[i].size(); ++c) {
      const Cell &x = ra[i][c], &y = rb[i][c];
      bool ok = x.index() == y.index() &&
                (std::holds_alternative<double>(x) ? close(std::get<double>(x), std::get<double>(y)) : x == y);
      if (!ok) return "cell mismatch at row " + std::to_string(i) + " column " + a.columns()[c].name;
    }
  }
  return "";
}

int failures = 0;
int g_gpus = 1;  // --gpus: ranks of the sharded drop-in executor

void check(const std::string& name, const PlanPtr& plan, const Catalog& cat, const TableSet& tables) {
  OperatorPlan op = plan_operators(optimize(plan, cat), cat);
  std::string want_err, got_err;
  EncodedTable want, got;
  try {
    ParallelBackend par;
    want = Executor(op, par).execute(tables);
  } catch (const std::exception& e) {
    want_err = e.what();
  }
  for (int mode = 0; mode < 3; ++mode) {
    // 0 fused, 1 per instruction, 2 fused over g_gpus ranks (row shards of
    // every table, tqp_executor_execute_sharded), when g_gpus > 1
    if (mode == 2 && g_gpus < 2) break;
    const bool fuse = mode != 1;
    try {
      tqp_integration::B200Executor ex(op, mode == 2 ? g_gpus : 1, fuse);
      if (mode == 0) {
        ProfileTrace tr;
        got = ex.profile_execute(tables, tr);
        if (tr.backend != "b200" || tr.operators.empty()) throw std::runtime_error("profile_execute left the trace empty");
      } else {
        got = ex.execute(tables);
      }
      got_err.clear();
    } catch (const std::exception& e) {
      got_err = e.what();
    }
    std::string d = !want_err.empty() || !got_err.empty() ? (want_err == got_err ? "" : "error '" + got_err + "' vs '" + want_err + "'")
                                                          : diff(got, want);
    std::printf("%s %s [%s]%s%s\n", d.empty() ? "PASS" : "FAIL", name.c_str(),
                mode == 2 ? ("fused x" + std::to_string(g_gpus) + " ranks").c_str() : fuse ? "fused" : "per-instruction",
                d.empty() ? "" : ": ", d.c_str());
    if (!d.empty()) ++failures;
  }
}

}  // namespace

int main(int argc, char** argv) {
  std::map<std::string, std::string> fl;
  for (int i = 1; i + 1 < argc; i += 2) fl[argv[i]] = argv[i + 1];
  const double sf = fl.count("--sf") ? std::stod(fl["--sf"]) : 0.01;
  g_gpus = fl.count("--gpus") ? std::stoi(fl["--gpus"]) : 1;
  std::string exe = argv[0];
  const std::string qdir = fl.count("--qdir") ? fl["--qdir"] : exe.substr(0, exe.rfind('/')) + "/queries";
  try {
    Catalog cat = tqp_oracle::tpch_catalog();
    TableSet tables = tqp_oracle::tpch_tables(sf, 7);
    for (const std::string q : {"q6", "q14", "q1"}) check(q, sql::parse_and_plan(read_file(qdir + "/" + q + ".sql"), cat), cat, tables);
    check("q3", plan_from_json(read_file(qdir + "/q3.json")), cat, tables);
    // the SQL frontend extension (ORDER BY, n-way joins): Q3 written in SQL,
    // and ORDER BY over grouped / joined statements, through the same path
    check("q3.sql (tensql_sql_ext)", tqp_sqlx::parse_and_plan(read_file(qdir + "/q3.sql"), cat), cat, tables);
    for (const char* q : {
             "SELECT l_returnflag, l_linestatus, SUM(l_quantity) AS q, COUNT(*) AS n FROM lineitem GROUP BY "
             "l_returnflag, l_linestatus ORDER BY q DESC",
             "SELECT c_mktsegment, SUM(l_extendedprice * (1 - l_discount)) AS rev, COUNT(*) AS n FROM customer JOIN "
             "orders ON o_custkey = c_custkey JOIN lineitem ON l_orderkey = o_orderkey WHERE o_orderdate < DATE "
             "'1995-03-15' GROUP BY c_mktsegment ORDER BY rev DESC",
             "SELECT o_orderkey, o_orderdate FROM orders JOIN customer ON o_custkey = c_custkey WHERE c_mktsegment = "
             "'MACHINERY' ORDER BY o_orderdate DESC, o_orderkey LIMIT 20",
         }) {
      check(std::string("sqlx: ") + q, tqp_sqlx::parse_and_plan(q, cat), cat, tables);
    }
    // ad-hoc SQL the reference frontend accepts, through the same path
    for (const char* q : {
             "SELECT l_returnflag, COUNT(*) AS n, SUM(l_quantity) AS q FROM lineitem WHERE l_discount > 0.05 GROUP BY l_returnflag",
             "SELECT SUM(l_extendedprice * l_discount) AS r, AVG(l_tax) AS t FROM lineitem WHERE l_quantity BETWEEN 10 AND 20",
             "SELECT l_orderkey, l_extendedprice FROM lineitem WHERE l_orderkey < 40",
             "SELECT o_orderkey, c_mktsegment FROM orders, customer WHERE o_custkey = c_custkey AND o_orderkey < 30",
             "SELECT 1.0 / (l_discount - l_discount) AS bad FROM lineitem WHERE l_orderkey < 3",
         }) {
      check(q, sql::parse_and_plan(q, cat), cat, tables);
    }
  } catch (const std::exception& e) {
    std::printf("FAIL setup: %s\n", e.what());
    return 1;
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
