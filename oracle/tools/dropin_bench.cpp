// tqp_dropin_bench - the drop-in path a tensql caller gets, timed end to end:
// host EncodedTables (the reference's layout, pageable std::vectors) ->
// tqp_integration::B200Executor::execute(TableSet) (uploads the columns the
// plan loads, Utf8 narrowed on the host; runs; downloads the result) ->
// EncodedTable, median wall time per query, next to tensql::Executor (par) on
// the same tables. Bench infrastructure (bench.py's `dropin_e2e` leg).
//
//   tqp_dropin_bench [--sf 1] [--reps 5] [--qdir DIR]
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <fstream>
#include <map>
#include <sstream>
#include <thread>

#include "tensql/exec/executor.hpp"
#include "tensql/optimizer.hpp"
#include "tensql/plan_json.hpp"
#include "tensql/sql.hpp"
#include "tensql_b200_executor.hpp"
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
double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v.empty() ? 0.0 : v[v.size() / 2];
}
}  // namespace

int main(int argc, char** argv) {
  std::map<std::string, std::string> fl;
  for (int i = 1; i + 1 < argc; i += 2) fl[argv[i]] = argv[i + 1];
  const double sf = fl.count("--sf") ? std::stod(fl["--sf"]) : 1.0;
  const int reps = fl.count("--reps") ? std::stoi(fl["--reps"]) : 5;
  std::string exe = argv[0];
  const std::string qdir = fl.count("--qdir") ? fl["--qdir"] : exe.substr(0, exe.rfind('/')) + "/queries";
  Catalog cat = tqp_oracle::tpch_catalog();
  const double g0 = now_ms();
  TableSet tables = tqp_oracle::tpch_tables(sf, 7);
  const double gen_ms = now_ms() - g0;
  const int64_t L = tables.at("lineitem").row_count();
  std::printf("{\"sf\": %g, \"lineitem_rows\": %lld, \"host_gen_ms\": %.1f, \"threads\": %u, \"queries\": {", sf,
              static_cast<long long>(L), gen_ms, std::thread::hardware_concurrency());
  bool first = true;
  for (const std::string q : {"q1", "q6", "q14", "q3"}) {
    PlanPtr plan = q == "q3" ? plan_from_json(read_file(qdir + "/q3.json")) : sql::parse_and_plan(read_file(qdir + "/" + q + ".sql"), cat);
    OperatorPlan op = plan_operators(optimize(plan, cat), cat);
    tqp_integration::B200Executor ex(op);
    for (int i = 0; i < 2; ++i) ex.execute(tables);
    std::vector<double> t;
    for (int i = 0; i < reps; ++i) {
      const double a = now_ms();
      EncodedTable out = ex.execute(tables);
      t.push_back(now_ms() - a);
    }
    ParallelBackend par;
    Executor ref(op, par);
    ref.execute(tables);
    std::vector<double> rt;
    for (int i = 0; i < std::max(1, reps / 2); ++i) {
      const double a = now_ms();
      EncodedTable out = ref.execute(tables);
      rt.push_back(now_ms() - a);
    }
    const double m = median(t), rm = median(rt);
    std::printf("%s\"%s\": {\"b200_ms\": %.3f, \"b200_rows_per_s\": %.4g, \"reference_ms\": %.3f, \"reference_rows_per_s\": %.4g, "
                "\"speedup\": %.1f, \"fallbacks\": %lld}",
                first ? "" : ", ", q.c_str(), m, L / (m / 1e3), rm, L / (rm / 1e3), rm / m, ex.fallbacks());
    first = false;
  }
  std::printf("}}\n");
  return 0;
}
