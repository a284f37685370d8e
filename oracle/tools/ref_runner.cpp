// tqp_ref_runner — drives the UNMODIFIED reference library (oracle/_ref/
// libtensql.a, built from /root/reference/proj/src) through its public API:
// sql::parse_and_plan / plan_from_json -> optimize -> plan_operators ->
// Executor(plan, backend).execute (executor.hpp:43-59). Test/bench
// infrastructure only: it is the CPU baseline arm of bench.py and the
// generator of the golden fixtures under tests/golden/.
//
//   tqp_ref_runner run    --sf 0.01 --queries q1,q3,q6,q14 --backend par
//                         [--threads N] [--repeat 5] [--warmup 5] [--seed 7]
//                         [--qdir DIR] [--results FILE]
//   tqp_ref_runner opplan --qdir DIR --out DIR     (lowered OperatorPlans)
//   tqp_ref_runner tables --sf 0.001 --out FILE    (generated tables as JSON)
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "dump.hpp"
#include "tensql/exec/executor.hpp"
#include "tensql/optimizer.hpp"
#include "tensql/plan_json.hpp"
#include "tensql/sql.hpp"
#include "tpch_tables.hpp"

using namespace tensql;
using namespace tqp_oracle;

namespace {

std::string read_file(const std::string& p) {
  std::ifstream in(p);
  if (!in) throw std::runtime_error("cannot open " + p);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

std::vector<std::string> split(const std::string& s, char d) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string x;
  while (std::getline(ss, x, d))
    if (!x.empty()) out.push_back(x);
  return out;
}

PlanPtr query_plan(const std::string& qdir, const std::string& q, const Catalog& cat) {
  if (q == "q3") return plan_from_json(read_file(qdir + "/q3.json"));
  return sql::parse_and_plan(read_file(qdir + "/" + q + ".sql"), cat);
}

std::string exe_dir(const char* argv0) {
  std::string s = argv0;
  auto p = s.rfind('/');
  return p == std::string::npos ? std::string(".") : s.substr(0, p);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: tqp_ref_runner run|opplan|tables [flags]\n");
    return 2;
  }
  std::string mode = argv[1];
  std::map<std::string, std::string> fl;
  for (int i = 2; i + 1 < argc; i += 2) fl[argv[i]] = argv[i + 1];
  auto get = [&](const char* k, std::string d) { return fl.count(k) ? fl[k] : d; };
  std::string qdir = get("--qdir", exe_dir(argv[0]) + "/queries");
  uint64_t seed = std::stoull(get("--seed", "7"));
  double sf = std::stod(get("--sf", "0.01"));
  Catalog cat = tpch_catalog();

  try {
    if (mode == "opplan") {
      std::string out = get("--out", ".");
      // qg: GROUP BY l_partkey (2 M groups at SF10), the hash-group workload
      for (const std::string q : {"q1", "q3", "q6", "q14", "qg"}) {
        PlanPtr plan = optimize(query_plan(qdir, q, cat), cat);
        OperatorPlan op = plan_operators(plan, cat);
        std::ofstream f(out + "/" + q + ".opplan.json");
        f << opplan_to_json(op).dump(1) << "\n";
      }
      return 0;
    }
    if (mode == "tables") {
      TableSet ts = tpch_tables(sf, seed);
      json j;
      for (auto& [name, t] : ts) j[name] = table_to_json(t);
      std::ofstream f(get("--out", "tables.json"));
      f << j.dump() << "\n";
      return 0;
    }
    if (mode != "run") throw std::runtime_error("unknown mode " + mode);

    std::string backend = get("--backend", "par");
    int threads = std::stoi(get("--threads", "0"));
    int repeat = std::stoi(get("--repeat", "5"));
    int warmup = std::stoi(get("--warmup", "5"));
    auto queries = split(get("--queries", "q1,q3,q6,q14"), ',');
    std::unique_ptr<ParallelBackend> par;
    const KernelBackend* be = &reference_backend();
    if (backend == "par") {
      par = std::make_unique<ParallelBackend>(threads);
      be = par.get();
    }

    auto t0 = std::chrono::steady_clock::now();
    TableSet ts = tpch_tables(sf, seed);
    double gen_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    int64_t L = ts["lineitem"].row_count();

    json results = json::object();
    for (const auto& q : queries) {
      PlanPtr plan = optimize(query_plan(qdir, q, cat), cat);
      Executor ex(plan_operators(plan, cat), *be);
      EncodedTable res;
      for (int i = 0; i < warmup; ++i) res = ex.execute(ts);
      std::vector<double> ms;
      for (int i = 0; i < repeat; ++i) {
        auto a = std::chrono::steady_clock::now();
        res = ex.execute(ts);
        auto b = std::chrono::steady_clock::now();
        ms.push_back(std::chrono::duration<double, std::milli>(b - a).count());
      }
      if (ms.empty()) res = ex.execute(ts);
      std::vector<double> sorted = ms;
      std::sort(sorted.begin(), sorted.end());
      double med = sorted.empty() ? 0.0 : sorted[sorted.size() / 2];
      json line = {{"query", q},       {"sf", sf},          {"seed", seed},
                   {"backend", backend}, {"threads", be->threads()},
                   {"lineitem_rows", L}, {"times_ms", ms},   {"median_ms", med},
                   {"gen_s", gen_s}};
      std::cout << line.dump() << std::endl;
      results[q] = table_to_json(res);
    }
    if (fl.count("--results")) {
      std::ofstream f(fl["--results"]);
      json j = {{"sf", sf}, {"seed", seed}, {"lineitem_rows", L}, {"results", results}};
      f << j.dump(1) << "\n";
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
