// tqp_random_plans — random-plan parity harness. The
// reference declares a random plan generator (tests/support/random_plans.hpp:
// 12-35) but never implements it; this one builds seeded random tables and
// random well-typed plans over the reference's whole plan API (make_scan /
// make_filter / make_project / make_join / make_aggregate / make_sort /
// make_limit, plan.hpp:76-83; expressions expr.hpp:76-89, typed as
// infer_expr_type, plan.cpp:180-270), lowers them with the reference's own
// optimize + plan_operators, and runs the OperatorPlan on
//   * tensql::Executor with the `par` backend (the oracle), and
//   * the B200 executor through integration/tensql_b200_executor.hpp, fused
//     and per-instruction,
// comparing results as tables_diff_ordered does (fp64 within 1e-9 relative,
// everything else exact, row order included) and errors by their text.
// Test infrastructure (links the oracle); run by tests/test_random_plans_gpu.py.
//
//   tqp_random_plans [--seed 1] [--plans 300] [--verbose 0]
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "tensql/exec/executor.hpp"
#include "tensql/optimizer.hpp"
#include "tensql/plan_json.hpp"
#include "tensql/plan.hpp"
#include "tensql_b200_executor.hpp"

using namespace tensql;

namespace {

using Rng = std::mt19937_64;

int pick(Rng& r, int n) { return static_cast<int>(r() % static_cast<uint64_t>(n)); }
bool chance(Rng& r, double p) { return std::uniform_real_distribution<double>(0, 1)(r) < p; }

const std::vector<std::string> kWords = {"",      "A",        "AB",    "N",     "R",       "PROMO",
                                         "PROMO X", "PROMOTION", "xyzzy", "BUILDING", "MACHINERY", "zz top"};

std::string iso_day(int64_t day) {  // days since 1970-01-01 -> ISO text
  return decode_date(day * 86400LL * 1000000000LL);
}

struct Shape {
  int64_t n_fact, n_dim;
  bool dim_dups, huge_ints, nans;
  // --profile groups: group-key columns k (Int64 over [0, k_range), sparse
  // when k_sparse) and c (short Utf8 codes), dim keys spread over
  // [0, n_dim * dim_spread)
  bool groups = false;
  int64_t k_range = 0;
  bool k_sparse = false;
  int64_t dim_spread = 1;
};

// fact(fk, a, x, d, s, b), dim(dk, y, t, e)
void make_tables(Rng& r, const Shape& sh, Catalog& cat, TableSet& tables) {
  TableSchema fs = {{"fk", LogicalType::Int64}, {"a", LogicalType::Int64}, {"x", LogicalType::Float64},
                    {"d", LogicalType::Date},   {"s", LogicalType::Utf8},  {"b", LogicalType::Bool}};
  if (sh.groups) {
    fs.push_back({"k", LogicalType::Int64});
    fs.push_back({"c", LogicalType::Utf8});
  }
  static const std::vector<std::string> kCodes = {"", "A", "B", "AB", "BA", "ZZ", "Q7", "AIR", "MAIL", "SHIP", "TRUCK",
                                                  "RAIL", "REG", "FOB", "X", "XYZW"};
  // sparse k values: a fixed pool of wide-range keys
  std::vector<int64_t> kpool;
  if (sh.groups && sh.k_sparse)
    for (int64_t i = 0; i < sh.k_range; ++i) kpool.push_back(static_cast<int64_t>(r() >> 20) - (int64_t{1} << 42));
  TableSchema ds = {{"dk", LogicalType::Int64}, {"y", LogicalType::Float64}, {"t", LogicalType::Utf8},
                    {"e", LogicalType::Date}};
  const int64_t d0 = days_from_civil(1992, 1, 1), d1 = days_from_civil(1998, 12, 31);
  std::vector<Row> fr, dr;
  for (int64_t i = 0; i < sh.n_fact; ++i) {
    int64_t a = static_cast<int64_t>(pick(r, 101)) - 50;
    if (sh.huge_ints && chance(r, 0.05)) a = (chance(r, 0.5) ? 1 : -1) * ((int64_t{1} << 62) - pick(r, 1000));
    double x = static_cast<double>(static_cast<int64_t>(pick(r, 20001)) - 10000) / 100.0;
    if (chance(r, 0.03)) x = -0.0;
    if (sh.nans && chance(r, 0.02)) x = std::nan("");
    const int64_t fk_span = sh.n_dim * sh.dim_spread + 4;
    fr.push_back({Cell{static_cast<int64_t>(r() % static_cast<uint64_t>(fk_span))}, Cell{a}, Cell{x},
                  Cell{iso_day(d0 + pick(r, static_cast<int>(d1 - d0 + 1)))}, Cell{kWords[pick(r, kWords.size())]},
                  Cell{chance(r, 0.5)}});
    if (sh.groups) {
      const int64_t kv = sh.k_sparse ? kpool[r() % kpool.size()] : static_cast<int64_t>(r() % static_cast<uint64_t>(sh.k_range));
      fr.back().push_back(Cell{kv});
      fr.back().push_back(Cell{kCodes[pick(r, kCodes.size())]});
    }
  }
  std::vector<int64_t> keys(sh.n_dim);
  for (int64_t i = 0; i < sh.n_dim; ++i)
    keys[i] = sh.dim_dups ? static_cast<int64_t>(r() % static_cast<uint64_t>(sh.n_dim * sh.dim_spread / 2 + 1))
                          : i * sh.dim_spread + (sh.dim_spread > 1 ? pick(r, static_cast<int>(sh.dim_spread)) : 0);
  std::shuffle(keys.begin(), keys.end(), r);
  for (int64_t i = 0; i < sh.n_dim; ++i) {
    dr.push_back({Cell{keys[i]}, Cell{static_cast<double>(pick(r, 100001)) / 100.0}, Cell{kWords[pick(r, kWords.size())]},
                  Cell{iso_day(d0 + pick(r, static_cast<int>(d1 - d0 + 1)))}});
  }
  cat.add_table("fact", fs);
  cat.add_table("dim", ds);
  tables["fact"] = encode_table(fs, fr);
  tables["dim"] = encode_table(ds, dr);
}

// ---- well-typed random expressions ------------------------------------------
struct Gen {
  Rng& r;
  const Schema* schema = nullptr;
  int budget = 0;

  std::vector<std::string> cols_of(LogicalType t) const {
    std::vector<std::string> out;
    for (const auto& c : *schema)
      if (c.type == t) out.push_back(c.name);
    return out;
  }
  ExprPtr literal(LogicalType t) {
    switch (t) {
      case LogicalType::Int64: return lit_i64(static_cast<int64_t>(pick(r, 61)) - 30);
      case LogicalType::Float64: {
        static const double ks[] = {0.0, 1.0, -1.0, 0.5, 2.5, 100.0, 0.05, 50.0, -7.25};
        return lit_f64(ks[pick(r, 9)]);
      }
      case LogicalType::Date: return lit_date(iso_day(days_from_civil(1992, 1, 1) + pick(r, 2555)));
      case LogicalType::Utf8: return lit_str(kWords[pick(r, kWords.size())]);
      default: return lit_bool(chance(r, 0.5));
    }
  }
  ExprPtr value(LogicalType t, int depth) {
    auto cs = cols_of(t);
    if (depth <= 0 || budget <= 0 || chance(r, 0.45)) {
      if (!cs.empty() && !chance(r, 0.25)) return col(cs[pick(r, cs.size())]);
      return literal(t);
    }
    --budget;
    if ((t == LogicalType::Int64 || t == LogicalType::Float64) && chance(r, 0.7)) {
      ArithOp ops[] = {ArithOp::ADD, ArithOp::SUB, ArithOp::MUL, ArithOp::DIV};
      ArithOp op = ops[pick(r, t == LogicalType::Float64 ? 4 : 3)];
      return make_arith(op, value(t, depth - 1), value(t, depth - 1));
    }
    if (t == LogicalType::Bool) return predicate(depth);
    std::vector<CaseExpr::Branch> br;
    const int nb = 1 + pick(r, 2);
    for (int i = 0; i < nb; ++i) br.push_back({predicate(depth - 1), value(t, depth - 1)});
    return make_case(std::move(br), value(t, depth - 1));
  }
  ExprPtr predicate(int depth) {
    if (depth <= 0 || budget <= 0) return compare_leaf();
    --budget;
    switch (pick(r, 7)) {
      case 0: return make_logical(LogicalOp::AND, predicate(depth - 1), predicate(depth - 1));
      case 1: return make_logical(LogicalOp::OR, predicate(depth - 1), predicate(depth - 1));
      case 2: return make_not(predicate(depth - 1));
      case 3: {
        LogicalType ts[] = {LogicalType::Int64, LogicalType::Float64, LogicalType::Date};
        LogicalType t = ts[pick(r, 3)];
        return make_between(value(t, depth - 1), literal(t), literal(t));
      }
      case 4: {
        auto cs = cols_of(LogicalType::Utf8);
        if (cs.empty()) return compare_leaf();
        static const char* pats[] = {"PROMO%", "%X", "%MO%", "A", "%", "BUILDING", "%ING", "PRO%", ""};
        return make_like(col(cs[pick(r, cs.size())]), pats[pick(r, 9)]);
      }
      case 5: {
        auto cs = cols_of(LogicalType::Bool);
        if (!cs.empty()) return col(cs[pick(r, cs.size())]);
        return compare_leaf();
      }
      default: return compare_leaf();
    }
  }
  ExprPtr compare_leaf() {
    LogicalType ts[] = {LogicalType::Int64, LogicalType::Float64, LogicalType::Date, LogicalType::Utf8,
                        LogicalType::Bool};
    LogicalType t = ts[pick(r, 5)];
    CompareOp ops[] = {CompareOp::EQ, CompareOp::NE, CompareOp::LT, CompareOp::LE, CompareOp::GT, CompareOp::GE};
    return make_compare(ops[pick(r, 6)], value(t, 1), value(t, 1));
  }
};

// ---- random plans --------------------------------------------------------------
struct Built {
  PlanPtr plan;
  std::string text;
};

Built random_plan(Rng& r, const Catalog& cat) {
  Built b;
  Gen g{r};
  PlanPtr p = make_scan("fact");
  Schema sch = infer_schema(p, cat);
  std::string txt = "scan(fact)";
  auto refresh = [&] { sch = infer_schema(p, cat); };
  g.schema = &sch;
  if (chance(r, 0.55)) {
    g.budget = 6;
    p = make_filter(p, g.predicate(3));
    txt += " > filter";
    refresh();
  }
  if (chance(r, 0.35)) {
    PlanPtr right = make_scan("dim");
    if (chance(r, 0.4)) {
      Schema ds = infer_schema(right, cat);
      Gen gd{r, &ds, 4};
      right = make_filter(right, gd.predicate(2));
    }
    p = make_join(p, right, "fk", "dk");
    txt += " > join(dim)";
    refresh();
  }
  if (chance(r, 0.45)) {
    std::vector<ProjectNode::Item> items;
    std::vector<std::string> names;
    for (const auto& c : sch)
      if (chance(r, 0.5)) items.push_back({c.name, col(c.name)});
    const int ne = 1 + pick(r, 3);
    LogicalType ts[] = {LogicalType::Int64, LogicalType::Float64, LogicalType::Date, LogicalType::Utf8,
                        LogicalType::Bool};
    for (int i = 0; i < ne; ++i) {
      g.budget = 5;
      items.push_back({"e" + std::to_string(i), g.value(ts[pick(r, 5)], 3)});
    }
    p = make_project(p, std::move(items));
    txt += " > project";
    refresh();
  }
  bool grouped = false;
  std::vector<std::string> exact_sort_cols;  // sort keys whose values are exact
  if (chance(r, 0.5)) {
    std::vector<std::string> keys;
    for (const auto& c : sch)
      if (c.type != LogicalType::Float64 && keys.size() < 2 && chance(r, 0.3)) keys.push_back(c.name);
    std::vector<AggregateNode::Agg> aggs;
    const int na = 1 + pick(r, 3);
    for (int i = 0; i < na; ++i) {
      const std::string name = "g" + std::to_string(i);
      const auto& c = sch[pick(r, sch.size())];
      AggFn fn;
      if (c.type == LogicalType::Int64 || c.type == LogicalType::Float64) {
        AggFn fs[] = {AggFn::Sum, AggFn::Count, AggFn::Avg, AggFn::Min, AggFn::Max};
        fn = fs[pick(r, 5)];
      } else if (c.type == LogicalType::Date) {
        AggFn fs[] = {AggFn::Count, AggFn::Min, AggFn::Max};
        fn = fs[pick(r, 3)];
      } else {
        fn = AggFn::Count;
      }
      // exact on both sides: counts, min/max, int64 sums and averages of int64
      if (fn == AggFn::Count || fn == AggFn::Min || fn == AggFn::Max || c.type == LogicalType::Int64)
        exact_sort_cols.push_back(name);
      aggs.push_back({name, fn, col(c.name)});
    }
    for (const auto& k : keys) exact_sort_cols.push_back(k);
    p = make_aggregate(p, keys, std::move(aggs));
    txt += " > aggregate(" + std::to_string(keys.size()) + " keys)";
    grouped = true;
    refresh();
  } else {
    for (const auto& c : sch) exact_sort_cols.push_back(c.name);
  }
  if (chance(r, 0.45) && !exact_sort_cols.empty()) {
    // fp64 sums/averages are compared within 1e-9, so they are not used as
    // sort keys (two nearly equal sums may legitimately order either way)
    std::vector<SortNode::Key> keys;
    const int nk = 1 + pick(r, 3);
    for (int i = 0; i < nk; ++i) keys.push_back({exact_sort_cols[pick(r, exact_sort_cols.size())], chance(r, 0.5)});
    p = make_sort(p, keys);
    txt += " > sort(" + std::to_string(nk) + ")";
    if (chance(r, 0.6)) {
      p = make_limit(p, pick(r, 25));
      txt += " > limit";
    }
  } else if (!grouped && chance(r, 0.15)) {
    p = make_limit(p, pick(r, 40));
    txt += " > limit";
  }
  b.plan = p;
  b.text = txt;
  return b;
}

// --profile groups: scan(fact) > [filter] > [join(dim)] > aggregate over 1-3
// group keys drawn from the int64 / date / short-string columns (k, c, d, a,
// fk and the dim's dk, e) with SUM / COUNT / AVG (the fused hash-group
// family; MIN/MAX now and then) > [sort > limit]
Built random_group_plan(Rng& r, const Catalog& cat) {
  Built b;
  Gen g{r};
  PlanPtr p = make_scan("fact");
  Schema sch = infer_schema(p, cat);
  std::string txt = "scan(fact)";
  auto refresh = [&] { sch = infer_schema(p, cat); };
  g.schema = &sch;
  if (chance(r, 0.5)) {
    g.budget = 4;
    p = make_filter(p, g.predicate(2));
    txt += " > filter";
    refresh();
  }
  bool joined = false;
  if (chance(r, 0.4)) {
    PlanPtr right = make_scan("dim");
    if (chance(r, 0.3)) {
      Schema ds = infer_schema(right, cat);
      Gen gd{r, &ds, 3};
      right = make_filter(right, gd.predicate(2));
    }
    p = make_join(p, right, "fk", "dk");
    txt += " > join(dim)";
    joined = true;
    refresh();
  }
  std::vector<std::string> pool = {"k", "k", "c", "d", "a", "fk"};
  if (joined) {
    pool.push_back("dk");
    pool.push_back("e");
  }
  std::vector<std::string> keys;
  const int nk = 1 + pick(r, 3);
  for (int i = 0; i < nk; ++i) {
    const std::string k = pool[pick(r, pool.size())];
    if (std::find(keys.begin(), keys.end(), k) == keys.end()) keys.push_back(k);
  }
  std::vector<std::string> vals = {"a", "x", "k"};
  if (joined) vals.push_back("y");
  std::vector<AggregateNode::Agg> aggs;
  std::vector<std::string> exact_sort_cols = keys;
  const int na = 1 + pick(r, 3);
  for (int i = 0; i < na; ++i) {
    const std::string name = "g" + std::to_string(i);
    const std::string c = vals[pick(r, vals.size())];
    AggFn fs[] = {AggFn::Sum, AggFn::Sum, AggFn::Count, AggFn::Avg, AggFn::Min};
    AggFn fn = fs[pick(r, chance(r, 0.9) ? 4 : 5)];
    if (fn == AggFn::Count || fn == AggFn::Min || c == "a" || c == "k") exact_sort_cols.push_back(name);
    aggs.push_back({name, fn, col(c)});
  }
  p = make_aggregate(p, keys, std::move(aggs));
  txt += " > aggregate(" + std::to_string(keys.size()) + " keys)";
  if (chance(r, 0.35)) {
    std::vector<SortNode::Key> sk;
    const int ns = 1 + pick(r, 2);
    for (int i = 0; i < ns; ++i) sk.push_back({exact_sort_cols[pick(r, exact_sort_cols.size())], chance(r, 0.5)});
    p = make_sort(p, sk);
    txt += " > sort(" + std::to_string(ns) + ")";
    if (chance(r, 0.7)) {
      p = make_limit(p, 1 + pick(r, 20));
      txt += " > limit";
    }
  }
  b.plan = p;
  b.text = txt;
  return b;
}

// ---- comparison (tables_diff_ordered, tests/support/table_compare.hpp:37-64) ----
bool close(double a, double b) {
  if (std::isnan(a) || std::isnan(b)) return std::isnan(a) && std::isnan(b);
  if (a == b) return true;
  double m = std::max({1.0, std::fabs(a), std::fabs(b)});
  return std::fabs(a - b) <= 1e-9 * m;
}

std::string diff(const EncodedTable& a, const EncodedTable& b) {
  if (a.columns().size() != b.columns().size()) return "column count differs";
  for (size_t c = 0; c < a.columns().size(); ++c)
    if (a.columns()[c].name != b.columns()[c].name || a.columns()[c].logical != b.columns()[c].logical)
      return "schema differs at column " + std::to_string(c);
  if (a.row_count() != b.row_count())
    return "row count " + std::to_string(a.row_count()) + " vs " + std::to_string(b.row_count());
  auto ra = decode_table(a), rb = decode_table(b);
  for (size_t i = 0; i < ra.size(); ++i) {
    for (size_t c = 0; c < ra[i].size(); ++c) {
      const Cell &x = ra[i][c], &y = rb[i][c];
      bool ok = x.index() == y.index() &&
                (std::holds_alternative<double>(x) ? close(std::get<double>(x), std::get<double>(y)) : x == y);
      if (!ok)
        return "cell mismatch at row " + std::to_string(i) + " column " + a.columns()[c].name + ": " +
               cell_to_text(x, a.columns()[c].logical) + " vs " + cell_to_text(y, b.columns()[c].logical);
    }
  }
  return "";
}

}  // namespace

int main(int argc, char** argv) {
  std::map<std::string, std::string> fl;
  for (int i = 1; i + 1 < argc; i += 2) fl[argv[i]] = argv[i + 1];
  const uint64_t seed = fl.count("--seed") ? std::stoull(fl["--seed"]) : 1;
  const int nplans = fl.count("--plans") ? std::stoi(fl["--plans"]) : 300;
  const bool verbose = fl.count("--verbose") && fl["--verbose"] != "0";
  // --only N: run just plan N of the seeded sequence (the sequence is still
  // generated, so N is the same plan as in the full run) and dump it
  const int only = fl.count("--only") ? std::stoi(fl["--only"]) : -1;
  // --profile groups: wide group-by / join key shapes (random_group_plan);
  // --require-fused 1: a fused unit handing its steps to the exact path counts
  // as a failure (the fused contract must cover these shapes)
  const bool groups = fl.count("--profile") && fl["--profile"] == "groups";
  const bool require_fused = fl.count("--require-fused") && fl["--require-fused"] != "0";
  long long fallbacks = 0;
  Rng r(seed);
  int failures = 0, compared = 0, invalid = 0, errors_matched = 0;
  std::map<std::string, int> shapes;
  const int64_t sizes[] = {0, 1, 7, 100, 1000, 5000, 40000};
  const int64_t dsizes[] = {0, 1, 5, 50, 500, 3000};
  int plans_per_table = 10;
  for (int done = 0; done < nplans;) {
    Shape sh{sizes[pick(r, 7)], dsizes[pick(r, 6)], chance(r, 0.3), chance(r, 0.2), chance(r, 0.2)};
    if (groups) {
      // 1 k .. 10 M distinct k values over up to 1 M fact rows; dim keys
      // dense, spread (non-dense) or duplicated
      static const int64_t gsizes[] = {0, 1, 1000, 20000, 200000, 1000000};
      static const int64_t granges[] = {7, 1000, 50000, 1000000, 10000000};
      static const int64_t gdims[] = {0, 5, 500, 20000, 200000};
      sh = Shape{gsizes[pick(r, 6)], gdims[pick(r, 5)], chance(r, 0.2), false, chance(r, 0.1)};
      sh.groups = true;
      sh.k_range = granges[pick(r, 5)];
      sh.k_sparse = chance(r, 0.3);
      if (sh.k_sparse) sh.k_range = std::min<int64_t>(sh.k_range, 200000);
      static const int64_t spreads[] = {1, 1, 3, 1000, 1000000};
      sh.dim_spread = spreads[pick(r, 5)];
    }
    Catalog cat;
    TableSet tables;
    make_tables(r, sh, cat, tables);
    for (int q = 0; q < plans_per_table && done < nplans; ++q, ++done) {
      Built b;
      OperatorPlan op;
      try {
        b = groups ? random_group_plan(r, cat) : random_plan(r, cat);
        op = plan_operators(optimize(b.plan, cat), cat);
      } catch (const std::exception& e) {
        ++invalid;  // rejected by the reference's own planner: nothing to compare
        if (verbose) std::printf("SKIP %s: %s\n", b.text.c_str(), e.what());
        continue;
      }
      if (only >= 0 && done != only) continue;
      if (only >= 0) {
        std::printf("plan %d: %s\n%s\n", done, b.text.c_str(), plan_to_json(b.plan).c_str());
        for (const auto& [tn, tt] : tables) {
          std::printf("table %s (%lld rows):\n", tn.c_str(), static_cast<long long>(tt.row_count()));
          auto rows = decode_table(tt);
          for (size_t i = 0; i < rows.size() && i < 40; ++i) {
            std::string line;
            for (size_t c = 0; c < rows[i].size(); ++c)
              line += (c ? " | " : "  ") + cell_to_text(rows[i][c], tt.columns()[c].logical);
            std::printf("%s\n", line.c_str());
          }
        }
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
        long long fb = 0;
        try {
          tqp_integration::B200Executor ex(op, fuse);
          try {
            got = ex.execute(tables);
          } catch (...) {
            fb = ex.fallbacks();
            throw;
          }
          fb = ex.fallbacks();
        } catch (const std::exception& e) {
          got_err = e.what();
        }
        fallbacks += fb;
        if (fb && (verbose || require_fused))
          std::printf("FALLBACK plan %d (%lld fused unit(s) to the exact path) [%s] %s\n", done, fb,
                      fuse ? "fused" : "per-instruction", b.text.c_str());
        std::string d = !want_err.empty() || !got_err.empty()
                            ? (want_err == got_err ? "" : "error '" + got_err + "' vs '" + want_err + "'")
                            : diff(got, want);
        ++compared;
        if (!want_err.empty() && d.empty()) ++errors_matched;
        shapes[b.text]++;
        if (only >= 0 && d.empty() && want_err.empty()) {
          auto rows = decode_table(want);
          std::printf("result (%zu rows):\n", rows.size());
          for (size_t i = 0; i < rows.size() && i < 20; ++i) {
            std::string line;
            for (size_t c = 0; c < rows[i].size(); ++c) line += (c ? " | " : "  ") + cell_to_text(rows[i][c], want.columns()[c].logical);
            std::printf("%s\n", line.c_str());
          }
        }
        if (only >= 0 && !d.empty() && got_err.empty() && want_err.empty()) {
          for (const EncodedTable* t : {&want, &got}) {
            auto rows = decode_table(*t);
            std::printf("%s (%zu rows):\n", t == &want ? "reference" : "b200", rows.size());
            for (size_t i = 0; i < rows.size() && i < 20; ++i) {
              std::string line;
              for (size_t c = 0; c < rows[i].size(); ++c) line += (c ? " | " : "  ") + cell_to_text(rows[i][c], t->columns()[c].logical);
              std::printf("%s\n", line.c_str());
            }
          }
        }
        if (!d.empty() || verbose || only >= 0) {
          std::printf("%s plan %d (fact %lld rows, dim %lld%s%s%s) [%s] %s%s%s\n", d.empty() ? "PASS" : "FAIL", done,
                      static_cast<long long>(sh.n_fact), static_cast<long long>(sh.n_dim), sh.dim_dups ? ", dup keys" : "",
                      sh.huge_ints ? ", huge ints" : "", sh.nans ? ", NaN" : "", fuse ? "fused" : "per-instruction",
                      b.text.c_str(), d.empty() ? "" : ": ", d.c_str());
        }
        if (!d.empty()) ++failures;
        if (require_fused && fb && want_err.empty()) ++failures;
      }
    }
  }
  std::printf("random plans: seed %llu, %d plans, %d comparisons (%d matched errors), %d rejected by the planner, "
              "%zu distinct shapes, %lld fused fallback(s), %d failure(s)\n",
              static_cast<unsigned long long>(seed), nplans, compared, errors_matched, invalid, shapes.size(), fallbacks,
              failures);
  return failures ? 1 : 0;
}
