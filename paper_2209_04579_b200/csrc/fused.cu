// Fusion planner: recognises the reference's lowering recipes
// (operator_plan.cpp: lower_filter :227-237, lower_join :249-294,
// lower_aggregate :309-388, lower_sort :390-404, lower_limit :406-414) in a
// lowered OperatorPlan, rebuilds the relational pipeline they came from, and
// replaces [scan -> filter -> join(unique build) -> aggregate -> sort/limit]
// runs of steps with fused device pipelines (fused_kernels.cuh). Anything
// outside that contract stays on the per-instruction device path, and a
// fused unit whose data preconditions fail at run time (duplicate build keys,
// > 64 groups, fixed-point range, int64 near overflow) hands its steps back
// to the per-instruction path, which reproduces the reference exactly.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <limits>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <new>
#include <type_traits>
#include <mutex>
#include <set>
#include <sstream>

#include "comm.hpp"
#include "executor.hpp"
#include "fused_kernels.cuh"
#include "jit.hpp"
#include "scan.cuh"

namespace tqp {
namespace {

using namespace fz;

// ---- symbolic expressions ----------------------------------------------------
struct SExpr {
  enum K { COL, CONST, CMP, ARITH, LOGIC, NOT, LIKE, STRCMP, SELECT, CAST, BAD } k = BAD;
  int slot = -1;       // COL
  int op = 0;          // CMP/ARITH/LOGIC op, LIKE anchor, CAST target
  std::string pattern; // LIKE
  int a = -1, b = -1, c = -1;
  const Instr* cinstr = nullptr;  // CONST
};

struct AggOut {
  int fn;  // 0 sum 1 count 2 avg 3 min 4 max
  int expr = -1;
  int slot = -1;
};

struct Rel {
  enum Kind { SCAN, FILTER, JOIN, AGG, PROJECT, SORT, LIMIT, OTHER } kind = OTHER;
  int step = -1;
  std::vector<int> cols;
  int input = -1;  // rel (step index)
  int left = -1, right = -1, lk = -1, rk = -1;
  int pred = -1;
  std::vector<int> keys;  // AGG: input-relation slots
  std::vector<AggOut> aggs;
  std::vector<std::pair<int, bool>> sort_keys;  // SORT: input slots, priority order
  int64_t limit = -1;
  std::map<int, int> out_of_in;  // FILTER/SORT/LIMIT/JOIN: output slot -> input slot
};

struct ColSrc {
  int scan = -1;  // step index of the SCAN
  std::string table, column;
};

struct Analysis {
  const Plan& plan;
  std::vector<SExpr> ex;
  std::vector<Rel> rels;
  std::map<int, int> def_step;          // slot -> producing step
  std::map<int, const Instr*> def;      // slot -> producing instr
  std::map<int, int> rel_of;            // relation column slot -> step
  std::map<int, ColSrc> src;            // relation column slot -> base column

  explicit Analysis(const Plan& p) : plan(p) {}

  int add(SExpr e) {
    ex.push_back(std::move(e));
    return static_cast<int>(ex.size()) - 1;
  }

  // expression for `slot` inside step s; leaves resolve through `leaf`
  int build(int slot, int s, const std::function<int(int)>& leaf) {
    auto it = def.find(slot);
    if (it == def.end() || def_step[slot] != s) return leaf(slot);
    const Instr& in = *it->second;
    SExpr e;
    switch (in.op) {
      case Op::ConstTensor: e.k = SExpr::CONST; e.cinstr = &in; return add(e);
      case Op::Compare: e.k = SExpr::CMP; e.op = in.cmp; break;
      case Op::StringCompare: e.k = SExpr::STRCMP; e.op = in.cmp; break;
      case Op::Arith: e.k = SExpr::ARITH; e.op = in.arith; break;
      case Op::Logical: e.k = SExpr::LOGIC; e.op = in.logic; break;
      case Op::Not: e.k = SExpr::NOT; break;
      case Op::SubstringMatch: e.k = SExpr::LIKE; e.op = in.anchor; e.pattern = in.pattern; break;
      case Op::SelectWhere: e.k = SExpr::SELECT; break;
      case Op::Cast: e.k = SExpr::CAST; e.op = in.cast_to; break;
      case Op::BroadcastScalar: return build(in.inputs[0], s, leaf);
      case Op::Gather: return leaf(slot);  // sorted/filtered view of an input column
      default: return -1;
    }
    int kids[3] = {-1, -1, -1};
    for (size_t i = 0; i < in.inputs.size() && i < 3; ++i) {
      kids[i] = build(in.inputs[i], s, leaf);
      if (kids[i] < 0) return -1;
    }
    e.a = kids[0];
    e.b = kids[1];
    e.c = kids[2];
    return add(e);
  }

  int col_leaf(int slot) {
    SExpr e;
    e.k = SExpr::COL;
    e.slot = slot;
    return add(e);
  }

  bool analyse() {
    for (size_t s = 0; s < plan.steps.size(); ++s)
      for (const auto& in : plan.steps[s].instrs) {
        def[in.output] = &in;
        def_step[in.output] = static_cast<int>(s);
      }
    rels.resize(plan.steps.size());
    for (size_t s = 0; s < plan.steps.size(); ++s) {
      Rel& r = rels[s];
      r.step = static_cast<int>(s);
      r.cols = plan.steps[s].output_slots;
      const std::string& kind = plan.steps[s].kind;
      bool ok = false;
      if (kind == "scan") ok = an_scan(r);
      else if (kind == "filter") ok = an_filter(r);
      else if (kind == "join") ok = an_join(r);
      else if (kind == "aggregate") ok = an_agg(r);
      else if (kind == "project") ok = an_project(r);
      else if (kind == "sort") ok = an_sort(r);
      else if (kind == "limit") ok = an_limit(r);
      if (!ok) {
        r.kind = Rel::OTHER;
        if (std::getenv("TQP_FUSION_DEBUG")) std::fprintf(stderr, "[tqp] step %s not recognised\n", plan.steps[s].id.c_str());
      }
      for (int c : r.cols) rel_of[c] = static_cast<int>(s);
    }
    return true;
  }

  const std::vector<Instr>& ins(const Rel& r) { return plan.steps[r.step].instrs; }

  bool an_scan(Rel& r) {
    for (const auto& in : ins(r)) {
      if (in.op != Op::LoadColumn) return false;
      src[in.output] = {r.step, in.table, in.column};
    }
    r.kind = Rel::SCAN;
    return true;
  }

  // input relation that owns every slot in `slots` (same step), or -1
  int owner(const std::vector<int>& slots) {
    int o = -1;
    for (int x : slots) {
      auto it = rel_of.find(x);
      if (it == rel_of.end()) return -1;
      if (o >= 0 && it->second != o) return -1;
      o = it->second;
    }
    return o;
  }

  bool an_filter(Rel& r) {
    const auto& v = ins(r);
    const Instr* compact = nullptr;
    for (const auto& in : v)
      if (in.op == Op::Compact) compact = &in;
    if (!compact) return false;
    const Instr* io = def.count(compact->inputs[0]) ? def[compact->inputs[0]] : nullptr;
    if (!io || io->op != Op::IotaRows || io->param >= 0) return false;
    std::vector<int> in_cols;
    for (const auto& in : v) {
      if (in.op == Op::Gather && in.inputs[1] == compact->output) {
        in_cols.push_back(in.inputs[0]);
        r.out_of_in[in.output] = in.inputs[0];
      }
    }
    r.input = owner(in_cols);
    if (r.input < 0 || rels[r.input].cols != in_cols) return false;
    if (r.cols.size() != in_cols.size()) return false;
    for (size_t i = 0; i < r.cols.size(); ++i) {
      if (r.out_of_in[r.cols[i]] != in_cols[i]) return false;
      if (src.count(in_cols[i])) src[r.cols[i]] = src[in_cols[i]];
    }
    r.pred = build(compact->inputs[1], r.step, [&](int x) { return col_leaf(x); });
    if (r.pred < 0) return false;
    r.kind = Rel::FILTER;
    return true;
  }

  bool an_join(Rel& r) {
    const auto& v = ins(r);
    static const Op recipe[] = {Op::ArgsortStable, Op::Gather, Op::SearchSorted, Op::SearchSorted, Op::Arith,
                                Op::PrefixSum, Op::ConstTensor, Op::Arith, Op::SegmentedReduce, Op::IotaLen,
                                Op::ConstTensor, Op::SearchSorted, Op::Arith, Op::ExpandSegments, Op::Gather};
    const size_t nr = sizeof(recipe) / sizeof(recipe[0]);
    if (v.size() < nr) return false;
    for (size_t i = 0; i < nr; ++i)
      if (v[i].op != recipe[i]) return false;
    r.rk = v[0].inputs[0];
    r.lk = v[2].inputs[1];
    int left_ids = v[12].output, right_ids = v[14].output;
    std::vector<int> lc, rc;
    for (size_t i = nr; i < v.size(); ++i) {
      if (v[i].op != Op::Gather) return false;
      if (v[i].inputs[1] == left_ids) lc.push_back(v[i].inputs[0]);
      else if (v[i].inputs[1] == right_ids) rc.push_back(v[i].inputs[0]);
      else return false;
      r.out_of_in[v[i].output] = v[i].inputs[0];
      if (src.count(v[i].inputs[0])) src[v[i].output] = src[v[i].inputs[0]];
    }
    r.left = owner(lc);
    r.right = owner(rc);
    if (r.left < 0 || r.right < 0 || rels[r.left].cols != lc || rels[r.right].cols != rc) return false;
    if (rel_of[r.lk] != r.left || rel_of[r.rk] != r.right) return false;
    r.kind = Rel::JOIN;
    return true;
  }

  bool an_agg(Rel& r) {
    const auto& v = ins(r);
    bool keyed = false;
    for (const auto& in : v) keyed |= in.op == Op::SortPermRows;
    std::map<int, int> sorted_to_in;  // keyed: sorted slot -> input slot
    int perm = -1;
    if (keyed) {
      // iota, sort_perm_rows (keys last->first), gathers by perm
      size_t i = 0;
      if (v.empty() || v[0].op != Op::IotaRows) return false;
      ++i;
      std::vector<int> rev_keys;
      while (i < v.size() && v[i].op == Op::SortPermRows) {
        if (v[i].param != 1) return false;
        rev_keys.push_back(v[i].inputs[0]);
        perm = v[i].output;
        ++i;
      }
      r.keys.assign(rev_keys.rbegin(), rev_keys.rend());
      std::vector<int> in_cols;
      for (; i < v.size() && v[i].op == Op::Gather && v[i].inputs[1] == perm; ++i) {
        sorted_to_in[v[i].output] = v[i].inputs[0];
        in_cols.push_back(v[i].inputs[0]);
      }
      r.input = owner(in_cols);
      if (r.input < 0 || rels[r.input].cols != in_cols) return false;
    } else {
      if (v.size() < 3 || v[0].op != Op::ConstTensor || v[1].op != Op::IotaRows || v[2].op != Op::Arith) return false;
      r.input = rel_of.count(v[1].inputs[0]) ? rel_of[v[1].inputs[0]] : -1;
      if (r.input < 0) return false;
    }
    auto leaf = [&](int x) {
      if (keyed) {
        auto it = sorted_to_in.find(x);
        if (it == sorted_to_in.end()) return -1;
        x = it->second;
      }
      if (!rel_of.count(x) || rel_of[x] != r.input) return -1;
      return col_leaf(x);
    };
    const size_t nk = r.keys.size();
    if (r.cols.size() < nk) return false;
    for (size_t k = 0; k < nk; ++k) {
      // key output k = gather(sorted key col, first_idx)
      const Instr* g = def.count(r.cols[k]) ? def[r.cols[k]] : nullptr;
      if (!g || g->op != Op::Gather || sorted_to_in[g->inputs[0]] != r.keys[k]) return false;
    }
    for (size_t j = nk; j < r.cols.size(); ++j) {
      int out = r.cols[j];
      const Instr* d = def.count(out) ? def[out] : nullptr;
      if (!d) return false;
      AggOut a;
      a.slot = out;
      auto segred_sum_expr = [&](const Instr* sr) -> int {
        if (!sr || sr->op != Op::SegmentedReduce || sr->reduce != TQP_SUM) return -1;
        return build(sr->inputs[0], r.step, leaf);
      };
      if (d->op == Op::SegmentedReduce) {
        if (d->reduce == TQP_COUNT) {
          a.fn = 1;
        } else {
          a.fn = d->reduce == TQP_SUM ? 0 : d->reduce == TQP_MIN ? 3 : 4;
          a.expr = build(d->inputs[0], r.step, leaf);
          if (a.expr < 0) return false;
        }
      } else if (d->op == Op::Arith && d->arith == TQP_DIV) {
        const Instr* x = def.count(d->inputs[0]) ? def[d->inputs[0]] : nullptr;
        if (x && x->op == Op::Cast) x = def.count(x->inputs[0]) ? def[x->inputs[0]] : nullptr;
        a.fn = 2;
        a.expr = segred_sum_expr(x);
        if (a.expr < 0) return false;
      } else {
        return false;
      }
      r.aggs.push_back(a);
    }
    r.kind = Rel::AGG;
    return true;
  }

  bool an_project(Rel& r) {
    if (!ins(r).empty()) return false;
    int o = -1;
    for (int c : r.cols) {
      if (!rel_of.count(c)) return false;
      if (o >= 0 && rel_of[c] != o) return false;
      o = rel_of[c];
    }
    r.input = o;
    r.kind = Rel::PROJECT;
    return o >= 0;
  }

  bool an_sort(Rel& r) {
    const auto& v = ins(r);
    if (v.empty() || v[0].op != Op::IotaRows || v[0].param >= 0) return false;
    size_t i = 1;
    int perm = v[0].output;
    std::vector<std::pair<int, bool>> rev;
    for (; i < v.size() && v[i].op == Op::SortPermRows; ++i) {
      if (v[i].inputs[1] != perm) return false;
      rev.push_back({v[i].inputs[0], v[i].param == 1});
      perm = v[i].output;
    }
    r.sort_keys.assign(rev.rbegin(), rev.rend());
    std::vector<int> in_cols;
    for (; i < v.size(); ++i) {
      if (v[i].op != Op::Gather || v[i].inputs[1] != perm) return false;
      in_cols.push_back(v[i].inputs[0]);
      r.out_of_in[v[i].output] = v[i].inputs[0];
    }
    r.input = step_of_cols(in_cols);
    if (r.input < 0) return false;
    r.kind = Rel::SORT;
    return true;
  }

  bool an_limit(Rel& r) {
    const auto& v = ins(r);
    if (v.empty() || v[0].op != Op::IotaRows) return false;
    r.limit = v[0].param;
    std::vector<int> in_cols;
    for (size_t i = 1; i < v.size(); ++i) {
      if (v[i].op != Op::Gather || v[i].inputs[1] != v[0].output) return false;
      in_cols.push_back(v[i].inputs[0]);
      r.out_of_in[v[i].output] = v[i].inputs[0];
    }
    r.input = step_of_cols(in_cols);
    if (r.input < 0) return false;
    r.kind = Rel::LIMIT;
    return true;
  }

  // relation (step) whose output columns are exactly `cols`
  int step_of_cols(const std::vector<int>& cols) {
    for (int s = static_cast<int>(rels.size()) - 1; s >= 0; --s)
      if (rels[s].cols == cols && rels[s].step >= 0) return s;
    return -1;
  }
};

// ---- pipeline description -----------------------------------------------------
struct TermDesc {  // conjunct over a base table column
  std::string column;
  int kind;        // 0 numeric compare, 1 string compare, 2 like, 3 const true, 4 const false
  int op = 0;
  bool f64 = false;
  long long ik = 0;
  double fk = 0.0;
  std::string lit;  // string compare / like pattern
  int anchor = 0;
};

struct BuildDesc {
  int scan = -1;  // root scan step
  std::string table, key_column;
  std::vector<TermDesc> terms;
  struct Child {
    std::string fact_column;  // column of this root
    int build = -1;           // index into builds
  };
  std::vector<Child> children;
  std::vector<TermDesc> flags;  // string predicates evaluated per root row
  bool assign_groups = false;
};

struct OperandDesc {
  int probe = -1;  // -1 fact
  std::string column;
};

struct FactorDesc {
  OperandDesc x;
  int kind = FK_X;
  double k = 0.0;
};

struct AccDesc {
  bool is_int = false;
  std::vector<FactorDesc> f;
  int gate_probe = -1, gate_bit = 0;
  double gate_else = 0.0;
  std::string sig() const {
    std::ostringstream os;
    os << is_int << "|" << gate_probe << "," << gate_bit << "," << gate_else << "|";
    for (auto& x : f) os << x.x.probe << ":" << x.x.column << ":" << x.kind << ":" << x.k << ";";
    return os.str();
  }
};

constexpr int kMaxEpiConst = 8;  // constants of a scalar epilogue
// err[3] reason codes of a scalar epilogue (the exact path reports these
// errors with the reference's text)
constexpr long long kReasonEpiDivZero = 20;
constexpr long long kReasonEpiOverflow = 21;

struct OutDesc {  // aggregate outputs, in the AGG step's output order
  int fn;         // 0 sum 1 count 2 avg, 3 scalar epilogue arith, 10 + i: group key i
  int acc = -1;
  int slot = -1;
  bool is_int = false;
  int op = 0, a = 0, b = 0;  // fn 3 (OutKind)
};

struct PipeDesc {
  int first_step = 0, last_step = 0;
  int fact_scan = -1;
  std::string fact_table;
  std::vector<TermDesc> terms;
  struct ProbeD {
    std::string fact_column;
    int build = -1;
  };
  std::vector<ProbeD> probes;
  std::vector<BuildDesc> builds;
  std::vector<AccDesc> accs;
  std::vector<OutDesc> outs;  // AGG outputs
  int mode = MODE_SCALAR;
  std::vector<std::string> key_columns;     // MODE_SMALL fact key columns
  std::vector<int> key_width;               // 1-byte strings
  // MODE_BUILDGRP: keys resolved to root columns of probes[group_probe]
  int group_probe = -1;
  std::vector<std::string> group_key_root_columns;
  // MODE_HASH: group keys (fact or probe root columns) with their logical
  // types; a MODE_SMALL unit with hash_alt reruns as MODE_HASH when a CTA
  // meets more codes than its slots
  std::vector<OperandDesc> hkeys;
  std::vector<int> hkey_lt;
  bool hash_alt = false;
  // fused sort + limit (MODE_BUILDGRP)
  bool topk = false;
  int64_t k = 0;
  std::vector<std::pair<int, bool>> sort_outs;  // (index into outs, asc)
  std::vector<unsigned long long> konst;        // scalar epilogue constants (bits)
  std::string epi_step;                         // id of the absorbed epilogue step
  std::vector<int> final_cols;                  // unit output slots -> outs index
  std::vector<int> final_slots;
  std::string explain;
};

// flatten AND conjuncts
void conjuncts(Analysis& A, int e, std::vector<int>& out) {
  const SExpr& x = A.ex[e];
  if (x.k == SExpr::LOGIC && x.op == TQP_AND) {
    conjuncts(A, x.a, out);
    conjuncts(A, x.b, out);
  } else {
    out.push_back(e);
  }
}

const ColSrc* col_src(Analysis& A, int slot) {
  auto it = A.src.find(slot);
  return it == A.src.end() ? nullptr : &it->second;
}

std::string const_string(const Instr* c) {
  if (!c || c->const_dtype != TQP_I32 || c->const_rows != 1) return {};
  std::string s;
  const int32_t* d = reinterpret_cast<const int32_t*>(c->const_host.data());
  for (int64_t j = 0; j < c->const_cols && d[j] != 0; ++j) s.push_back(static_cast<char>(d[j]));
  return s;
}

bool const_scalar(const Instr* c, bool* is_f64, long long* ik, double* fk, bool* is_bool = nullptr) {
  if (!c || c->const_rows != 1 || c->const_cols != 1) return false;
  if (is_bool) *is_bool = c->const_dtype == TQP_BOOL;
  if (c->const_dtype == TQP_F64) {
    *is_f64 = true;
    std::memcpy(fk, c->const_host.data(), 8);
    return true;
  }
  if (c->const_dtype == TQP_I64) {
    *is_f64 = false;
    std::memcpy(ik, c->const_host.data(), 8);
    return true;
  }
  if (c->const_dtype == TQP_BOOL) {
    *is_f64 = false;
    *ik = c->const_host[0];
    return true;
  }
  return false;
}

int flip(int op) {
  switch (op) {
    case TQP_LT: return TQP_GT;
    case TQP_LE: return TQP_GE;
    case TQP_GT: return TQP_LT;
    case TQP_GE: return TQP_LE;
    default: return op;
  }
}

// conjunct over columns of scan `scan` -> TermDesc
bool term_of(Analysis& A, int e, int scan, const Plan& plan, TermDesc& t) {
  const SExpr& x = A.ex[e];
  auto col_of = [&](int ei, std::string& name) {
    const SExpr& c = A.ex[ei];
    if (c.k != SExpr::COL) return false;
    const ColSrc* s = col_src(A, c.slot);
    if (!s || s->scan != scan) return false;
    name = s->column;
    return true;
  };
  if (x.k == SExpr::CONST) {
    bool f, b;
    long long ik;
    double fk;
    if (!const_scalar(x.cinstr, &f, &ik, &fk, &b) || !b) return false;
    t.kind = ik ? 3 : 4;
    return true;
  }
  if (x.k == SExpr::CMP) {
    bool f;
    long long ik = 0;
    double fk = 0;
    if (col_of(x.a, t.column) && A.ex[x.b].k == SExpr::CONST && const_scalar(A.ex[x.b].cinstr, &f, &ik, &fk)) {
      t.op = x.op;
    } else if (col_of(x.b, t.column) && A.ex[x.a].k == SExpr::CONST && const_scalar(A.ex[x.a].cinstr, &f, &ik, &fk)) {
      t.op = flip(x.op);
    } else {
      return false;
    }
    // Bool-column compares are not fused terms (either operand order)
    if (A.ex[x.b].k == SExpr::CONST && A.ex[x.b].cinstr->const_dtype == TQP_BOOL) return false;
    if (A.ex[x.a].k == SExpr::CONST && A.ex[x.a].cinstr->const_dtype == TQP_BOOL) return false;
    t.kind = 0;
    t.f64 = f;
    t.ik = ik;
    t.fk = fk;
    return true;
  }
  if (x.k == SExpr::STRCMP) {
    if (!col_of(x.a, t.column) || A.ex[x.b].k != SExpr::CONST) return false;
    t.lit = const_string(A.ex[x.b].cinstr);
    if (t.lit.size() > 48) return false;
    t.kind = 1;
    t.op = x.op;
    return true;
  }
  if (x.k == SExpr::LIKE) {
    if (!col_of(x.a, t.column) || x.pattern.size() > 48) return false;
    t.kind = 2;
    t.lit = x.pattern;
    t.anchor = x.op;
    return true;
  }
  (void)plan;
  return false;
}

struct Planner {
  Analysis& A;
  const Plan& plan;
  PipeDesc P;
  std::string why;

  Planner(Analysis& a, const Plan& p) : A(a), plan(p) {}

  bool fail(const std::string& w) {
    why = w;
    return false;
  }

  // root scan of a build subtree; collects filters + nested joins
  bool parse_build(int rel, int key_slot, int& out_idx) {
    BuildDesc b;
    std::vector<int> chain;
    int r = rel;
    while (true) {
      const Rel& R = A.rels[r];
      if (R.kind == Rel::SCAN) break;
      if (R.kind == Rel::FILTER) {
        chain.push_back(r);
        r = R.input;
        continue;
      }
      if (R.kind == Rel::JOIN) {
        chain.push_back(r);
        r = R.left;
        continue;
      }
      return fail("build side is not scan/filter/join");
    }
    b.scan = r;
    b.table = A.plan.steps[r].instrs.empty() ? "" : A.plan.steps[r].instrs[0].table;
    const ColSrc* ks = col_src(A, key_slot);
    if (!ks || ks->scan != b.scan) return fail("build key not a root column");
    b.key_column = ks->column;
    for (int c : chain) {
      const Rel& R = A.rels[c];
      if (R.kind == Rel::FILTER) {
        std::vector<int> cs;
        conjuncts(A, R.pred, cs);
        for (int e : cs) {
          TermDesc t;
          if (!term_of(A, e, b.scan, plan, t)) return fail("build filter term unsupported");
          b.terms.push_back(t);
        }
      } else {
        const ColSrc* ls = col_src(A, R.lk);
        if (!ls || ls->scan != b.scan) return fail("nested join key not on build root");
        int child;
        if (!parse_build(R.right, R.rk, child)) return false;
        b.children.push_back({ls->column, child});
      }
    }
    P.builds.push_back(b);
    out_idx = static_cast<int>(P.builds.size()) - 1;
    return true;
  }

  // the steps (rels) a build subtree covers
  void build_steps(int rel, std::set<int>& s) {
    s.insert(rel);
    const Rel& R = A.rels[rel];
    if (R.kind == Rel::FILTER) build_steps(R.input, s);
    if (R.kind == Rel::JOIN) {
      build_steps(R.left, s);
      build_steps(R.right, s);
    }
  }

  // operand: column slot of the fact pipeline relation -> fact col or probe root col
  bool operand(int slot, OperandDesc& o, int* type) {
    const ColSrc* s = col_src(A, slot);
    if (!s) return false;
    int lt = -1;
    for (const auto& it : plan.input_tables)
      if (iequals(it.name, s->table))
        for (const auto& [c, t] : it.schema)
          if (iequals(c, s->column)) lt = t;
    if (type) *type = lt;
    o.column = s->column;
    if (s->scan == P.fact_scan) {
      o.probe = -1;
      return true;
    }
    for (size_t p = 0; p < P.probes.size(); ++p) {
      if (P.builds[P.probes[p].build].scan == s->scan) {
        o.probe = static_cast<int>(p);
        return true;
      }
    }
    return false;
  }

  bool factor_list(int e, std::vector<FactorDesc>& out) {
    const SExpr& x = A.ex[e];
    if (x.k == SExpr::ARITH && x.op == TQP_MUL) {
      // left-deep product: left is a product chain, right is one factor
      if (!factor_list(x.a, out)) return false;
      FactorDesc f;
      if (!one_factor(x.b, f)) return false;
      out.push_back(f);
      return true;
    }
    FactorDesc f;
    if (!one_factor(e, f)) return false;
    out.push_back(f);
    return true;
  }

  bool f64_col(int e, OperandDesc& o) {
    const SExpr& x = A.ex[e];
    int lt;
    return x.k == SExpr::COL && operand(x.slot, o, &lt) && lt == TQP_LT_FLOAT64;
  }

  bool one_factor(int e, FactorDesc& f) {
    const SExpr& x = A.ex[e];
    if (f64_col(e, f.x)) {
      f.kind = FK_X;
      return true;
    }
    if (x.k == SExpr::CONST) {
      bool isf;
      long long ik;
      double fk;
      if (!const_scalar(x.cinstr, &isf, &ik, &fk) || !isf) return false;
      f.kind = FK_CONST;
      f.k = fk;
      return true;
    }
    if (x.k != SExpr::ARITH) return false;
    bool isf;
    long long ik;
    double fk;
    const SExpr& a = A.ex[x.a];
    const SExpr& b = A.ex[x.b];
    if (a.k == SExpr::CONST && f64_col(x.b, f.x) && const_scalar(a.cinstr, &isf, &ik, &fk) && isf) {
      f.k = fk;
      switch (x.op) {
        case TQP_SUB: f.kind = FK_K_MINUS_X; return true;
        case TQP_ADD: f.kind = FK_K_PLUS_X; return true;
        case TQP_MUL: f.kind = FK_X_TIMES_K; return true;  // k*x == x*k exactly
        default: return false;
      }
    }
    if (b.k == SExpr::CONST && f64_col(x.a, f.x) && const_scalar(b.cinstr, &isf, &ik, &fk) && isf) {
      f.k = fk;
      switch (x.op) {
        case TQP_SUB: f.kind = FK_X_MINUS_K; return true;
        case TQP_ADD: f.kind = FK_X_PLUS_K; return true;
        case TQP_MUL: f.kind = FK_X_TIMES_K; return true;
        default: return false;
      }
    }
    return false;
  }

  // gate: a flag predicate over a probe's root string column
  bool gate_of(int e, int& probe, int& bit) {
    const SExpr& x = A.ex[e];
    if (x.k != SExpr::LIKE && x.k != SExpr::STRCMP) return false;
    const SExpr& c = A.ex[x.a];
    if (c.k != SExpr::COL) return false;
    OperandDesc o;
    int lt;
    if (!operand(c.slot, o, &lt) || o.probe < 0 || lt != TQP_LT_UTF8) return false;
    BuildDesc& b = P.builds[P.probes[o.probe].build];
    TermDesc t;
    if (!term_of(A, e, b.scan, plan, t)) return false;
    if (b.flags.size() >= static_cast<size_t>(kMaxFlags)) return false;
    probe = o.probe;
    bit = static_cast<int>(b.flags.size());
    b.flags.push_back(t);
    return true;
  }

  bool acc_of(int e, AccDesc& a) {
    const SExpr& x = A.ex[e];
    if (x.k == SExpr::COL) {
      OperandDesc o;
      int lt;
      if (!operand(x.slot, o, &lt)) return false;
      if (lt == TQP_LT_INT64) {
        a.is_int = true;
        a.f.push_back({o, FK_X, 0.0});
        return true;
      }
    }
    if (x.k == SExpr::SELECT) {
      const SExpr& el = A.ex[x.c];
      bool isf;
      long long ik;
      double fk;
      if (el.k != SExpr::CONST || !const_scalar(el.cinstr, &isf, &ik, &fk) || !isf) return false;
      if (!gate_of(x.a, a.gate_probe, a.gate_bit)) return false;
      a.gate_else = fk;
      return factor_list(x.b, a.f) && a.f.size() <= static_cast<size_t>(kMaxFactors);
    }
    return factor_list(e, a.f) && a.f.size() <= static_cast<size_t>(kMaxFactors);
  }

  int acc_index(const AccDesc& a) {
    for (size_t i = 0; i < P.accs.size(); ++i)
      if (P.accs[i].sig() == a.sig()) return static_cast<int>(i);
    P.accs.push_back(a);
    return static_cast<int>(P.accs.size()) - 1;
  }

  bool plan_agg(int agg_step) {
    const Rel& G = A.rels[agg_step];
    // fact pipeline below the aggregate
    std::vector<int> chain;
    int r = G.input;
    while (true) {
      const Rel& R = A.rels[r];
      if (R.kind == Rel::SCAN) break;
      if (R.kind == Rel::FILTER || R.kind == Rel::JOIN) {
        chain.push_back(r);
        r = R.kind == Rel::FILTER ? R.input : R.left;
        continue;
      }
      return fail("aggregate input is not a scan/filter/join pipeline");
    }
    P.fact_scan = r;
    P.fact_table = plan.steps[r].instrs.empty() ? "" : plan.steps[r].instrs[0].table;
    std::set<int> covered = {r, agg_step};
    std::reverse(chain.begin(), chain.end());  // bottom-up
    for (int c : chain) {
      const Rel& R = A.rels[c];
      covered.insert(c);
      if (R.kind == Rel::FILTER) {
        std::vector<int> cs;
        conjuncts(A, R.pred, cs);
        for (int e : cs) {
          TermDesc t;
          if (!term_of(A, e, P.fact_scan, plan, t)) return fail("fact filter term unsupported");
          if (t.kind == 1 || t.kind == 2) return fail("string predicate on fact table");
          P.terms.push_back(t);
        }
      } else {
        const ColSrc* ls = col_src(A, R.lk);
        if (!ls || ls->scan != P.fact_scan) return fail("join probe key not on fact table");
        int b;
        if (!parse_build(R.right, R.rk, b)) return false;
        build_steps(R.right, covered);
        P.probes.push_back({ls->column, b});
      }
    }
    if (static_cast<int>(P.probes.size()) > kMaxProbes || static_cast<int>(P.terms.size()) > kMaxTerms)
      return fail("too many probes/terms");
    // group keys
    if (G.keys.empty()) {
      P.mode = MODE_SCALAR;
    } else {
      bool small = G.keys.size() <= static_cast<size_t>(kMaxKeys);
      for (int k : G.keys) {
        OperandDesc o;
        int lt;
        if (!operand(k, o, &lt) || o.probe >= 0 || lt != TQP_LT_UTF8) small = false;
        else P.key_columns.push_back(o.column);
      }
      // hashable: <= kMaxKeys int64 / date / string keys, each a fact column
      // or a probe's root column
      bool hashable = G.keys.size() <= static_cast<size_t>(kMaxKeys);
      for (int k : G.keys) {
        OperandDesc o;
        int lt;
        if (!hashable) break;
        if (!operand(k, o, &lt) || (lt != TQP_LT_INT64 && lt != TQP_LT_DATE && lt != TQP_LT_UTF8)) {
          hashable = false;
          break;
        }
        // a key equal to a probe's build key is the fact probe column itself
        // (no read of the matched root row, so it survives repeated build keys)
        if (o.probe >= 0 && iequals(o.column, P.builds[P.probes[o.probe].build].key_column)) {
          o.column = P.probes[o.probe].fact_column;
          o.probe = -1;
        }
        P.hkeys.push_back(o);
        P.hkey_lt.push_back(lt);
      }
      if (!hashable) {
        P.hkeys.clear();
        P.hkey_lt.clear();
      }
      if (small) {
        P.mode = MODE_SMALL;
        P.hash_alt = hashable;
      } else {
        // group = matched build row of one probe
        P.key_columns.clear();
        int gp = -1;
        for (size_t p = 0; p < P.probes.size() && gp < 0; ++p) {
          bool ok = true, has_row_key = false;
          std::vector<std::string> cols;
          const std::string& bkey = P.builds[P.probes[p].build].key_column;
          for (int k : G.keys) {
            OperandDesc o;
            int lt;
            if (!operand(k, o, &lt) || (lt != TQP_LT_INT64 && lt != TQP_LT_DATE)) {
              ok = false;
              break;
            }
            if (o.probe == static_cast<int>(p)) {
              cols.push_back(o.column);
              has_row_key = has_row_key || iequals(o.column, bkey);
            } else if (o.probe < 0 && iequals(o.column, P.probes[p].fact_column)) {
              cols.push_back(bkey);  // l_orderkey == o_orderkey
              has_row_key = true;
            } else {
              ok = false;
              break;
            }
          }
          // a group is one build row only if the keys include the build's
          // (unique) key; other build columns may repeat across build rows
          if (ok && has_row_key) {
            gp = static_cast<int>(p);
            P.group_key_root_columns = cols;
          }
        }
        if (gp >= 0) {
          P.mode = MODE_BUILDGRP;
          P.group_probe = gp;
          P.builds[P.probes[gp].build].assign_groups = true;
        } else if (hashable) {
          P.mode = MODE_HASH;
          P.group_key_root_columns.clear();
        } else {
          return fail("group keys are neither small byte keys, a build row, nor hashable int/date/string columns");
        }
      }
    }
    // aggregates
    for (size_t i = 0; i < G.keys.size(); ++i) P.outs.push_back({10 + static_cast<int>(i), -1, G.cols[i], false});
    for (const auto& a : G.aggs) {
      OutDesc o;
      o.slot = a.slot;
      if (a.fn == 1) {
        o.fn = 1;
        o.is_int = true;
      } else if (a.fn == 0 || a.fn == 2) {
        AccDesc ad;
        if (!acc_of(a.expr, ad)) return fail("aggregate expression outside the fused family");
        o.fn = a.fn;
        o.acc = acc_index(ad);
        o.is_int = a.fn == 0 && ad.is_int;
      } else {
        return fail("MIN/MAX aggregate");
      }
      P.outs.push_back(o);
    }
    if (P.accs.size() > static_cast<size_t>(kMaxAcc)) return fail("too many accumulators");
    // accumulator operands on a probe's root row: only the hash-group kernel
    // reads them (at the matched row); other modes stage fact columns only
    bool probe_operand = false;
    for (const auto& a : P.accs)
      for (const auto& f : a.f) probe_operand = probe_operand || (f.kind != FK_CONST && f.x.probe >= 0);
    if (probe_operand && P.mode != MODE_HASH) {
      if (P.hkeys.empty()) return fail("aggregate operand on a build-side row outside a hash-group unit");
      if (P.mode == MODE_BUILDGRP) P.builds[P.probes[P.group_probe].build].assign_groups = false;
      P.mode = MODE_HASH;
      P.group_probe = -1;
      P.hash_alt = false;
      P.key_columns.clear();
      P.group_key_root_columns.clear();
    }
    // the unit must cover a contiguous step range
    P.first_step = *covered.begin();
    P.last_step = agg_step;
    for (int s = P.first_step; s <= P.last_step; ++s)
      if (!covered.count(s)) return fail("pipeline steps are not contiguous");
    for (int o : G.cols) P.final_slots.push_back(o);
    for (size_t i = 0; i < P.outs.size(); ++i) P.final_cols.push_back(static_cast<int>(i));
    // fused sort + limit after the aggregate (through an instruction-free project)
    int next = agg_step + 1;
    std::map<int, int> slot_to_out;
    for (size_t i = 0; i < P.outs.size(); ++i) slot_to_out[P.outs[i].slot] = static_cast<int>(i);
    if ((P.mode == MODE_BUILDGRP || P.mode == MODE_HASH) && next + 1 < static_cast<int>(A.rels.size())) {
      int s = next;
      std::vector<int> proj_cols = G.cols;
      if (A.rels[s].kind == Rel::PROJECT && A.rels[s].input == agg_step) {
        proj_cols = A.rels[s].cols;
        ++s;
      }
      if (s + 1 < static_cast<int>(A.rels.size()) && A.rels[s].kind == Rel::SORT && A.rels[s + 1].kind == Rel::LIMIT &&
          A.rels[s + 1].input == s && A.rels[s + 1].limit >= 0 && A.rels[s + 1].limit <= 32) {
        const Rel& S = A.rels[s];
        const Rel& L = A.rels[s + 1];
        bool ok = S.input >= 0;
        std::vector<std::pair<int, bool>> keys;
        for (auto [slot, asc] : S.sort_keys) {
          if (!slot_to_out.count(slot)) ok = false;
          else keys.push_back({slot_to_out[slot], asc});
        }
        std::vector<int> cols;
        for (int out : L.cols) {
          int in_sort = S.out_of_in.count(L.out_of_in.at(out)) ? S.out_of_in.at(L.out_of_in.at(out)) : -1;
          if (!slot_to_out.count(in_sort)) ok = false;
          else cols.push_back(slot_to_out[in_sort]);
        }
        if (ok && keys.size() <= 4) {
          P.topk = true;
          P.k = L.limit;
          P.sort_outs = keys;
          P.final_cols = cols;
          P.final_slots = L.cols;
          P.last_step = s + 1;
        }
      }
    }
    if (P.mode == MODE_SCALAR) absorb_scalar_epilogue(next);
    return true;
  }

  // A project step right after a scalar aggregate whose instructions are 1x1
  // constants and + - * / over the aggregate's outputs (Q14's 100.00 *
  // promo / total) is evaluated by k_final_scalar: no per-instruction step,
  // no second round trip. Anything else (other ops, int division, a bool
  // constant) leaves the step to the exact path.
  void absorb_scalar_epilogue(int next) {
    if (next >= static_cast<int>(plan.steps.size())) return;
    const Step& st = plan.steps[next];
    if (st.kind != "project" || st.instrs.empty()) return;
    std::map<int, int> out_of;  // slot -> outs index
    for (size_t i = 0; i < P.outs.size(); ++i) out_of[P.outs[i].slot] = static_cast<int>(i);
    std::map<int, std::pair<int, bool>> konst_of;  // slot -> (const index, is_int)
    std::vector<OutDesc> outs = P.outs;
    std::vector<unsigned long long> konst;
    auto is_int_out = [&](const OutDesc& o) { return o.fn == 1 || ((o.fn == 0 || o.fn == 3) && o.is_int); };
    for (const Instr& in : st.instrs) {
      if (in.op == Op::ConstTensor) {
        bool f = false, b = false;
        long long ik = 0;
        double fk = 0;
        if (!const_scalar(&in, &f, &ik, &fk, &b) || b || konst.size() >= static_cast<size_t>(kMaxEpiConst)) return;
        unsigned long long bits;
        if (f) std::memcpy(&bits, &fk, 8);
        else bits = static_cast<unsigned long long>(ik);
        konst_of[in.output] = {static_cast<int>(konst.size()), !f};
        konst.push_back(bits);
        continue;
      }
      if (in.op != Op::Arith || in.inputs.size() != 2 || in.arith < TQP_ADD || in.arith > TQP_DIV) return;
      int opnd[2];
      bool ints[2];
      for (int k = 0; k < 2; ++k) {
        const int x = in.inputs[k];
        auto o = out_of.find(x);
        auto q = konst_of.find(x);
        if (o != out_of.end()) {
          opnd[k] = o->second;
          ints[k] = is_int_out(outs[o->second]);
        } else if (q != konst_of.end()) {
          opnd[k] = -1 - q->second.first;
          ints[k] = q->second.second;
        } else {
          return;
        }
      }
      if (ints[0] != ints[1] || (ints[0] && in.arith == TQP_DIV) || outs.size() >= 16) return;
      OutDesc d;
      d.fn = 3;
      d.slot = in.output;
      d.is_int = ints[0];
      d.op = in.arith;
      d.a = opnd[0];
      d.b = opnd[1];
      out_of[in.output] = static_cast<int>(outs.size());
      outs.push_back(d);
    }
    // the step's outputs (and any slot passing through it) must come from the unit
    std::vector<int> slots = P.final_slots, cols = P.final_cols;
    for (int x : st.output_slots) {
      auto o = out_of.find(x);
      if (o == out_of.end()) return;
      if (std::find(slots.begin(), slots.end(), x) == slots.end()) {
        slots.push_back(x);
        cols.push_back(o->second);
      }
    }
    for (size_t i = P.outs.size(); i < outs.size(); ++i) {
      if (std::find(slots.begin(), slots.end(), outs[i].slot) == slots.end()) {
        slots.push_back(outs[i].slot);
        cols.push_back(static_cast<int>(i));
      }
    }
    P.outs = outs;
    P.konst = konst;
    P.final_slots = slots;
    P.final_cols = cols;
    P.epi_step = st.id;
    P.last_step = next;
  }
};

// ---- finalize kernels ------------------------------------------------------------
struct OutKind {
  int fn;  // 0 sum 1 count 2 avg, 3 scalar epilogue arith, 10+i key
  int acc;
  int is_int;
  // fn 3: op (TQP_ADD..TQP_DIV) over operands a, b: >= 0 an earlier output,
  // < 0 the constant konst[-1 - x]
  int op = 0, a = 0, b = 0;
};

struct FinalSpec {
  int nouts = 0;
  OutKind outs[16];
  void* out_ptr[16];
  int nacc = 0;
  int acc_is_int[kMaxAcc];
  unsigned long long konst[kMaxEpiConst];
};

constexpr int kMerged = 256;

// Deterministic warp sum of get(i), i < m: lane l adds i = l, l + 32, ... in
// order, then a fixed xor-shuffle tree; every lane returns the total. The
// association is fixed by m alone, so a merge is reproducible run to run
// (fp64 sums need not be sequential: SURVEY.md 8(a) a7 allows the
// reference's own 4096-chunk order, within the fp64 tolerance).
template <typename Get>
__device__ __forceinline__ unsigned long long warp_sum_fixed(bool is_int, int m, Get get) {
  const int lane = threadIdx.x & 31;
  unsigned long long t = 0;
#pragma unroll 4
  for (int i = lane; i < m; i += 32) t = add_acc(is_int, t, get(i));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t = add_acc(is_int, t, __shfl_xor_sync(0xffffffffu, t, o));
  return t;
}

__global__ void k_final_scalar(const unsigned long long* __restrict__ part, int nparts, FinalSpec f, long long* err) {
  // one warp per accumulator (and the count), warp_sum_fixed over the CTAs
  __shared__ unsigned long long s_tot[kMaxAcc + 1];
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int a = warp; a <= kMaxAcc; a += nwarps) {
    if (a != kMaxAcc && a >= f.nacc) continue;
    const bool is_int = a == kMaxAcc || f.acc_is_int[a];
    const unsigned long long t =
        warp_sum_fixed(is_int, nparts, [&](int i) { return part[static_cast<long long>(i) * (kMaxAcc + 1) + a]; });
    if ((threadIdx.x & 31) == 0) s_tot[a] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long cnt = static_cast<long long>(s_tot[kMaxAcc]);
    unsigned long long val[16];
    for (int j = 0; j < f.nouts; ++j) {
      const OutKind& o = f.outs[j];
      unsigned long long v = 0;
      if (o.fn == 1) {
        v = static_cast<unsigned long long>(cnt);
      } else if (o.fn == 0) {
        v = s_tot[o.acc];
      } else if (o.fn == 3) {
        // scalar epilogue, arith's semantics (kernels.cpp:211-283): fp64
        // with IEEE rounding, int64 checked; a division by zero or an
        // overflow hands the unit to the exact path, which raises it
        const unsigned long long x = o.a >= 0 ? val[o.a] : f.konst[-1 - o.a];
        const unsigned long long y = o.b >= 0 ? val[o.b] : f.konst[-1 - o.b];
        if (o.is_int) {
          int64_t r = 0;
          const int64_t xi = static_cast<int64_t>(x), yi = static_cast<int64_t>(y);
          const bool ovf = o.op == TQP_ADD ? add_ovf(xi, yi, &r) : o.op == TQP_SUB ? sub_ovf(xi, yi, &r) : mul_ovf(xi, yi, &r);
          if (ovf) {
            err[0] = 1;
            err[3] = kReasonEpiOverflow;
          }
          v = static_cast<unsigned long long>(r);
        } else {
          const double xd = __longlong_as_double(static_cast<long long>(x));
          const double yd = __longlong_as_double(static_cast<long long>(y));
          double r;
          switch (o.op) {
            case TQP_ADD: r = __dadd_rn(xd, yd); break;
            case TQP_SUB: r = __dsub_rn(xd, yd); break;
            case TQP_MUL: r = __dmul_rn(xd, yd); break;
            default:
              if (yd == 0.0) {
                err[0] = 1;
                err[3] = kReasonEpiDivZero;
                r = 0.0;
              } else {
                r = __ddiv_rn(xd, yd);
              }
          }
          v = static_cast<unsigned long long>(__double_as_longlong(r));
        }
      } else {
        if (cnt == 0) {
          err[0] = 1;  // AVG over zero rows: the reference raises division by zero
          val[j] = 0;
          continue;
        }
        double sum = f.acc_is_int[o.acc] ? static_cast<double>(static_cast<long long>(s_tot[o.acc]))
                                         : __longlong_as_double(static_cast<long long>(s_tot[o.acc]));
        v = static_cast<unsigned long long>(__double_as_longlong(__ddiv_rn(sum, static_cast<double>(cnt))));
      }
      val[j] = v;
      static_cast<unsigned long long*>(f.out_ptr[j])[0] = v;
    }
  }
}

// MODE_SMALL merge: distinct codes -> sorted -> per (group, acc) sums. One
// thread per CTA part inserts its codes and later records the group rank of
// each of its slots (rank[part][slot]); one warp per (group, accumulator |
// count) then sums the parts' values with warp_sum_fixed (absent slots
// contribute +0.0 / 0, which never changes a sum that starts at +0.0).
constexpr int kFinalSmallThreads = 1024;
constexpr size_t kFinalSmallStageMax = 180 * 1024;  // dynamic shared memory for staged parts
static_assert(kFinalSmallThreads >= kMerged, "one thread per merge slot when compacting the codes");
// kStaged: the parts (and the rank table) are first copied into dynamic
// shared memory with every load in flight at once, so the phases below make
// no further global round trips (Q1: 148 parts, 90 KB); otherwise (many
// shards' parts) they are read from global memory in place.
template <bool kStaged>
__global__ void __launch_bounds__(kFinalSmallThreads) k_final_small(const SmallPart* __restrict__ parts_g, int nparts,
                                                                    FinalSpec f, int nkeys, void* key_ptr0,
                                                                    void* key_ptr1, void* key_ptr2, void* key_ptr3,
                                                                    int* rank_g /*[nparts][kGroups]*/,
                                                                    long long* ngroups_out, long long* err) {
  extern __shared__ __align__(16) unsigned char s_parts_raw[];
  const SmallPart* parts = parts_g;
  int* rank = rank_g;
  if constexpr (kStaged) {
    const int n16 = static_cast<int>(nparts * sizeof(SmallPart) / 16);
    const uint4* src = reinterpret_cast<const uint4*>(parts_g);
    uint4* dst = reinterpret_cast<uint4*>(s_parts_raw);
    for (int i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = __ldg(src + i);
    parts = reinterpret_cast<const SmallPart*>(s_parts_raw);
    rank = reinterpret_cast<int*>(s_parts_raw + nparts * sizeof(SmallPart));
    __syncthreads();
  }
  __shared__ unsigned s_set[kMerged];
  __shared__ unsigned s_sorted[kMerged];
  __shared__ unsigned long long s_tot[kMerged][kMaxAcc + 1];
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int i = threadIdx.x; i < kMerged; i += blockDim.x) s_set[i] = 0xffffffffu;
  __syncthreads();
  for (int c = threadIdx.x; c < nparts; c += blockDim.x) {
    unsigned code[kGroups];
    unsigned long long cnt[kGroups];
#pragma unroll
    for (int sl = 0; sl < kGroups; ++sl) {
      code[sl] = parts[c].codes[sl];
      cnt[sl] = parts[c].cnt[sl];
    }
#pragma unroll
    for (int sl = 0; sl < kGroups; ++sl) {
      const unsigned cd = code[sl];
      if (cd == 0xffffffffu || cnt[sl] == 0) continue;
      unsigned h = (cd * 2654435761u) >> 24;
      bool placed = false;
      for (int p = 0; p < kMerged; ++p) {
        unsigned cur = s_set[h];
        if (cur == cd) { placed = true; break; }
        if (cur == 0xffffffffu) {
          unsigned prev = atomicCAS(&s_set[h], 0xffffffffu, cd);
          if (prev == 0xffffffffu || prev == cd) { placed = true; break; }
        }
        h = (h + 1) & (kMerged - 1);
      }
      if (!placed) err[0] = 1;
    }
  }
  __syncthreads();
  // rank sort of the distinct codes (codes are unique): the occupied slots
  // are compacted first, so each code is compared with the n codes only
  __shared__ unsigned s_list[kMerged];
  __shared__ int s_n;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  if (threadIdx.x < kMerged && s_set[threadIdx.x] != 0xffffffffu) s_list[atomicAdd(&s_n, 1)] = s_set[threadIdx.x];
  __syncthreads();
  const int n = s_n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned v = s_list[i];
    int r = 0;
    for (int j = 0; j < n; ++j) r += s_list[j] < v;
    s_sorted[r] = v;
  }
  if (threadIdx.x == 0) *ngroups_out = n;
  __syncthreads();
  for (int c = threadIdx.x; c < nparts; c += blockDim.x) {
#pragma unroll
    for (int sl = 0; sl < kGroups; ++sl) {
      const unsigned code = parts[c].codes[sl];
      int r = -1;
      if (code != 0xffffffffu && parts[c].cnt[sl] != 0) {
        int lo = 0, hi = n;
        while (lo < hi) {
          int m = (lo + hi) / 2;
          if (s_sorted[m] < code) lo = m + 1;
          else hi = m;
        }
        r = lo;
      }
      rank[static_cast<long long>(c) * kGroups + sl] = r;
    }
  }
  __syncthreads();
  const int per = f.nacc + 1;
  for (int p = warp; p < n * per; p += nwarps) {
    const int g = p / per, a = p % per;  // a == f.nacc: the row count
    const bool is_int = a == f.nacc || f.acc_is_int[a];
    const unsigned long long tot = warp_sum_fixed(is_int, nparts, [&](int c) {
      const int* rk = rank + static_cast<long long>(c) * kGroups;
      int sl = -1;
#pragma unroll
      for (int q = 0; q < kGroups; ++q) sl = rk[q] == g ? q : sl;
      return sl < 0 ? 0ULL : (a == f.nacc ? parts[c].cnt[sl] : parts[c].acc[sl][a]);
    });
    if ((threadIdx.x & 31) == 0) s_tot[g][a] = tot;
  }
  __syncthreads();
  void* kp[4] = {key_ptr0, key_ptr1, key_ptr2, key_ptr3};
  for (int g = threadIdx.x; g < n; g += blockDim.x) {
    unsigned code = s_sorted[g];
    for (int k = 0; k < nkeys; ++k) static_cast<uint8_t*>(kp[k])[g] = (code >> (8 * (nkeys - 1 - k))) & 0xff;
    const long long cnt = static_cast<long long>(s_tot[g][f.nacc]);
    for (int j = 0; j < f.nouts; ++j) {
      const OutKind& o = f.outs[j];
      if (o.fn >= 10) continue;
      if (o.fn == 1) static_cast<long long*>(f.out_ptr[j])[g] = cnt;
      else if (o.fn == 0) static_cast<unsigned long long*>(f.out_ptr[j])[g] = s_tot[g][o.acc];
      else {
        double sum = f.acc_is_int[o.acc] ? static_cast<double>(static_cast<long long>(s_tot[g][o.acc]))
                                         : __longlong_as_double(static_cast<long long>(s_tot[g][o.acc]));
        static_cast<double*>(f.out_ptr[j])[g] = __ddiv_rn(sum, static_cast<double>(cnt));
      }
    }
  }
}

// MODE_BUILDGRP outputs
struct GroupSpec {
  FinalSpec f;
  const unsigned long long* gacc;
  const unsigned long long* gcnt;
  // group -> build row through the build table entry (rowid + 1 in bits
  // 0-31); nullptr: merged groups (identity)
  const unsigned long long* group_table;
  long long cnt_stride = 1;  // words between groups' counts
  long long acc_stride = 0;  // words between groups' accumulator blocks
  int nkeyc;
  const long long* key_cols[kMaxKeys];  // root columns for the group keys
  int nsort;
  int sort_out[4];  // index into f.outs
  int sort_asc[4];
  const unsigned* present = nullptr;  // group g exists iff bit g is set (nullptr: every slot, zeroed)
  int acc_words = 2;                  // per accumulator: 2 = int128 (lo, hi), kLimbWords = limbs
  // MODE_HASH: group keys decoded from the group's code (tag - 1, ProbeSpec
  // GKey), counts packed as rows | adds << 40
  const unsigned long long* codes = nullptr;
  long long kmin[kMaxKeys] = {0, 0, 0, 0}, kstep[kMaxKeys] = {1, 1, 1, 1};
  unsigned long long krange[kMaxKeys] = {1, 1, 1, 1}, kstride[kMaxKeys] = {1, 1, 1, 1};
  int key_w[kMaxKeys] = {0, 0, 0, 0};  // output width of key i: 0 int64, else STR8 bytes
  int cnt_packed = 0;
  const long long* dvals[kMaxKeys] = {nullptr, nullptr, nullptr, nullptr};  // dictionary keys: value by rank
  const long long* absmax = nullptr;  // MODE_HASH: int sums exact iff absmax x rows < 2^63
  int flag_word = -1;                 // MODE_HASH special run: record word of the NaN/Inf bits
  int qfrac = 64;                     // fixed-point fraction bits of the sums
  int limb2 = 0;                      // MODE_HASH 2-limb sums (checked per group against fmax)
  int acc_off[kMaxAcc] = {};           // limb2: word of accumulator a (ProbeSpec::hoff)
  unsigned acc_int1 = 0;              // limb2: accumulator a is one int64 word (bit a)
  const long long* fmax = nullptr;    // max |fp64 value| (bits) of the scan
  int direct_codes = 0;               // MODE_HASH direct table: the group's code is its slot
  int row_in_cnt = 0;                 // BUILDGRP row_rec build: count word = (row + 1) << 32 | rows
};

__device__ __forceinline__ long long group_src_row(const GroupSpec& s, unsigned g);

// group key i of group g (STR8 keys: the row's bytes big-endian)
__device__ __forceinline__ long long group_key_value(const GroupSpec& s, int i, unsigned g) {
  if (s.codes || s.direct_codes) {
    const unsigned long long code = s.direct_codes ? static_cast<unsigned long long>(g) : s.codes[g] - 1ULL;
    // one key (stride 1, code < range): the digit is the code, no 64-bit divide
    const unsigned long long dg = (s.kstride[i] == 1 && code < s.krange[i]) ? code : (code / s.kstride[i]) % s.krange[i];
    if (s.dvals[i]) return s.dvals[i][dg];
    return s.key_w[i] ? static_cast<long long>(dg) : s.kmin[i] + static_cast<long long>(dg * static_cast<unsigned long long>(s.kstep[i]));
  }
  return s.key_cols[i][group_src_row(s, g)];
}
__device__ __forceinline__ long long group_count(const GroupSpec& s, unsigned g) {
  const unsigned long long w = s.gcnt[g * s.cnt_stride];
  return static_cast<long long>(s.cnt_packed ? (w & kCntMask) : s.row_in_cnt ? (w & 0xffffffffULL) : w);
}
// limb words exact: fewer than kLimbMaxRows adds reached them
__device__ __forceinline__ bool group_limbs_ok(const GroupSpec& s, unsigned g) {
  if (s.limb2) {
    const unsigned long long w = s.gcnt[g * s.cnt_stride];
    const double fm = s.fmax ? __longlong_as_double(*s.fmax) : 0.0;
    return (w >> 40) < (1ULL << 22) && fm * static_cast<double>(w & kCntMask) < 2.1990232555520000e12;  // 2^41
  }
  if (s.acc_words != kLimbWords) return true;
  const unsigned long long w = s.gcnt[g * s.cnt_stride];
  return (s.cnt_packed ? (w >> 40) : s.row_in_cnt ? (w & 0xffffffffULL) : w) < static_cast<unsigned long long>(kLimbMaxRows);
}

// accumulator a of group g as int128
__device__ __forceinline__ __int128 group_acc(const GroupSpec& s, unsigned g, int a) {
  if (s.limb2) {
    const unsigned long long* w = s.gacc + static_cast<long long>(g) * s.acc_stride + s.acc_off[a];
    if ((s.acc_int1 >> a) & 1u) return static_cast<__int128>(static_cast<long long>(w[0]));
    return limbs2_to_i128(w);
  }
  const unsigned long long* w = s.gacc + static_cast<long long>(g) * s.acc_stride + a * s.acc_words;
  if (s.acc_words == kLimbWords) return limbs_to_i128(w);
  return static_cast<__int128>((static_cast<unsigned __int128>(w[1]) << 64) | w[0]);
}

__device__ __forceinline__ long long group_src_row(const GroupSpec& s, unsigned g) {
  if (s.row_in_cnt) return static_cast<long long>(s.gcnt[g * s.cnt_stride] >> 32) - 1;
  return s.group_table ? static_cast<long long>(s.group_table[g] & 0xffffffffULL) - 1 : static_cast<long long>(g);
}

// not inlined: its int128 / limb / division cases are several thousand
// instructions, and the top-k kernel calls it from many sites - inlined
// copies made k_topk_groups ~26 k instructions and its walk instruction-fetch
// bound (kernels passing a GroupSpec take it as __grid_constant__, so a call
// does not copy the struct to local memory)
__device__ __noinline__ bool group_out_value(const GroupSpec& s, int j, unsigned g, unsigned long long& bits,
                                                bool& is_f64) {
  const OutKind& o = s.f.outs[j];
  long long cnt = group_count(s, g);
  if (o.fn >= 10) {
    bits = static_cast<unsigned long long>(group_key_value(s, o.fn - 10, g));
    is_f64 = false;
    return true;
  }
  if (o.fn == 1) {
    bits = static_cast<unsigned long long>(cnt);
    is_f64 = false;
    return true;
  }
  const __int128 v128 = group_acc(s, g, o.acc);
  const unsigned long long lo = static_cast<unsigned long long>(v128);
  const unsigned long long hi = static_cast<unsigned long long>(static_cast<unsigned __int128>(v128) >> 64);
  const bool limbs_ok = group_limbs_ok(s, g);
  if (s.f.acc_is_int[o.acc]) {
    long long v = static_cast<long long>(lo);
    bool fits = static_cast<long long>(hi) == (v >> 63);
    if (s.absmax && static_cast<double>(*s.absmax) * static_cast<double>(cnt) >= 9.0e18) fits = false;
    if (o.fn == 0) {
      bits = static_cast<unsigned long long>(v);
      is_f64 = false;
      return fits && limbs_ok;
    }
    bits = static_cast<unsigned long long>(__double_as_longlong(__ddiv_rn(static_cast<double>(v), static_cast<double>(cnt))));
    is_f64 = true;
    return fits && limbs_ok;
  }
  double sum = s.qfrac == 64 ? q64_to_f64(lo, hi)
                             : ldexp(i128_to_f64_rn(static_cast<__int128>((static_cast<unsigned __int128>(hi) << 64) | lo)), -s.qfrac);
  if (s.flag_word >= 0) {  // NaN / +Inf / -Inf among the group's values (IEEE sum)
    const unsigned f = static_cast<unsigned>(s.gcnt[g * s.cnt_stride + s.flag_word] >> (3 * o.acc)) & 7u;
    if ((f & 1u) || (f & 6u) == 6u) sum = __longlong_as_double(0x7ff8000000000000LL);
    else if (f & 2u) sum = __longlong_as_double(0x7ff0000000000000LL);
    else if (f & 4u) sum = __longlong_as_double(static_cast<long long>(0xfff0000000000000ULL));
  }
  is_f64 = true;
  bits = static_cast<unsigned long long>(__double_as_longlong(o.fn == 0 ? sum : __ddiv_rn(sum, static_cast<double>(cnt))));
  return limbs_ok;
}

// output row r of group output j (a hash unit's STR8 key: the big-endian
// bytes of its digit)
__device__ __forceinline__ void store_group_out(const GroupSpec& s, int j, long long r, unsigned long long bits) {
  const int w = s.f.outs[j].fn >= 10 ? s.key_w[s.f.outs[j].fn - 10] : 0;
  if (w) {
    uint8_t* o = static_cast<uint8_t*>(s.f.out_ptr[j]) + r * w;
    for (int b = 0; b < w; ++b) o[b] = static_cast<uint8_t>(bits >> (8 * (w - 1 - b)));
  } else {
    static_cast<unsigned long long*>(s.f.out_ptr[j])[r] = bits;
  }
}

// lexicographic candidate key: sort keys (with direction), then group keys asc
__device__ __forceinline__ unsigned long long sort_key_word(const GroupSpec& s, int i, unsigned g) {
  unsigned long long bits;
  bool f;
  group_out_value(s, s.sort_out[i], g, bits, f);
  unsigned long long u = f ? radix_key(__longlong_as_double(static_cast<long long>(bits)))
                           : radix_key(static_cast<int64_t>(bits));
  return s.sort_asc[i] ? u : ~u;
}

__device__ __forceinline__ int cand_keys(const GroupSpec& s, unsigned g, unsigned long long* k) {
  int n = 0;
  for (int i = 0; i < s.nsort; ++i) k[n++] = sort_key_word(s, i, g);
  for (int i = 0; i < s.nkeyc; ++i) k[n++] = radix_key(static_cast<int64_t>(group_key_value(s, i, g)));
  return n;
}

__device__ __forceinline__ bool key_less(const unsigned long long* a, const unsigned long long* b, int n) {
  for (int i = 0; i < n; ++i)
    if (a[i] != b[i]) return a[i] < b[i];
  return false;
}

// Top-k with the reference's tie order over the groups that have rows, in
// one launch. The candidate key (sort keys with direction, then the unique
// group keys ascending) totally orders the groups exactly as the reference's
// stable sort of the ascending group-by output does. NK (key words) is a
// template parameter so every key lives in registers.
//
// Each warp keeps a sorted list of its k (<= 32) best candidates in registers,
// one entry per lane. A group whose first key word already loses to the
// list's k-th key is dropped without computing the rest; a lane that beats it
// is inserted with one ballot (its position) and one shuffle-up per key word.
// The block's warp lists meet in warp 0 the same way, and the last block to
// finish folds every block list in and writes the output rows.
constexpr int kTopkMaxK = 32;
constexpr int kTopkUnroll = 4;
constexpr int kTopkThreads = 256;

template <int NK>
struct TopkList {
  unsigned long long e[NK];  // lane i: the i-th best key (i < cnt)
  unsigned gid = 0;
  int cnt = 0;
  unsigned long long thr[NK];  // k-th best key once cnt == k

  __device__ static bool less(const unsigned long long* a, const unsigned long long* b) {
    bool lt = false, eq = true;
#pragma unroll
    for (int q = 0; q < NK; ++q) {
      lt = lt || (eq && a[q] < b[q]);
      eq = eq && a[q] == b[q];
    }
    return lt;
  }
  __device__ bool beats(const unsigned long long* kk, int k) const { return cnt < k || less(kk, thr); }
  // warp-uniform: insert the key of lane `src` (kk, g valid in that lane)
  __device__ void insert_from(const unsigned long long* kk, unsigned g, int src, int k) {
    const int lane = threadIdx.x & 31;
    unsigned long long bk[NK];
#pragma unroll
    for (int q = 0; q < NK; ++q) bk[q] = __shfl_sync(0xffffffffu, kk[q], src);
    const unsigned bg = __shfl_sync(0xffffffffu, g, src);
    if (!beats(bk, k)) return;
    const int pos = __popc(__ballot_sync(0xffffffffu, lane < cnt && less(e, bk)));
#pragma unroll
    for (int q = 0; q < NK; ++q) {
      const unsigned long long up = __shfl_up_sync(0xffffffffu, e[q], 1);
      e[q] = lane > pos ? up : (lane == pos ? bk[q] : e[q]);
    }
    const unsigned upg = __shfl_up_sync(0xffffffffu, gid, 1);
    gid = lane > pos ? upg : (lane == pos ? bg : gid);
    if (cnt < k) ++cnt;
    if (cnt == k) {
#pragma unroll
      for (int q = 0; q < NK; ++q) thr[q] = __shfl_sync(0xffffffffu, e[q], k - 1);
    }
  }
  // offer one candidate per lane (valid where `cand`)
  __device__ void offer(bool cand, const unsigned long long* kk, unsigned g, int k) {
    unsigned mask = __ballot_sync(0xffffffffu, cand && beats(kk, k));
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      insert_from(kk, g, src, k);
      if (cnt == k) mask &= __ballot_sync(0xffffffffu, cand && less(kk, thr));
    }
  }
};

// key word q of group g's candidate key (not inlined: one copy for every
// call site of the top-k kernel)
__device__ __noinline__ unsigned long long cand_key_word(const GroupSpec& s, int q, unsigned g) {
  return q < s.nsort ? sort_key_word(s, q < 4 ? q : 3, g)
                     : radix_key(static_cast<int64_t>(group_key_value(s, q - s.nsort, g)));
}

template <int NK>
__device__ __forceinline__ void cand_keys_nk(const GroupSpec& s, unsigned g, unsigned long long* k) {
#pragma unroll
  for (int q = 0; q < NK; ++q) k[q] = cand_key_word(s, q, g);
}

// Exact top-k in one launch, without per-group full keys. The walk only
// forms each group's FIRST key word k0 (one accumulator read):
//   * every warp keeps the k smallest k0 values it has seen (one per lane) and
//     logs (k0, group) for every group with k0 <= its current k-th value;
//     since a warp's k-th value only decreases and never drops below the
//     global k-th value T, every group with k0 <= T is in some warp's log;
//   * a block merges its warps' values (k-way, heads in lanes) to its own k-th
//     value T_b >= T and publishes its values and the log entries <= T_b;
//   * the last block finds the exact T (every warp keeps the k smallest of a
//     share of the block values, warp 0 merges the 8 lists), keeps the
//     published entries with k0 <= T (the top k plus ties on k0; one flat pass
//     over all blocks' entries through a prefix of their counts), computes
//     their full keys in parallel, orders them with TopkList and writes the
//     output values with one thread per (row, column).
// Every step of the last block is a few rounds of independent loads: the
// tail no longer grows with the block count, so the walk runs 4 blocks per
// SM (more warps in flight for its dependent presence -> count -> limb loads)
// and each warp takes 4 presence words per lane (4096 slots) per round.
// A warp log that cannot hold the entries still at or below its k-th value
// (more than kTopkLog ties) flags the unit for the exact per-instruction path.
constexpr int kTopkLog = 64;
constexpr int kTopkBlkCand = 128;
constexpr int kTopkFinal = 128;
constexpr int kTopkSuperSlots = 512;   // compaction buffer per warp (slots)
constexpr int kTopkWords = 4;          // presence words per lane per round
constexpr int kTopkMaxBlocks = 1024;   // last block: prefix of the published counts in shared memory
constexpr int kTopkCollect = 1024;     // last block: published entries <= T1 held at once

// k-th smallest (k >= 1) of a warp's vals[0..m) in shared memory, ~0 when
// m < k (rank selection, as block_kth); every lane calls it
__device__ __noinline__ unsigned long long warp_kth(const unsigned long long* vals, int m, int k) {
  unsigned long long best = 0;
  for (int i = static_cast<int>(threadIdx.x & 31); i < m; i += 32) {
    const unsigned long long v = vals[i];
    int less = 0;
#pragma unroll 8
    for (int j = 0; j < m; ++j) less += vals[j] < v ? 1 : 0;
    if (less < k && v > best) best = v;
  }
  __syncwarp();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  return m < k ? ~0ULL : best;
}

// k-th smallest (k >= 1) of vals[0..m) in shared memory, ~0 when m < k:
// the largest v_i with fewer than k values below it (rank selection, all
// threads in parallel, no serial insert chain). Every thread of the block
// calls it; red holds one word per warp. Not inlined: the top-k kernel's
// last block runs its code cold (each new instruction line is an L2 fetch,
// ~0.15 us), and one copy shared by every call site is already in the
// instruction cache from the block phase.
__device__ __noinline__ unsigned long long block_kth(const unsigned long long* vals, int m, int k, unsigned long long* red) {
  unsigned long long best = 0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const unsigned long long v = vals[i];
    int less = 0;
#pragma unroll 8
    for (int j = 0; j < m; ++j) less += vals[j] < v ? 1 : 0;
    if (less < k && v > best) best = v;
  }
  __syncwarp();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  unsigned long long r = 0;
  for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) r = max(r, red[w]);
  __syncthreads();
  return m < k ? ~0ULL : r;
}

template <int NK>
__global__ void __launch_bounds__(kTopkThreads) k_topk_groups(const __grid_constant__ GroupSpec s, long long ngroups, int k,
                                                              unsigned long long* __restrict__ blk_ck,
                                                              unsigned* __restrict__ blk_cg, int* __restrict__ blk_nc,
                                                              unsigned* __restrict__ ticket,
                                                              long long* __restrict__ nout, long long* __restrict__ err,
                                                              unsigned long long* __restrict__ trace) {
  constexpr int kW = kTopkThreads / 32;
  // TQP_TOPK_TRACE: %globaltimer at the phase boundaries (debug aid)
  auto stamp = [&](long long at) {
    if (trace && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[at] = t;
    }
  };
  stamp(8LL * blockIdx.x);
  constexpr long long kSuper = 32LL * 32 * kTopkWords;  // slots per warp round
  __shared__ unsigned long long s_logk[kW][kTopkLog];
  __shared__ unsigned s_logg[kW][kTopkLog];
  __shared__ __align__(16) unsigned s_scratch[kW * kTopkSuperSlots];  // slot compaction; last block: prefix / keys
  __shared__ unsigned long long s_k0[kW][32 * kTopkUnroll];
  __shared__ unsigned s_gq[kW][32 * kTopkUnroll];
  __shared__ unsigned long long s_red[kW];
  __shared__ int s_nc, s_np, s_last, s_err;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  if (threadIdx.x == 0) {
    s_nc = 0;
    s_np = 0;
    s_err = 0;
  }
  __syncthreads();
  const long long n = ngroups;
  // the warp's log: every group it has seen with k0 <= tw; tw starts at ~0
  // and drops to the log's k-th value whenever the log fills (a parallel
  // rank selection, then the entries above it dropped), so it never falls
  // below the global k-th value T and no per-group serial list insert runs
  unsigned long long tw = ~0ULL;
  int nlog = 0;
  bool log_ok = true;
  unsigned* sidx = s_scratch + warp * kTopkSuperSlots;
  // keep the log entries <= the log's k-th value; tw = that value
  auto prune = [&]() {
    const unsigned long long t = warp_kth(s_logk[warp], nlog, k);
    int kept = 0;
    for (int i0 = 0; i0 < nlog; i0 += 32) {
      const int i = i0 + lane;
      const unsigned long long lk = i < nlog ? s_logk[warp][i] : ~0ULL;
      const unsigned lg = i < nlog ? s_logg[warp][i] : 0u;
      const bool keep = i < nlog && lk <= t;
      const unsigned km = __ballot_sync(0xffffffffu, keep);
      __syncwarp();
      if (keep) {
        const int pos = kept + __popc(km & lt_mask);
        s_logk[warp][pos] = lk;
        s_logg[warp][pos] = lg;
      }
      kept += __popc(km);
      __syncwarp();
    }
    nlog = kept;
    tw = t;
  };

  // the groups whose slots (relative to `base`) are sidx[0..total): their
  // counts and first key words are formed kTopkUnroll x 32 at a time (loads
  // together), then logged one 32-lane batch at a time
  long long cy_load = 0, cy_key = 0, cy_offer = 0, cy_t = 0;  // TQP_TOPK_TRACE: warp 0's cycles per walk part
  auto walk = [&](long long base, int total) {
    __syncwarp();
    for (int c0 = 0; c0 < total; c0 += 32 * kTopkUnroll) {
      if (trace) cy_t = clock64();
      unsigned gq[kTopkUnroll];
      unsigned long long gc[kTopkUnroll];
#pragma unroll
      for (int u = 0; u < kTopkUnroll; ++u) {
        const int i = c0 + u * 32 + lane;
        gq[u] = i < total ? static_cast<unsigned>(base) + sidx[i] : 0u;
        gc[u] = i < total ? s.gcnt[gq[u] * s.cnt_stride] : 0ULL;
        if (s.row_in_cnt) gc[u] &= 0xffffffffULL;
      }
#pragma unroll
      for (int u = 0; u < kTopkUnroll; ++u) {
        if (c0 + u * 32 >= total) break;  // warp-uniform: no slots left
        // limb sums are exact below kLimbMaxRows rows per group
        if (gc[u] && !group_limbs_ok(s, gq[u])) {
          err[0] = 1;
          err[3] = FR_LIMB_ROWS;
        }
        const unsigned long long k0 = gc[u] ? cand_key_word(s, 0, gq[u]) : ~0ULL;
        // reconverge: after a call from divergent lanes the warp stayed
        // split and every later shuffle took the slow (diverged) path -
        // measured 10x on a warp merge
        __syncwarp();
        if (trace && u == 0) {
          const long long t1 = clock64();
          cy_key += t1 - cy_t;
          cy_t = t1;
        }
        unsigned mask = __ballot_sync(0xffffffffu, gc[u] != 0 && k0 <= tw);
        if (!mask) continue;
        int m = __popc(mask);
        if (log_ok && nlog + m > kTopkLog) {
          prune();  // tw drops: only the lanes still at or below it are logged
          mask = __ballot_sync(0xffffffffu, gc[u] != 0 && k0 <= tw);
          m = __popc(mask);
          if (nlog + m > kTopkLog) log_ok = false;  // more ties than the log holds
        }
        if (log_ok && ((mask >> lane) & 1u)) {
          const int pos = nlog + __popc(mask & lt_mask);
          s_logk[warp][pos] = k0;
          s_logg[warp][pos] = gq[u];
        }
        nlog += m;
        __syncwarp();
      }
      if (trace) cy_offer += clock64() - cy_t;
    }
  };

  long long sb = static_cast<long long>(blockIdx.x) * kW + warp;
  const long long sb_step = static_cast<long long>(gridDim.x) * kW;
  // kTopkWords presence words per lane per round, the next round's loaded
  // while this one is walked
  auto load_words = [&](long long sbx, unsigned* w) {
    const long long base = sbx * kSuper;
#pragma unroll
    for (int u = 0; u < kTopkWords; ++u) {
      const long long wb = base + 32LL * (u * 32 + lane);
      w[u] = 0u;
      if (wb < n) {
        w[u] = s.present ? __ldg(s.present + (wb >> 5)) : ~0u;
        if (n - wb < 32) w[u] &= (1u << (n - wb)) - 1u;
      }
    }
  };
  unsigned wnext[kTopkWords];
  load_words(sb, wnext);
  for (; sb * kSuper < n; sb += sb_step) {
    // this round's present slots compacted into sidx, handed to walk() (one
    // call site) whenever the next word's slots would overflow it, and after
    // the last word
    const long long base = sb * kSuper;
    const long long cl0 = trace ? clock64() : 0;
    unsigned w[kTopkWords];
#pragma unroll
    for (int u = 0; u < kTopkWords; ++u) w[u] = wnext[u];
    load_words(sb + sb_step, wnext);
    // half a word-round (16 lanes' words, <= 512 slots) at a time, so one
    // step never exceeds the compaction buffer
    static_assert(kTopkSuperSlots >= 16 * 32, "compaction buffer below half a word-round");
    int fill = 0;
#pragma unroll 1
    for (int h = 0; h <= 2 * kTopkWords; ++h) {
      const bool last = h == 2 * kTopkWords;
      const unsigned xw = w[0];
      if (h & 1) {
#pragma unroll
        for (int v = 0; v + 1 < kTopkWords; ++v) w[v] = w[v + 1];  // next word to the front
        w[kTopkWords - 1] = 0u;
      }
      const unsigned x0 = !last && (lane >> 4) == (h & 1) ? xw : 0u;
      const int c = __popc(x0);
      int off = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, off, o);
        if (lane >= o) off += y;
      }
      const int total = __shfl_sync(0xffffffffu, off, 31);
      if (fill && (last || fill + total > kTopkSuperSlots)) {
        if (trace && last) cy_load += clock64() - cl0;
        walk(base, fill);
        fill = 0;
      }
      if (last) break;
      off += fill - c;
      unsigned x = x0;
      const unsigned rel = static_cast<unsigned>(32 * ((h >> 1) * 32 + lane));
      while (x) {
        const int bit = __ffs(x) - 1;
        x &= x - 1;
        sidx[off++] = rel + bit;
      }
      __syncwarp();
      fill += total;
    }
  }
  if (trace && threadIdx.x == 0) {
    trace[8LL * blockIdx.x + 5] = static_cast<unsigned long long>(cy_load);
    trace[8LL * blockIdx.x + 6] = static_cast<unsigned long long>(cy_key);
    trace[8LL * blockIdx.x + 7] = static_cast<unsigned long long>(cy_offer);
  }
  // the warp's own k-th value: its log shrinks to <= k entries plus ties
  if (log_ok && nlog > k) prune();
  if (!log_ok && lane == 0) s_err = 1;
  __syncthreads();
  stamp(8LL * blockIdx.x + 1);
  unsigned long long* cv = &s_k0[0][0];  // collection: values (kTopkCollect)
  unsigned* cg = &s_gq[0][0];            // collection: groups
  // block: every warp's log in one list, T_b = its k-th value (rank
  // selection), and the entries <= T_b published sorted by value
  {
    const int nl = log_ok ? nlog : 0;
    int basepos = 0;
    if (lane == 0 && nl) basepos = atomicAdd(&s_nc, nl);
    basepos = __shfl_sync(0xffffffffu, basepos, 0);
    for (int i = lane; i < nl; i += 32) {
      cv[basepos + i] = s_logk[warp][i];
      cg[basepos + i] = s_logg[warp][i];
    }
    __syncthreads();
    const int ncv = s_nc;  // <= kW * kTopkLog <= kTopkCollect
    const unsigned long long tb = block_kth(cv, ncv, k, s_red);
    for (int t = threadIdx.x; t < ncv; t += kTopkThreads) {
      const unsigned long long v = cv[t];
      if (v > tb) continue;
      int r = 0;  // rank by (value, position) among the entries <= T_b
#pragma unroll 8
      for (int j = 0; j < ncv; ++j) r += cv[j] <= tb && (cv[j] < v || (cv[j] == v && j < t)) ? 1 : 0;
      if (r < kTopkBlkCand) {
        blk_ck[static_cast<long long>(blockIdx.x) * kTopkBlkCand + r] = v;
        blk_cg[static_cast<long long>(blockIdx.x) * kTopkBlkCand + r] = cg[t];
      }
      atomicAdd(&s_np, 1);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (s_np > kTopkBlkCand) s_err = 1;
    blk_nc[blockIdx.x] = s_np < kTopkBlkCand ? s_np : kTopkBlkCand;
    if (s_err) {
      err[0] = 1;
      err[3] = FR_TOPK_BLOCK;
    }
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  stamp(8LL * blockIdx.x + 2);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int nb = static_cast<int>(gridDim.x);
  const long long tl = 8LL * nb;
  // last block. Every block published its groups with k0 <= T_b sorted, and
  // T (the global k-th value) <= every T_b, so the groups with k0 <= T are
  // all published. T1 = the k-th smallest of the first kTopkThreads blocks'
  // minima is >= T (k distinct groups at or below it); the published entries
  // <= T1 (a short sorted prefix per block) hold every group <= T, and T is
  // their k-th smallest.
  static_assert(sizeof(int) * kTopkMaxBlocks + sizeof(unsigned long long) * kTopkThreads +
                        sizeof(unsigned) * (kTopkFinal + 2) + 8 + sizeof(unsigned long long) * kTopkFinal * 8 +
                        sizeof(unsigned) * kTopkMaxK <=
                    sizeof(unsigned) * kTopkThreads / 32 * kTopkSuperSlots,
                "last-block scratch exceeds the compaction buffers");
  static_assert(kTopkThreads / 32 * 32 * kTopkUnroll >= kTopkCollect, "collection exceeds the staging buffers");
  static_assert(kTopkThreads / 32 * kTopkLog <= kTopkCollect, "block logs exceed the collection");
  int* cnb = reinterpret_cast<int*>(s_scratch);                        // [nb]
  unsigned long long* bmin = reinterpret_cast<unsigned long long*>(cnb + kTopkMaxBlocks);  // [kTopkThreads]
  for (int b = threadIdx.x; b < nb; b += kTopkThreads) cnb[b] = __ldcg(blk_nc + b);
  if (threadIdx.x < kTopkThreads) {
    const int b = threadIdx.x;
    bmin[b] = b < nb && __ldcg(blk_nc + b) > 0 ? __ldcg(blk_ck + static_cast<long long>(b) * kTopkBlkCand) : ~0ULL;
  }
  if (threadIdx.x == 0) s_nc = 0;
  __syncthreads();
  stamp(tl + 6);
  const unsigned long long T1 = block_kth(bmin, min(nb, kTopkThreads), k, s_red);
  for (int b = threadIdx.x; b < nb; b += kTopkThreads) {
    const int nc = cnb[b];
    for (int i0 = 0; i0 < nc; i0 += 4) {
      unsigned long long v[4];
      unsigned g[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // keys and groups loaded together
        v[u] = i0 + u < nc ? __ldcg(blk_ck + static_cast<long long>(b) * kTopkBlkCand + i0 + u) : ~0ULL;
        g[u] = i0 + u < nc ? __ldcg(blk_cg + static_cast<long long>(b) * kTopkBlkCand + i0 + u) : 0u;
      }
      bool more = true;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (i0 + u < nc && v[u] <= T1) {
          const int pos = atomicAdd(&s_nc, 1);
          if (pos < kTopkCollect) {
            cv[pos] = v[u];
            cg[pos] = g[u];
          }
        } else {
          more = false;
        }
      }
      if (!more) break;  // sorted: the rest is above T1
    }
  }
  __syncthreads();
  stamp(tl + 7);
  const int m = s_nc;
  if (m > kTopkCollect) {  // ties: more entries at or below T1 than the collection holds
    if (threadIdx.x == 0) {
      err[0] = 1;
      err[3] = FR_TOPK_FINAL;
      *nout = 0;
    }
    return;
  }
  const unsigned long long T = block_kth(cv, m, k, s_red);
  stamp(tl);
  // final candidates: the collected entries <= T (the top k plus ties on k0)
  unsigned* fg = reinterpret_cast<unsigned*>(bmin + kTopkThreads);
  if (threadIdx.x == 0) s_nc = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += kTopkThreads) {
    if (cv[i] <= T) {
      const int pos = atomicAdd(&s_nc, 1);
      if (pos < kTopkFinal) fg[pos] = cg[i];
    }
  }
  __syncthreads();
  stamp(tl + 1);
  const int nfc = s_nc < kTopkFinal ? s_nc : kTopkFinal;
  if (threadIdx.x == 0 && s_nc > kTopkFinal) {
    err[0] = 1;
    err[3] = FR_TOPK_FINAL;
  }
  // full keys, one thread per (candidate, key word); then each candidate's
  // rank among the candidates (keys are unique: the group keys end them)
  unsigned long long* fk = reinterpret_cast<unsigned long long*>(fg + kTopkFinal + 2);
  fk = reinterpret_cast<unsigned long long*>((reinterpret_cast<uintptr_t>(fk) + 7) & ~uintptr_t(7));
  unsigned* og = reinterpret_cast<unsigned*>(fk + kTopkFinal * NK);  // output groups in order
  for (int t = threadIdx.x; t < nfc * NK; t += kTopkThreads) {
    const int i = t % nfc, q = t / nfc;
    fk[i * NK + q] = cand_key_word(s, q, fg[i]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nfc; i += kTopkThreads) {
    int r = 0;
    for (int j = 0; j < nfc; ++j) {
      bool lt = false, eq = true;
#pragma unroll
      for (int q = 0; q < NK; ++q) {
        const unsigned long long a = fk[j * NK + q], c = fk[i * NK + q];
        lt = lt || (eq && a < c);
        eq = eq && a == c;
      }
      r += lt;
    }
    if (r < k) og[r] = fg[i];
  }
  __syncthreads();
  stamp(tl + 2);
  // output values: a thread per (row, column)
  const int nrow = min(nfc, k);
  if (threadIdx.x == 0) *nout = nrow;
  for (int t = threadIdx.x; t < nrow * s.f.nouts; t += blockDim.x) {
    const int r = t % nrow, j = t / nrow;
    unsigned long long bits;
    bool f;
    if (!group_out_value(s, j, og[r], bits, f)) {
      err[0] = 1;
      err[3] = FR_GROUP_VALUE;
    }
    store_group_out(s, j, r, bits);
  }
  __syncthreads();
  stamp(tl + 3);
  if (trace && threadIdx.x == 0) {
    trace[tl + 4] = static_cast<unsigned long long>(m);
    trace[tl + 5] = static_cast<unsigned long long>(nfc);
  }
}

// TQP_TOPK_TRACE: phase times of one k_topk_groups launch (stderr, us from
// the first block's start): walk end and publish end over the blocks
// (median / max), warp 0's walk cycles by part, then the last block's phases
void topk_trace_report(Ctx& c, const std::shared_ptr<DevBuf>& tb, int nb) {
  std::vector<unsigned long long> t(8 * nb + 12);
  TQP_CUDA(cudaMemcpyAsync(t.data(), tb->ptr, sizeof(unsigned long long) * t.size(), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  unsigned long long t0 = ~0ULL;
  for (int b = 0; b < nb; ++b) t0 = std::min(t0, t[8 * b]);
  std::vector<double> we, pe, w5, w6, w7;
  for (int b = 0; b < nb; ++b) {
    we.push_back((t[8 * b + 1] - t0) / 1e3);
    pe.push_back((t[8 * b + 2] - t0) / 1e3);
    w5.push_back(t[8 * b + 5] / 1.965e3);
    w6.push_back(t[8 * b + 6] / 1.965e3);
    w7.push_back(t[8 * b + 7] / 1.965e3);
  }
  auto med = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
  auto mx = [](const std::vector<double>& v) { return *std::max_element(v.begin(), v.end()); };
  const long long tl = 8LL * nb;
  auto at = [&](long long i) { return (t[tl + i] - t0) / 1e3; };
  std::fprintf(stderr,
               "topk trace nb=%d walk end med %.1f max %.1f | publish end med %.1f max %.1f | warp0 walk: presence "
               "%.2f keys %.2f offers %.2f us\n",
               nb, med(we), mx(we), med(pe), mx(pe), med(w5), med(w6), med(w7));
  std::fprintf(stderr,
               "topk trace last block: loads %.1f collect %.1f T %.1f finals %.1f keys+rank %.1f out %.1f | "
               "collected %llu finals %llu\n",
               at(6), at(7), at(0), at(1), at(2), at(3), t[tl + 4], t[tl + 5]);
}

// walk blocks per SM (TQP_TOPK_BPS tuning knob)
int topk_bps() {
  static const int v = [] {
    const char* e = std::getenv("TQP_TOPK_BPS");
    const int x = e ? std::atoi(e) : 4;
    return x >= 1 && x <= 8 ? x : 4;
  }();
  return v;
}

using TopkKernel = void (*)(GroupSpec, long long, int, unsigned long long*, unsigned*, int*, unsigned*, long long*,
                            long long*, unsigned long long*);
TopkKernel topk_kernel(int nk) {
  switch (nk) {
    case 1: return k_topk_groups<1>;
    case 2: return k_topk_groups<2>;
    case 3: return k_topk_groups<3>;
    case 4: return k_topk_groups<4>;
    case 5: return k_topk_groups<5>;
    case 6: return k_topk_groups<6>;
    case 7: return k_topk_groups<7>;
    case 8: return k_topk_groups<8>;
    default: return nullptr;
  }
}

__global__ void k_group_rows(const __grid_constant__ GroupSpec s, const long long* __restrict__ gids, const long long* __restrict__ order,
                             long long n, long long* err) {
  for (long long r = gtid(); r < n; r += gstride()) {
    unsigned g = static_cast<unsigned>(gids[order ? order[r] : r]);
    for (int j = 0; j < s.f.nouts; ++j) {
      unsigned long long bits;
      bool f;
      if (!group_out_value(s, j, g, bits, f)) {
        err[0] = 1;
        err[3] = FR_GROUP_VALUE;
      }
      store_group_out(s, j, r, bits);
    }
  }
}

// ascending slots i < n with cnt[i * stride] != 0: one pass, a tile of
// kSlotTile slots per CTA (dynamic tile ids), ballot + popcount per warp item,
// the output offset from the decoupled lookback (scan.cuh)
constexpr int kSlotThreads = 256, kSlotItems = 8, kSlotTile = kSlotThreads * kSlotItems;
__global__ void __launch_bounds__(kSlotThreads) k_nonzero_slots(const unsigned long long* __restrict__ cnt, long long stride,
                                                                long long n, long long* __restrict__ out, longlong2* desc,
                                                                int* counter) {
  __shared__ int s_tile;
  __shared__ unsigned long long s_warp[kSlotThreads / 32 + 1];
  __shared__ long long s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1);
  __syncthreads();
  const int tile = s_tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long wbase = static_cast<long long>(tile) * kSlotTile + static_cast<long long>(warp) * 32 * kSlotItems + lane;
  unsigned ball[kSlotItems];
  unsigned mine = 0;
#pragma unroll
  for (int j = 0; j < kSlotItems; ++j) {
    const long long i = wbase + j * 32;
    ball[j] = __ballot_sync(0xffffffffu, i < n && __ldg(cnt + i * stride) != 0ULL);
    mine += __popc(ball[j]);
  }
  if (lane == 0) s_warp[warp] = mine;
  __syncthreads();
  if (warp == 0) {
    constexpr int kW = kSlotThreads / 32;
    const unsigned long long w = lane < kW ? s_warp[lane] : 0ULL;
    unsigned long long wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    __syncwarp();
    if (lane < kW) s_warp[lane] = wi - w;
    const unsigned long long total = __shfl_sync(0xffffffffu, wi, kW - 1);
    const long long pfx = tile_lookback(desc, tile, static_cast<long long>(total));
    if (lane == 0) s_prefix = pfx;
  }
  __syncthreads();
  unsigned long long pos = static_cast<unsigned long long>(s_prefix) + s_warp[warp];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kSlotItems; ++j) {
    if ((ball[j] >> lane) & 1u) out[pos + __popc(ball[j] & lt)] = wbase + j * 32;
    pos += __popc(ball[j]);
  }
}

__global__ void k_nonzero_groups(const unsigned long long* __restrict__ cnt, long long cnt_stride, long long n,
                                 const unsigned* present, unsigned long long cmask, uint8_t* __restrict__ mask) {
  for (long long i = gtid(); i < n; i += gstride())
    mask[i] = (!present || ((__ldg(present + (i >> 5)) >> (i & 31)) & 1u)) && (cnt[i * cnt_stride] & cmask) != 0;
}

// MODE_HASH direct tables: bit per slot with rows
__global__ void k_count_present(const unsigned long long* __restrict__ cnt, long long stride, long long cap,
                                unsigned* __restrict__ present) {
  const long long n32 = (cap + 31) & ~31LL;
  for (long long i = gtid(); i < n32; i += gstride()) {
    const unsigned bits = __ballot_sync(0xffffffffu, i < cap && cnt[i * stride] != 0ULL);
    if ((threadIdx.x & 31) == 0) present[i >> 5] = bits;
  }
}
// MODE_HASH: bit per claimed slot of the group table
__global__ void k_hash_present(const unsigned long long* __restrict__ tag, long long cap, unsigned* __restrict__ present) {
  const long long n32 = (cap + 31) & ~31LL;  // warp-uniform trip count (blockDim % 32 == 0)
  for (long long i = gtid(); i < n32; i += gstride()) {
    const unsigned bits = __ballot_sync(0xffffffffu, i < cap && tag[i] != 0ULL);
    if ((threadIdx.x & 31) == 0) present[i >> 5] = bits;
  }
}
// the build key of each group: through the group table, or (row_rec) the
// row kept in bits 32-63 of the group's count word
__global__ void k_group_keys(const unsigned long long* __restrict__ group_table, const unsigned long long* __restrict__ rowcnt,
                             long long cnt_stride, const long long* __restrict__ gids, long long n,
                             const long long* __restrict__ key_col, long long* __restrict__ out) {
  for (long long i = gtid(); i < n; i += gstride()) {
    const long long g = gids[i];
    const long long row = group_table ? static_cast<long long>(group_table[g] & 0xffffffffULL) - 1
                          : rowcnt    ? static_cast<long long>(rowcnt[g * cnt_stride] >> 32) - 1
                                      : g;
    out[i] = key_col ? key_col[row] : g;
  }
}

// ---- sharded-run partials ------------------------------------------------------
// A partial is a device buffer of u64 words: an 8-word header
//   [magic, mode, nrec, words per record, nacc, nouts, nkeys, 0]
// followed by nrec records: MODE_SCALAR per-CTA sums [kMaxAcc + 1];
// MODE_SMALL per-CTA SmallPart; MODE_BUILDGRP one record per touched group
//   [build key, group key columns..., count, (lo, hi) per accumulator].
constexpr unsigned long long kPartMagic = 0x3154524150505154ULL;  // "TQPPART1"
constexpr int kHdrWords = 8;
constexpr int kSmallPartWords = static_cast<int>(sizeof(SmallPart) / sizeof(unsigned long long));
static_assert(sizeof(SmallPart) % sizeof(unsigned long long) == 0, "SmallPart must be word-sized");
constexpr int record_words(int nkeyc, int nacc) { return 2 + nkeyc + 2 * nacc; }

__global__ void k_fill_records(const __grid_constant__ GroupSpec s, const long long* __restrict__ gids, long long n,
                               const long long* __restrict__ bkey, int words, unsigned long long* __restrict__ out,
                               long long* err) {
  for (long long i = gtid(); i < n; i += gstride()) {
    const unsigned g = static_cast<unsigned>(gids[i]);
    const long long row = group_src_row(s, g);
    unsigned long long* w = out + i * words;
    w[0] = s.direct_codes ? static_cast<unsigned long long>(g)
           : s.codes      ? s.codes[g] - 1ULL
                          : static_cast<unsigned long long>(bkey[row]);
    for (int k = 0; k < s.nkeyc; ++k) w[1 + k] = static_cast<unsigned long long>(group_key_value(s, k, g));
    w[1 + s.nkeyc] = static_cast<unsigned long long>(group_count(s, g));
    if (!group_limbs_ok(s, g)) {
      err[0] = 1;
      err[3] = FR_GROUP_VALUE;
    }
    for (int a = 0; a < s.f.nacc; ++a) {  // records carry int128 (lo, hi)
      const unsigned __int128 v = static_cast<unsigned __int128>(group_acc(s, g, a));
      w[2 + s.nkeyc + 2 * a] = static_cast<unsigned long long>(v);
      w[3 + s.nkeyc + 2 * a] = static_cast<unsigned long long>(v >> 64);
    }
  }
}

// records -> open-addressing table keyed by the build key (tag = key ^ 2^63,
// 0 = empty); counts and Q64.64 sums add exactly, so the merge is
// order-independent and equals the unsharded run bit for bit
__global__ void k_merge_records(const unsigned long long* __restrict__ rec, long long n, int words, int nkeyc, int nacc,
                                long long mask, unsigned long long* __restrict__ tag, long long* __restrict__ hbk,
                                long long* __restrict__ hkeys, unsigned long long* __restrict__ hcnt,
                                unsigned long long* __restrict__ hacc, long long* err) {
  const long long cap = mask + 1;
  for (long long i = gtid(); i < n; i += gstride()) {
    const unsigned long long* r = rec + i * words;
    const unsigned long long t = r[0] ^ 0x8000000000000000ULL;
    if (t == 0) {
      err[0] = 1;
      continue;
    }
    long long h = static_cast<long long>((r[0] * 0x9E3779B97F4A7C15ULL) >> 20) & mask;
    unsigned long long prev;
    for (;;) {
      prev = atomicCAS(&tag[h], 0ULL, t);
      if (prev == 0ULL || prev == t) break;
      h = (h + 1) & mask;
    }
    if (prev == 0ULL) {
      hbk[h] = static_cast<long long>(r[0]);
      for (int k = 0; k < nkeyc; ++k) hkeys[k * cap + h] = static_cast<long long>(r[1 + k]);
    }
    atomicAdd(&hcnt[h], r[1 + nkeyc]);
    for (int a = 0; a < nacc; ++a) {
      const unsigned long long lo = r[2 + nkeyc + 2 * a], hi = r[3 + nkeyc + 2 * a];
      const __int128 v = static_cast<__int128>((static_cast<unsigned __int128>(hi) << 64) | lo);
      // a shard's sum is < 2^62 (q64_range_check) so |v| < 2^126; partials
      // at or above 2^122 could wrap the int128 once 32 shards are added
      const __int128 lim = static_cast<__int128>(1) << 122;
      if (v >= lim || v <= -lim) err[0] = 1;
      atomic_add_q64(&hacc[(h * nacc + a) * 2], v);
    }
  }
}

// ---- unit runner ----------------------------------------------------------------
const Column* find_col(const TableSet& tables, const std::string& t, const std::string& c) {
  const Table* tab = bind_table(tables, t);
  return tab ? tab->find(c) : nullptr;
}

Operand make_operand(const TableSet& tables, const PipeDesc& P, const OperandDesc& o, bool* ok) {
  Operand r;
  const std::string& table = o.probe < 0 ? P.fact_table : P.builds[P.probes[o.probe].build].table;
  const Column* c = find_col(tables, table, o.column);
  if (!c) {
    *ok = false;
    return r;
  }
  r.ptr = c->t.data();
  r.type = c->t.dtype == TQP_F64 ? OT_F64 : (c->t.dtype == TQP_STR8 || c->t.dtype == TQP_BOOL) ? OT_U8 : OT_I64;
  r.src = o.probe;
  if (r.type == OT_U8 && c->t.cols != 1) *ok = false;
  if (reinterpret_cast<uintptr_t>(r.ptr) % 16) *ok = false;
  return r;
}

bool make_term(const TableSet& tables, const std::string& table, const TermDesc& t, Term* nt, StrTerm* st, bool* is_str) {
  *is_str = false;
  if (t.kind == 3 || t.kind == 4) {
    nt->kind = t.kind == 3 ? TK_TRUE : TK_FALSE;
    return true;
  }
  const Column* c = find_col(tables, table, t.column);
  if (!c) return false;
  if (t.kind == 0) {
    nt->x.ptr = c->t.data();
    nt->x.src = -1;
    if (c->t.dtype == TQP_F64) {
      if (!t.f64) return false;
      nt->x.type = OT_F64;
      nt->kind = TK_F64;
      nt->fk = t.fk;
    } else if (c->t.dtype == TQP_I64) {
      if (t.f64) return false;
      nt->x.type = OT_I64;
      nt->kind = TK_INT;
      nt->ik = t.ik;
    } else {
      return false;
    }
    nt->op = t.op;
    return true;
  }
  if (c->t.dtype != TQP_STR8) return false;
  *is_str = true;
  st->ptr = c->t.ptr<uint8_t>();
  st->width = static_cast<int>(c->t.cols);
  st->is_like = t.kind == 2;
  st->op = t.op;
  st->anchor = t.anchor;
  st->litlen = static_cast<int>(t.lit.size());
  std::memcpy(st->lit, t.lit.data(), t.lit.size());
  return true;
}

// Numeric conjuncts -> one branch-free range per column (RTerm). int64:
// x < K == x <= K-1 etc.; fp64: x < K == x <= nextafter(K, -inf) for every
// non-NaN x, and NaN fails lo <= x <= hi exactly as it fails `<`/`>`.
bool merge_range_terms(const std::vector<Term>& in, ProbeSpec& ps, std::vector<Operand>& cols) {
  struct R {
    Operand x;
    bool f64;
    long long ilo, ihi;
    double flo, fhi;
    bool empty = false;
  };
  std::vector<R> ranges;
  std::vector<std::pair<Operand, Term>> ne;
  bool any_false = false;
  for (const Term& t : in) {
    if (t.kind == TK_TRUE) continue;
    if (t.kind == TK_FALSE) {
      any_false = true;
      continue;
    }
    if (t.op == TQP_NE) {
      ne.push_back({t.x, t});
      continue;
    }
    R r;
    r.x = t.x;
    r.f64 = t.kind == TK_F64;
    r.ilo = std::numeric_limits<long long>::min();
    r.ihi = std::numeric_limits<long long>::max();
    r.flo = -std::numeric_limits<double>::infinity();
    r.fhi = std::numeric_limits<double>::infinity();
    if (r.f64) {
      const double k = t.fk;
      if (std::isnan(k)) {
        r.empty = true;
      } else {
        switch (t.op) {
          case TQP_EQ: r.flo = r.fhi = k; break;
          case TQP_LT: r.fhi = std::nextafter(k, -std::numeric_limits<double>::infinity()); break;
          case TQP_LE: r.fhi = k; break;
          case TQP_GT: r.flo = std::nextafter(k, std::numeric_limits<double>::infinity()); break;
          default: r.flo = k; break;
        }
        if (t.op == TQP_LT && k == -std::numeric_limits<double>::infinity()) r.empty = true;
        if (t.op == TQP_GT && k == std::numeric_limits<double>::infinity()) r.empty = true;
      }
    } else {
      const long long k = t.ik;
      switch (t.op) {
        case TQP_EQ: r.ilo = r.ihi = k; break;
        case TQP_LT:
          if (k == std::numeric_limits<long long>::min()) r.empty = true;
          else r.ihi = k - 1;
          break;
        case TQP_LE: r.ihi = k; break;
        case TQP_GT:
          if (k == std::numeric_limits<long long>::max()) r.empty = true;
          else r.ilo = k + 1;
          break;
        default: r.ilo = k; break;
      }
    }
    bool merged = false;
    for (auto& q : ranges) {
      if (q.x.ptr == r.x.ptr && q.f64 == r.f64) {
        q.ilo = std::max(q.ilo, r.ilo);
        q.ihi = std::min(q.ihi, r.ihi);
        q.flo = std::max(q.flo, r.flo);
        q.fhi = std::min(q.fhi, r.fhi);
        q.empty = q.empty || r.empty;
        merged = true;
      }
    }
    if (!merged) ranges.push_back(r);
  }
  auto push = [&](const RTerm& rt, const Operand& x) {
    if (ps.nterms >= kMaxTerms) return false;
    ps.terms[ps.nterms++] = rt;
    cols.push_back(x);
    return true;
  };
  if (any_false) {
    RTerm f;
    f.kind = RK_FALSE;
    return push(f, Operand{});
  }
  for (const auto& r : ranges) {
    RTerm rt;
    if (r.empty || (r.f64 ? !(r.flo <= r.fhi) : r.ilo > r.ihi)) {
      rt.kind = RK_FALSE;
    } else if (r.f64) {
      rt.kind = RK_F64;
      std::memcpy(&rt.lo, &r.flo, 8);
      std::memcpy(&rt.hi, &r.fhi, 8);
    } else {
      rt.kind = RK_INT;
      rt.lo = static_cast<unsigned long long>(r.ilo);
      rt.hi = static_cast<unsigned long long>(r.ihi);
    }
    if (!push(rt, r.x)) return false;
  }
  for (const auto& [x, t] : ne) {
    RTerm rt;
    rt.kind = t.kind == TK_F64 ? RK_F64_NE : RK_INT_NE;
    if (t.kind == TK_F64) std::memcpy(&rt.lo, &t.fk, 8);
    else rt.lo = static_cast<unsigned long long>(t.ik);
    if (!push(rt, x)) return false;
  }
  return true;
}

// k_tile<MODE, NA> instantiation for an accumulator count (nullptr: none)
const void* tile_kernel(int mode, int nacc) {
#define TQP_TK(M, N) \
  if (mode == M && nacc == N) return reinterpret_cast<const void*>(&k_tile<M, N>);
  TQP_TK(MODE_SCALAR, 0) TQP_TK(MODE_SCALAR, 1) TQP_TK(MODE_SCALAR, 2) TQP_TK(MODE_SCALAR, 3) TQP_TK(MODE_SCALAR, 4)
  TQP_TK(MODE_SMALL, 1) TQP_TK(MODE_SMALL, 2) TQP_TK(MODE_SMALL, 3) TQP_TK(MODE_SMALL, 4) TQP_TK(MODE_SMALL, 5)
  TQP_TK(MODE_SMALL, 6)
  TQP_TK(MODE_BUILDGRP, 0) TQP_TK(MODE_BUILDGRP, 1) TQP_TK(MODE_BUILDGRP, 2) TQP_TK(MODE_BUILDGRP, 3) TQP_TK(MODE_BUILDGRP, 4)
  TQP_TK(MODE_HASH, 0) TQP_TK(MODE_HASH, 1) TQP_TK(MODE_HASH, 2) TQP_TK(MODE_HASH, 3) TQP_TK(MODE_HASH, 4)
#undef TQP_TK
  return nullptr;
}

const void* tile_kernel_lean(int nacc) {
  switch (nacc) {
    case 1: return reinterpret_cast<const void*>(&k_tile<MODE_HASH, 1, true>);
    case 2: return reinterpret_cast<const void*>(&k_tile<MODE_HASH, 2, true>);
    case 3: return reinterpret_cast<const void*>(&k_tile<MODE_HASH, 3, true>);
    case 4: return reinterpret_cast<const void*>(&k_tile<MODE_HASH, 4, true>);
    default: return tile_kernel(MODE_HASH, nacc);
  }
}

// ---- run-time specialised pipeline kernels (jit.cu) ------------------------------
// The generic k_tile reads its pipeline description from shared memory and
// dispatches per term / factor at run time. For large scans the same pipeline
// is emitted as straight-line CUDA with every offset, bound and coefficient a
// literal, compiled once per process by NVRTC and run with the identical
// staging skeleton and partial layouts (jit_tile.cuh). The generated code keeps
// k_tile's exact floating-point operation order (__dadd_rn/__dmul_rn, no FMA
// contraction), so both kernels produce the same bits.
std::string hex64(unsigned long long v) {
  char b[40];
  std::snprintf(b, sizeof(b), "0x%016llxULL", v);
  return b;
}
std::string dlit(double d) {
  unsigned long long u;
  std::memcpy(&u, &d, 8);
  return "__longlong_as_double((long long)" + hex64(u) + ")";
}

// Small-group scans first run with 4 group slots per CTA: the per-thread
// shared-memory cells then take half the space, which goes to one more
// staging buffer (the scan is bound by the bytes each SM keeps in flight:
// 3 -> 4 stages of 43 KB). A CTA meeting a fifth key flags err[1] and the
// unit reruns with the 8-slot kernel. Per-thread row order is unchanged, so
// both give the same bits.
bool small_wide_wanted() {
  const char* e = std::getenv("TQP_SMALL_WIDE");
  return !(e && (e[0] == '0' || e[0] == 'n'));
}
constexpr int kWideSlots = 4;
constexpr int kWideCW = 8;
// 4-slot kernel with register accumulators (TQP_SMALL_REG=0: shared-memory
// cells); TQP_SMALL_CW / TQP_SMALL_ROWS: its consumer warps / tile rows.
// Q1 SF10 per launch (B200): cells 486 us; registers 14 warps x 4 rows per
// thread (1792-row tiles) 365 us, 12 x 4 402 us, 10 x 4 406 us, 14 x 3 418
// us, 12 x 2 660 us - four rows per thread keep the staged loads in flight.
bool small_regacc() {
  const char* e = std::getenv("TQP_SMALL_REG");
  return !(e && (e[0] == '0' || e[0] == 'n'));
}
int small_reg_cw() {
  static const int v = [] { const char* e = std::getenv("TQP_SMALL_CW"); const int x = e ? std::atoi(e) : 14;
                            return x >= 4 && x <= 24 ? x : 14; }();
  return v;
}
int small_reg_rows() {
  static const int v = [] { const char* e = std::getenv("TQP_SMALL_ROWS"); const int x = e ? std::atoi(e) : 1792;
                            return x >= 32 * small_reg_cw() && x <= 4096 && x % (32 * small_reg_cw()) == 0 ? x : 32 * small_reg_cw() * 4; }();
  return v;
}

bool jit_wanted(long long rows) {
  const char* e = std::getenv("TQP_JIT");
  if (e && (e[0] == '0' || e[0] == 'n')) return false;
  if (e && (e[0] == '1' || e[0] == 'a' || e[0] == 'y')) return true;
  return rows >= (1LL << 20);  // below this the NVRTC compile is not worth it
}

// How a generated fact probe asks a build side. Every build fills its
// presence bitmap; the table entry is only needed for the LIKE flag bits it
// carries. PM_TABLE: unfiltered build (every in-range key is a table hit or a
// zero entry), read the entry; PM_BITMAP_TABLE: filtered build with flags,
// presence word first, entry for the flags; PM_BITMAP: no flags wanted, the
// presence bit is the answer and the table is never read.
enum { PM_TABLE = 0, PM_BITMAP_TABLE = 1, PM_BITMAP = 2 };
bool build_filtered(const BuildDesc& B) { return !B.terms.empty() || !B.children.empty(); }
int probe_mode_of(const BuildDesc& B) {
  if (B.flags.empty()) return PM_BITMAP;
  return build_filtered(B) ? PM_BITMAP_TABLE : PM_TABLE;
}

std::string gen_pipeline(const TileSpec& ts, int mode, int cw, const std::vector<int>& probe_mode,
                         int slots = kGroups, bool regacc = false) {
  const ProbeSpec& s = ts.p;
  std::ostringstream o;
  unsigned int_mask = 0;
  for (int a = 0; a < s.nacc; ++a)
    if (s.acc[a].is_int) int_mask |= 1u << a;
  o << "#include \"fz_layout.cuh\"\n"
    << "#define Q_MODE " << mode << "\n#define Q_NA " << s.nacc << "\n#define Q_ROWS " << ts.rows << "\n#define Q_CW "
    << cw << "\n#define Q_INT_MASK " << int_mask << "u\n#define Q_SLOTS " << slots << "\n#define Q_REGACC "
    << (regacc ? 1 : 0) << "\n"
    << "namespace tqp { namespace fz {\n"
    << "__device__ __forceinline__ unsigned long long q_u64(const unsigned char* st, unsigned off, int ri) {\n"
    << "  return *reinterpret_cast<const unsigned long long*>(st + off + ri * 8); }\n"
    << "__device__ __forceinline__ double q_f64(const unsigned char* st, unsigned off, int ri) {\n"
    << "  return __longlong_as_double(static_cast<long long>(q_u64(st, off, ri))); }\n"
    << "__device__ __forceinline__ bool q_row(const TileSpec& t, const unsigned char* __restrict__ stage, int ri, bool valid,\n"
    << "    unsigned long long* v, unsigned& code, unsigned& gid, long long& absmax) {\n"
    << "  bool pass = valid;\n";
  auto off = [&](int col) { return std::to_string(ts.col_off[col]) + "u"; };
  for (int i = 0; i < s.nterms; ++i) {
    const RTerm& t = s.terms[i];
    switch (t.kind) {
      case RK_INT:
        o << "  pass = pass && (q_u64(stage, " << off(t.col) << ", ri) - " << hex64(t.lo) << ") <= " << hex64(t.hi - t.lo)
          << ";\n";
        break;
      case RK_F64: {
        double lo, hi;
        std::memcpy(&lo, &t.lo, 8);
        std::memcpy(&hi, &t.hi, 8);
        o << "  { const double x = q_f64(stage, " << off(t.col) << ", ri); pass = pass && x >= " << dlit(lo)
          << " && x <= " << dlit(hi) << "; }\n";
        break;
      }
      case RK_INT_NE: o << "  pass = pass && q_u64(stage, " << off(t.col) << ", ri) != " << hex64(t.lo) << ";\n"; break;
      case RK_F64_NE: {
        double k;
        std::memcpy(&k, &t.lo, 8);
        o << "  pass = pass && q_f64(stage, " << off(t.col) << ", ri) != " << dlit(k) << ";\n";
        break;
      }
      case RK_TRUE: break;
      default: o << "  pass = false;\n"; break;
    }
  }
  for (int p = 0; p < s.nprobes; ++p) {
    // branch-free: the loads of all of a thread's rows issue back to back
    o << "  unsigned fl" << p << " = 0u, gid" << p << " = 0u;\n"
      << "  { const Probe& pr = t.p.probes[" << p << "];\n"
      << "    const long long idx = static_cast<long long>(q_u64(stage, " << off(s.probes[p].key.col) << ", ri)) - pr.kmin;\n"
      << "    bool in = pass && static_cast<unsigned long long>(idx) < static_cast<unsigned long long>(pr.range);\n";
    if (probe_mode[p] != PM_TABLE)
      o << "    const unsigned w = in ? __ldg(pr.bitmap + (idx >> 5)) : 0u;\n"
        << "    in = in && ((w >> (idx & 31)) & 1u);\n";
    if (probe_mode[p] == PM_BITMAP) {
      // presence is the whole answer: no flags wanted, the group is the slot
      o << "    pass = pass && in;\n";
    } else {
      o << "    const unsigned long long e = in ? __ldg(pr.table + idx) : 0ULL;\n"
        << "    pass = pass && e != 0ULL;\n"
        << "    fl" << p << " = static_cast<unsigned>(e >> 57);\n";
    }
    o << "    gid" << p << " = static_cast<unsigned>(idx); }\n";
  }
  if (mode == MODE_BUILDGRP) {
    if (s.group_probe < 0 || s.group_probe >= s.nprobes) throw Error(TQP_ERR_EXEC, "internal: build-group pipeline without a group probe");
    o << "  gid = gid" << s.group_probe << ";\n";
  }
  if (mode == MODE_HASH) {
    // lean hash-group shape only (fact int keys, direct table): the group's
    // slot is its code, the mixed-radix number of the key digits
    o << "  { unsigned long long c = 0ULL;\n";
    for (int q = 0; q < s.nhkeys; ++q) {
      const GKey& K = s.hkeys[q];
      o << "    { unsigned long long d = q_u64(stage, " << off(K.x.col) << ", ri) - " << hex64(static_cast<unsigned long long>(K.kmin))
        << ";\n";
      if (K.step != 1) o << "      d /= " << hex64(static_cast<unsigned long long>(K.step)) << ";\n";
      o << "      if (pass && d >= " << hex64(K.range) << ") { set_fallback(t.p.err, FR_KEY_RANGE); pass = false; }\n"
        << "      c += d * " << hex64(K.stride) << "; }\n";
    }
    o << "    gid = pass ? static_cast<unsigned>(c) : 0u; }\n";
  }
  if (mode == MODE_SMALL) {
    o << "  code = 0u;\n";
    for (int q = 0; q < s.nkeys; ++q)
      o << "  code = (code << 8) | stage[" << ts.col_off[s.keys[q].col] << "u + ri];\n";
  }
  for (int a = 0; a < s.nacc; ++a) {
    const Acc& A = s.acc[a];
    if (A.is_int) {
      o << "  { const unsigned long long x = pass ? q_u64(stage, " << off(A.f[0].x.col) << ", ri) : 0ULL;\n"
        << "    long long iv = static_cast<long long>(x); iv = iv < 0 ? -iv : iv; absmax = iv > absmax ? iv : absmax;\n"
        << "    v[" << a << "] = x; }\n";
      o << "  const double d" << a << " = 1.0;\n";
      continue;
    }
    std::string prod = A.base >= 0 ? "d" + std::to_string(A.base) : "";
    for (int i = 0; i < A.nf; ++i) {
      const Factor& f = A.f[i];
      std::string x = f.kind != FK_CONST && f.x.col >= 0 ? "q_f64(stage, " + off(f.x.col) + ", ri)" : "0.0";
      std::string y;
      if (f.kind == FK_CONST) y = dlit(f.fa + 0.0);  // k_tile: fa + 0 * 0
      else if (f.fa == 0.0 && f.fb == 1.0) y = x;
      else if (f.fb == 1.0) y = "__dadd_rn(" + dlit(f.fa) + ", " + x + ")";
      else if (f.fb == -1.0) y = "__dsub_rn(" + dlit(f.fa) + ", " + x + ")";
      else y = "__dadd_rn(" + dlit(f.fa) + ", __dmul_rn(" + dlit(f.fb) + ", " + x + "))";
      prod = prod.empty() ? y : "__dmul_rn(" + prod + ", " + y + ")";
    }
    if (prod.empty()) prod = "1.0";
    o << "  const double d" << a << " = " << prod << ";\n";
    o << "  { double g = d" << a << ";\n";
    if (A.gate_probe >= 0)
      o << "    if (!((fl" << A.gate_probe << " >> " << A.gate_bit << ") & 1u)) g = " << dlit(A.gate_else) << ";\n";
    o << "    v[" << a << "] = pass ? static_cast<unsigned long long>(__double_as_longlong(g)) : 0ULL; }\n";
  }
  o << "  (void)code; (void)gid; (void)absmax;\n  return pass;\n}\n}}  // namespace tqp::fz\n"
    << "#include \"jit_tile.cuh\"\n";
  return o.str();
}

// Build-side kernel specialised the same way (jit_build.cuh): terms,
// string terms, LIKE flags and child probes with their constants folded.
// String predicates keep eval_str's semantics: a START/EXACT pattern or an
// equality literal without zero bytes compares the leading bytes directly
// (a zero-padded row shorter than the pattern cannot match a zero-free
// pattern); anything else calls eval_str.
// The TMA-staged build kernel (jit_build_tile.cuh) is opt-in: on B200 the
// Q3 orders build measured 144 us staged vs 148 us unstaged - the build is
// bound by its scattered inserts and dependent probes, not by reading its
// columns - so the simpler kernel stays the default.
bool build_tile_wanted(long long rows) {
  const char* e = std::getenv("TQP_BUILD_TILE");
  (void)rows;
  return e && (e[0] == '1' || e[0] == 'y');
}
// staged build shape: consumer warps and rows per tile (TQP_BUILD_TILE_CW /
// TQP_BUILD_TILE_ROWS tuning knobs; rows a multiple of 32 x warps)
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
int build_tile_cw() {
  static const int v = [] { const int x = env_int("TQP_BUILD_TILE_CW", 16); return x >= 4 && x <= 31 ? x : 16; }();
  return v;
}
int build_tile_rows() {
  static const int v = [] {
    const int x = env_int("TQP_BUILD_TILE_ROWS", 2048);
    return x >= 32 * build_tile_cw() && x <= 8192 && x % (32 * build_tile_cw()) == 0 ? x : 32 * build_tile_cw() * 4;
  }();
  return v;
}

int jit_build_rows() {
  static const int r = [] {
    const char* e = std::getenv("TQP_BUILD_ROWS");  // tuning knob: rows per thread of q_build
    // Q3 orders build SF10: 108 us at 2, 115 at 4, 150 at 8 with a table
    // entry per row; with the row in the group record: 89 us at 2, 81 at 4
    const int v = e ? std::atoi(e) : 4;
    return v == 1 || v == 2 || v == 4 || v == 8 ? v : 2;
  }();
  return r;
}

std::string str_pred(const StrTerm& t, const std::string& sref, const std::string& row) {
  bool zero_free = true;
  for (int i = 0; i < t.litlen; ++i) zero_free = zero_free && t.lit[i] != 0;
  const std::string p = "(" + sref + ".ptr + " + row + " * " + std::to_string(t.width) + "LL)";
  // compares joined with `&` (no short circuit): every load of the row is
  // independent and in flight at once (the row is in bounds). With an even
  // row width every row starts 2-byte aligned (columns are 256-byte
  // aligned), so byte pairs load as one 16-bit word
  const bool even = t.width % 2 == 0;
  auto byte_at = [&](int i) { return i < t.litlen ? static_cast<unsigned>(t.lit[i]) : 0u; };
  auto bytes_eq = [&](int n, auto&& want) {
    std::string e = "true";
    int i = 0;
    if (even)
      for (; i + 1 < n; i += 2)
        e += " & (__ldg(reinterpret_cast<const unsigned short*>(" + p + " + " + std::to_string(i) + ")) == " +
             std::to_string(want(i) | (want(i + 1) << 8)) + "u)";
    for (; i < n; ++i) e += " & (__ldg(" + p + " + " + std::to_string(i) + ") == " + std::to_string(want(i)) + "u)";
    return e;
  };
  auto prefix_eq = [&](int n) { return bytes_eq(n, byte_at); };
  if (t.is_like && zero_free && t.litlen <= t.width) {
    if (t.anchor == TQP_START) return "(" + prefix_eq(t.litlen) + ")";
    if (t.anchor == TQP_EXACT) {
      std::string e = prefix_eq(t.litlen);
      if (t.litlen < t.width) e += " & (__ldg(" + p + " + " + std::to_string(t.litlen) + ") == 0u)";
      return "(" + e + ")";
    }
  }
  if (!t.is_like && t.op == TQP_EQ && t.litlen <= t.width) {
    // zero-extended equality over max(width, litlen) = width bytes
    return "(" + bytes_eq(t.width, byte_at) + ")";
  }
  return "eval_str(" + sref + ", " + row + ")";
}

// staged: the TMA-staged skeleton (jit_build_tile.cuh); key / term / probe-key
// columns are read from the shared-memory tile at byte offsets `off`
// (indexed key, terms..., probe keys...), string columns from global memory.
std::string gen_build(const BuildSpec& b, bool staged = false,
                      const std::vector<int>& off = {}, int cw = 16, int tile_rows = 2048) {
  std::ostringstream o;
  auto ld = [&](const Operand& x, const std::string& ptr, const std::string& row) {
    if (x.type == OT_U8) return "static_cast<unsigned long long>(__ldg(static_cast<const uint8_t*>(" + ptr + ") + " + row + "))";
    return "static_cast<unsigned long long>(__ldg(static_cast<const unsigned long long*>(" + ptr + ") + " + row + "))";
  };
  auto lds = [&](const Operand& x, int byte_off) {
    if (x.type == OT_U8) return "static_cast<unsigned long long>(stage[" + std::to_string(byte_off) + "u + ri[j]])";
    return "*reinterpret_cast<const unsigned long long*>(stage + " + std::to_string(byte_off) + "u + ri[j] * 8)";
  };
  static const char* ops[] = {"==", "!=", "<", "<=", ">", ">="};
  o << "#include \"fz_layout.cuh\"\n#define B_ROWS " << (staged ? tile_rows / (cw * 32) : jit_build_rows())
    << "\n#define B_ASSIGN " << (b.assign_groups ? 1 : 0) << "\n#define B_ZREC " << b.zrec_words
    << "\n#define B_UNIQUE " << (b.unique ? 1 : 0) << "\n#define B_ROWREC " << (b.row_rec ? 1 : 0) << "\n";
  if (staged) o << "#define QB_CW " << cw << "\n#define QB_ROWS " << tile_rows << "\n";
  o << "namespace tqp { namespace fz {\n";
  if (staged) {
    o << "__device__ __forceinline__ void qb_rows(const TileSpec& t, const BuildSpec& s, const unsigned char* __restrict__ stage,\n"
      << "    int ct, long long row0, bool* pass, long long* key, unsigned* flags) {\n"
      << "  long long r[B_ROWS];\n  int ri[B_ROWS];\n"
      << "#pragma unroll\n  for (int j = 0; j < B_ROWS; ++j) { ri[j] = j * " << cw * 32
      << " + ct; r[j] = row0 + ri[j]; pass[j] = r[j] < s.n; flags[j] = 0u; }\n";
  } else {
    o << "__device__ __forceinline__ void b_rows(const BuildSpec& s, long long r0, int stride, bool* pass, long long* key,\n"
      << "                                       unsigned* flags) {\n"
      << "  long long r[B_ROWS];\n"
      << "#pragma unroll\n  for (int j = 0; j < B_ROWS; ++j) { r[j] = r0 + j * stride; pass[j] = r[j] < s.n; flags[j] = 0u; }\n";
  }
  // every independent column load first
  o << "  unsigned long long kv[B_ROWS]";
  for (int t = 0; t < b.nterms; ++t) o << ", tv" << t << "[B_ROWS]";
  for (int p = 0; p < b.nprobes; ++p) o << ", pv" << p << "[B_ROWS]";
  o << ";\n#pragma unroll\n  for (int j = 0; j < B_ROWS; ++j) {\n"
    << "    const long long rr = pass[j] ? r[j] : 0;\n    (void)rr;\n";
  int oi = 0;
  o << "    kv[j] = " << (staged ? lds(b.key, off.at(oi++)) : ld(b.key, "s.key.ptr", "rr")) << ";\n";
  for (int t = 0; t < b.nterms; ++t)
    if (b.terms[t].kind == TK_INT || b.terms[t].kind == TK_F64)
      o << "    tv" << t << "[j] = "
        << (staged ? lds(b.terms[t].x, off.at(oi++)) : ld(b.terms[t].x, "s.terms[" + std::to_string(t) + "].x.ptr", "rr"))
        << ";\n";
  for (int p = 0; p < b.nprobes; ++p)
    o << "    pv" << p << "[j] = "
      << (staged ? lds(b.probes[p].key, off.at(oi++)) : ld(b.probes[p].key, "s.probes[" + std::to_string(p) + "].key.ptr", "rr"))
      << ";\n";
  // phase by phase over all B_ROWS rows, so the rows' dependent probe loads
  // (presence word, then entry) are in flight together; the empty asm keeps
  // the compiler from sinking the column loads to their first use
  o << "  }\n  asm volatile(\"\" ::: \"memory\");\n"
    << "#pragma unroll\n  for (int j = 0; j < B_ROWS; ++j) {\n    bool ok = pass[j];\n    key[j] = static_cast<long long>(kv[j]);\n";
  for (int t = 0; t < b.nterms; ++t) {
    const Term& T = b.terms[t];
    const int op = T.op < 0 || T.op > 5 ? 5 : T.op;
    switch (T.kind) {
      case TK_INT:
        o << "    ok = ok && (static_cast<long long>(tv" << t << "[j]) " << ops[op] << " " << T.ik << "LL);\n";
        break;
      case TK_F64:
        o << "    ok = ok && (__longlong_as_double(static_cast<long long>(tv" << t << "[j])) " << ops[op] << " " << dlit(T.fk)
          << ");\n";
        break;
      case TK_TRUE: break;
      default: o << "    ok = false;\n"; break;
    }
  }
  for (int t = 0; t < b.nstr; ++t)
    o << "    ok = ok && " << str_pred(b.str[t], "s.str[" + std::to_string(t) + "]", "r[j]") << ";\n";
  o << "    pass[j] = ok;\n  }\n";
  for (int p = 0; p < b.nprobes; ++p) {
    const std::string pr = "s.probes[" + std::to_string(p) + "]";
    o << "  {\n    long long idx[B_ROWS];\n    bool in[B_ROWS];\n"
      << "#pragma unroll\n    for (int j = 0; j < B_ROWS; ++j) {\n"
      << "      idx[j] = static_cast<long long>(pv" << p << "[j]) - " << pr << ".kmin;\n"
      << "      in[j] = pass[j] && static_cast<unsigned long long>(idx[j]) < static_cast<unsigned long long>(" << pr
      << ".range);\n      if (!in[j]) idx[j] = 0;\n    }\n";
    // a child probe only asks whether the key was inserted: the presence bit
    // (filled by every build) answers it without touching the table
    o << "    unsigned w[B_ROWS];\n"
      << "#pragma unroll\n    for (int j = 0; j < B_ROWS; ++j) w[j] = __ldg(" << pr << ".bitmap + (idx[j] >> 5));\n"
      << "#pragma unroll\n    for (int j = 0; j < B_ROWS; ++j) pass[j] = in[j] && ((w[j] >> (idx[j] & 31)) & 1u);\n  }\n";
  }
  if (b.nflags) {
    o << "#pragma unroll\n  for (int j = 0; j < B_ROWS; ++j) {\n";
    for (int f = 0; f < b.nflags; ++f)
      o << "    if (pass[j] && " << str_pred(b.flags[f], "s.flags[" + std::to_string(f) + "]", "r[j]") << ") flags[j] |= "
        << (1u << f) << "u;\n";
    o << "  }\n";
  }
  o << "}\n}}  // namespace tqp::fz\n#include \"" << (staged ? "jit_build_tile.cuh" : "jit_build.cuh") << "\"\n";
  return o.str();
}

// Memo of the last kernel generated per call site of a fused unit. The
// generators are pure functions of their arguments, so byte-identical
// arguments (the same query over the same tables: pointers, ranges and
// constants all equal) reuse the kernel without generating its source
// again; any difference - or a padding byte that differs - regenerates.
struct JitMemo {
  std::mutex mu;
  struct Hit {
    std::string key;  // argument bytes
    const void* fn;
    long long epoch;  // jit_epoch() when stored: an unloaded library invalidates it
  };
  std::map<int, Hit> last;  // site -> last kernel
  template <typename Make>
  const void* get(int site, const std::string& key, Make&& make) {
    std::lock_guard<std::mutex> l(mu);
    auto it = last.find(site);
    if (it != last.end() && it->second.key == key && it->second.epoch == jit_epoch()) return it->second.fn;
    const long long e = jit_epoch();
    const void* fn = make();
    last[site] = {key, fn, e == jit_epoch() ? e : -1};
    return fn;
  }
};
template <typename T>
void append_bytes(std::string& k, const T& v) {
  k.append(reinterpret_cast<const char*>(&v), sizeof(T));
}
// re-creates a default-initialised spec over zeroed storage, so the padding
// between its members is zero and stays zero (member assignments do not
// touch it): byte-identical specs then compare equal
template <typename T>
void zero_padding(T& v) {
  static_assert(std::is_trivially_copyable_v<T> && std::is_trivially_destructible_v<T>, "plain spec structs only");
  std::memset(static_cast<void*>(&v), 0, sizeof(T));
  ::new (static_cast<void*>(&v)) T();
}

// memo keys: the generators' argument bytes without the per-execution
// buffers (partials, group records, build tables, presence bitmaps, error
// words), which the generated code only reaches through the kernel
// parameter, never as literals
std::string tile_key(TileSpec t) {
  t.p.part = nullptr;
  t.p.gacc = t.p.gcnt = nullptr;
  t.p.touched = nullptr;
  t.p.err = nullptr;
  for (auto& pr : t.p.probes) {
    pr.table = nullptr;
    pr.bitmap = nullptr;
    pr.rowrec = nullptr;
  }
  std::string k;
  append_bytes(k, t);
  return k;
}
std::string build_key(BuildSpec b) {
  b.table = nullptr;
  b.bitmap = nullptr;
  b.zrec = nullptr;
  b.err = nullptr;
  for (auto& pr : b.probes) {
    pr.table = nullptr;
    pr.bitmap = nullptr;
    pr.rowrec = nullptr;
  }
  std::string k;
  append_bytes(k, b);
  return k;
}

// min / max (and, for Date keys, day alignment) of int64 key columns, cached
// with the column (input columns are immutable): one launch per missing
// column and one host round trip for all of them
void ensure_key_info(Ctx& c, const std::vector<std::pair<const Column*, long long>>& cols, const std::vector<bool>& day) {
  std::vector<size_t> todo;
  for (size_t i = 0; i < cols.size(); ++i) {
    std::lock_guard<std::mutex> lk(cols[i].first->range->mu);
    const KeyRange& r = *cols[i].first->range;
    if (!r.ready || (day[i] && r.day < 0)) todo.push_back(i);
  }
  if (todo.empty()) return;
  std::vector<long long> init(3 * todo.size());
  for (size_t j = 0; j < todo.size(); ++j) {
    init[3 * j] = 0x7fffffffffffffffLL;
    init[3 * j + 1] = static_cast<long long>(0x8000000000000000ULL);
    init[3 * j + 2] = 0;
  }
  auto buf = c.alloc_bytes(sizeof(long long) * init.size());
  TQP_CUDA(cudaMemcpyAsync(buf->ptr, init.data(), sizeof(long long) * init.size(), cudaMemcpyHostToDevice, c.stream));
  for (size_t j = 0; j < todo.size(); ++j) {
    const auto& [col, rows] = cols[todo[j]];
    long long* out = static_cast<long long*>(buf->ptr) + 3 * j;
    if (rows <= 0) continue;
    if (day[todo[j]])
      k_minmax<true><<<c.grid_for(rows, 256, 8, 16), 256, 0, c.stream>>>(col->t.ptr<long long>(), rows, out);
    else
      k_minmax<false><<<c.grid_for(rows, 256, 8, 16), 256, 0, c.stream>>>(col->t.ptr<long long>(), rows, out);
    c.count_launch();
  }
  std::vector<long long> got(init.size());
  TQP_CUDA(cudaMemcpyAsync(got.data(), buf->ptr, sizeof(long long) * got.size(), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  for (size_t j = 0; j < todo.size(); ++j) {
    KeyRange& r = *cols[todo[j]].first->range;
    std::lock_guard<std::mutex> lk(r.mu);
    r.mn = got[3 * j];
    r.mx = got[3 * j + 1];
    r.ready = true;
    if (day[todo[j]]) r.day = got[3 * j + 2] ? 0 : 1;
  }
}

__global__ void k_fill_u64(unsigned long long* __restrict__ p, long long n, unsigned long long v) {
  for (long long i = gtid(); i < n; i += gstride()) p[i] = v;
}
void fill_u64(Ctx& c, unsigned long long* p, long long n, unsigned long long v) {
  if (n <= 0) return;
  k_fill_u64<<<c.grid_for(n, 256), 256, 0, c.stream>>>(p, n, v);
  c.count_launch();
}

__global__ void k_dict_insert(const long long* __restrict__ vals, long long d, long long* __restrict__ hk,
                              unsigned* __restrict__ hr, unsigned long long mask, long long empty) {
  for (long long i = gtid(); i < d; i += gstride()) {
    const long long v = vals[i];
    unsigned long long h = static_cast<unsigned long long>(v) * 0x9E3779B97F4A7C15ULL;
    unsigned long long sl = (h ^ (h >> 31)) & mask;
    while (atomicCAS(reinterpret_cast<unsigned long long*>(hk) + sl, static_cast<unsigned long long>(empty),
                     static_cast<unsigned long long>(v)) != static_cast<unsigned long long>(empty))
      sl = (sl + 1) & mask;
    hr[sl] = static_cast<unsigned>(i);
  }
}

// the column's KeyDict (distinct values by a device sort, then the value ->
// rank map), built once and kept with the column; false: not buildable
// (the column holds INT64_MIN, or more than 2^32 distinct values)
__global__ void k_pack_str8(const uint8_t* __restrict__ p, long long n, int w, long long* __restrict__ out) {
  for (long long i = gtid(); i < n; i += gstride()) {
    unsigned long long d = 0;
    for (int j = 0; j < w; ++j) d = (d << 8) | p[i * w + j];
    out[i] = static_cast<long long>(d);
  }
}

bool ensure_dict(Ctx& c, const Column* col, long long rows, long long mn) {
  KeyDict& D = *col->dict;
  std::lock_guard<std::mutex> lk(D.mu);
  if (D.ready) return true;
  Tensor t = col->t;
  t.rows = rows;
  if (t.dtype == TQP_STR8) {  // rows of <= 7 bytes, packed big-endian (>= 0)
    if (t.cols > 7) return false;
    Tensor packed = c.alloc(TQP_I64, rows, 1);
    if (rows) {
      k_pack_str8<<<c.grid_for(rows, 256), 256, 0, c.stream>>>(t.ptr<uint8_t>(), rows, static_cast<int>(t.cols),
                                                              packed.ptr<long long>());
      c.count_launch();
    }
    t = packed;
    mn = 0;
  }
  if (mn == static_cast<long long>(0x8000000000000000ULL)) return false;
  Tensor order = k::argsort_stable(c, t);
  Tensor sorted = k::gather(c, t, order);
  Tensor distinct = k::compact(c, sorted, k::segment_starts(c, sorted));
  const long long d = distinct.rows;
  if (d >= (1LL << 32)) return false;
  unsigned long long cap = 1024;
  while (cap < 2ULL * static_cast<unsigned long long>(d)) cap <<= 1;
  D.hkeys = c.alloc_bytes(sizeof(long long) * cap);
  D.hranks = c.alloc_bytes(sizeof(unsigned) * cap);
  fill_u64(c, static_cast<unsigned long long*>(D.hkeys->ptr), static_cast<long long>(cap), static_cast<unsigned long long>(mn - 1));
  if (d) {
    k_dict_insert<<<c.grid_for(d, 256), 256, 0, c.stream>>>(distinct.ptr<long long>(), d, static_cast<long long*>(D.hkeys->ptr),
                                                            static_cast<unsigned*>(D.hranks->ptr), cap - 1, mn - 1);
    c.count_launch();
  }
  D.vals = distinct;
  D.d = d;
  D.mask = cap - 1;
  D.empty = mn - 1;
  D.ready = true;
  return true;
}

// ---- sharded build sides ---------------------------------------------------------
// per-flag bitmaps of a local build (flag f of slot i where present)
__global__ void k_flag_bits(const unsigned long long* __restrict__ table, const unsigned* __restrict__ present,
                            long long range, int nflags, unsigned* __restrict__ out) {
  const long long nw = (range + 31) / 32;
  for (long long w = gtid(); w < nw; w += gstride()) {
    const unsigned p = present[w];
    unsigned f[kMaxFlags] = {0, 0, 0, 0, 0, 0, 0};
    for (unsigned m = p; m; m &= m - 1) {
      const int b = __ffs(m) - 1;
      const unsigned fl = static_cast<unsigned>(table[w * 32 + b] >> 57);
      for (int i = 0; i < nflags; ++i) f[i] |= ((fl >> i) & 1u) << b;
    }
    for (int i = 0; i < nflags; ++i) out[i * nw + w] = f[i];
  }
}

// all-gathered [presence | flag bitmaps] of every rank -> the merged presence
// bitmap and table entries (1 | flags << 57 where present, 0 elsewhere); a
// key present on two ranks is a repeated build key (err FR_DUP_KEY)
__global__ void k_merge_build_bits(const unsigned* __restrict__ all, int nranks, long long nw, int nflags, long long range,
                                   unsigned* __restrict__ present, unsigned long long* __restrict__ table, long long* err) {
  const long long per = nw * (1 + nflags);
  for (long long w = gtid(); w < nw; w += gstride()) {
    unsigned orp = 0, f[kMaxFlags] = {0, 0, 0, 0, 0, 0, 0};
    int pops = 0;
    for (int r = 0; r < nranks; ++r) {
      const unsigned pr = all[r * per + w];
      orp |= pr;
      pops += __popc(pr);
      for (int i = 0; i < nflags; ++i) f[i] |= all[r * per + (1 + i) * nw + w];
    }
    if (pops != __popc(orp)) set_fallback(err, FR_DUP_KEY);
    present[w] = orp;
    for (int b = 0; b < 32; ++b) {
      const long long slot = w * 32 + b;
      if (slot >= range) break;
      unsigned long long e = 0;
      if ((orp >> b) & 1u) {
        e = 1ULL;
        for (int i = 0; i < nflags; ++i) e |= static_cast<unsigned long long>((f[i] >> b) & 1u) << (57 + i);
      }
      table[slot] = e;
    }
  }
}

__global__ void k_range_mask(const long long* __restrict__ k, long long n, long long lo, long long hi,
                             uint8_t* __restrict__ out) {
  for (long long i = gtid(); i < n; i += gstride()) out[i] = k[i] >= lo && k[i] <= hi;
}

// Re-aligns a row-shard table to the fact shards: every row goes to each rank
// whose fact shard's probe-key range [lo_r, hi_r] holds its key (a row whose
// key no fact row can match goes nowhere); the received rows, in source-rank
// order, make this rank's copy, co-partitioned with its fact rows.
std::shared_ptr<Table> shuffle_table(Ctx& c, Comm& comm, const Table& t, const std::string& key_col,
                                     const std::vector<long long>& lo, const std::vector<long long>& hi) {
  const int G = comm.size;
  const Column* kc = t.find(key_col);
  if (!kc || kc->t.dtype != TQP_I64) throw Error(TQP_ERR_EXEC, "shuffle: key column " + key_col + " is not int64");
  std::vector<Tensor> idx(G);
  std::vector<long long> cnt(G, 0);
  for (int r = 0; r < G; ++r) {
    Tensor mask = c.alloc(TQP_BOOL, t.rows, 1);
    if (t.rows) {
      k_range_mask<<<c.grid_for(t.rows, 256), 256, 0, c.stream>>>(kc->t.ptr<long long>(), t.rows, lo[r], hi[r],
                                                                   mask.ptr<uint8_t>());
      c.count_launch();
    }
    idx[r] = k::compact(c, k::iota(c, t.rows), mask);
    cnt[r] = idx[r].rows;
  }
  const std::vector<long long> m = allgather_host(c, comm, cnt);  // m[src * G + dst]
  long long total = 0;
  for (int r = 0; r < G; ++r) total += m[r * G + comm.rank];
  auto out = std::make_shared<Table>();
  out->rows = total;
  for (const Column& col : t.cols) {
    std::vector<Tensor> parts(G);
    std::vector<const void*> send(G);
    std::vector<size_t> sb(G), rb(G);
    std::vector<void*> recv(G);
    const size_t rowb = col.t.elem_size() * static_cast<size_t>(col.t.cols);
    Column nc;
    nc.name = col.name;
    nc.type = col.type;
    nc.t = c.alloc(col.t.dtype, total, col.t.cols);
    long long off = 0;
    for (int r = 0; r < G; ++r) {
      parts[r] = k::gather(c, col.t, idx[r]);
      send[r] = parts[r].data();
      sb[r] = rowb * static_cast<size_t>(cnt[r]);
      recv[r] = static_cast<char*>(nc.t.data()) + rowb * static_cast<size_t>(off);
      rb[r] = rowb * static_cast<size_t>(m[r * G + comm.rank]);
      off += m[r * G + comm.rank];
    }
    comm.alltoallv(c, send, sb, recv, rb);
    c.sync();  // the gathered parts stay alive until the copies are done
    out->cols.push_back(std::move(nc));
  }
  return out;
}

// MODE_HASH table shape: shared-memory records per CTA when the whole code
// range fits kHashPrivBytes, a direct-address global table (slot = code)
// while the range is at most 4 slots per fact row (and <= 2^26), otherwise
// open addressing at load <= 1/2
// STR8 key widths of a MODE_HASH unit, 8 bits each (partial header word 7)
unsigned long long hash_key_widths(const ProbeSpec& ps) {
  unsigned long long w = 0;
  for (int i = 0; i < ps.nhkeys; ++i) w |= static_cast<unsigned long long>(ps.hkeys[i].width & 0xff) << (8 * i);
  return w;
}

GroupSpec hash_group_spec(const ProbeSpec& ps, const FinalSpec& fs, const unsigned* present,
                          const std::vector<const long long*>& dict_vals) {
  GroupSpec gs;
  gs.f = fs;
  gs.gacc = ps.gacc;
  gs.gcnt = ps.gcnt;
  gs.group_table = nullptr;
  gs.cnt_stride = ps.gstride;
  gs.acc_stride = ps.gstride;
  gs.present = present;
  gs.acc_words = kLimbWords;
  gs.nkeyc = ps.nhkeys;
  gs.nsort = 0;
  gs.codes = ps.htag;
  gs.direct_codes = ps.htag ? 0 : 1;
  gs.cnt_packed = 1;
  gs.absmax = ps.absmax_out;
  gs.flag_word = ps.hflags;
  gs.qfrac = ps.qfrac;
  gs.limb2 = ps.hlimbs == 2 ? 1 : 0;
  for (int a = 0; a < ps.nacc && a < kMaxAcc; ++a) {
    gs.acc_off[a] = ps.hoff[a];
    if (gs.limb2 && ps.acc[a].is_int) gs.acc_int1 |= 1u << a;
  }
  gs.fmax = ps.fmax_out;
  for (int i = 0; i < ps.nhkeys; ++i) {
    gs.key_cols[i] = nullptr;
    gs.kmin[i] = ps.hkeys[i].kmin;
    gs.kstep[i] = ps.hkeys[i].step;
    gs.krange[i] = ps.hkeys[i].range;
    gs.kstride[i] = ps.hkeys[i].stride;
    gs.key_w[i] = ps.hkeys[i].width;
    gs.dvals[i] = dict_vals[i];
  }
  return gs;
}

// a fused unit that cannot take this data (host-side contract check): the
// executor runs its steps per instruction; TQP_DEBUG_FALLBACK names the check
bool nofuse(int line) {
  if (std::getenv("TQP_DEBUG_FALLBACK")) std::fprintf(stderr, "tqp: fused unit not run (fused.cu:%d)\n", line);
  return false;
}

constexpr size_t kHashPrivBytes = 48 * 1024;
constexpr unsigned long long kHashDirectMax = 1ULL << 26;
constexpr size_t kHashMaxBytes = 24ULL << 30;

// re-run options of a fused unit (each set by the check that failed)
struct RunOpts {
  bool narrow = false;    // the 8-slot small-group kernel only (after a 4-slot overflow)
  bool weighted = false;  // repeated build keys: builds sum row weights, the scan counts by multiplicity
  bool fullsort = false;  // top-k ties: every group, then the reference's sort + limit
  bool special = false;   // NaN / Inf hash-group values flagged per group
  int qfrac = 64;         // hash-group fixed-point fraction bits
  int hlimbs = 2;         // hash-group sums in 2 limbs, or 3
  bool shuffled = false;  // sharded run: row-shard build sides already realigned to the fact shards
  RunOpts with_narrow(bool v) const {
    RunOpts r = *this;
    r.narrow = v;
    return r;
  }
};

struct Runner {
  PipeDesc P;
  std::shared_ptr<JitMemo> memo = std::make_shared<JitMemo>();
  // MODE_SMALL units with hashable keys: the MODE_HASH unit a CTA overflow
  // (more distinct codes than slots) reruns as, instead of the exact path
  std::shared_ptr<const Runner> alt;

  bool operator()(Ctx& c, std::vector<std::optional<Tensor>>& slots, const TableSet& tables, UnitPending* pend) const {
    return run(c, &slots, tables, nullptr, RunOpts{}, pend);
  }

  // po != nullptr: phase 1 of a sharded run (partial state into *po, no slots)
  // narrow: the 8-slot small-group kernel only (after a 4-slot overflow)
  // weighted: re-run after a build met a repeated key (1:N join): builds sum
  // row weights per key and the fact scan counts rows by multiplicity
  // special: re-run after a hash-group fp64 value was NaN or +-Inf: those are
  // flagged per group (IEEE sum semantics) instead of summed in fixed point
  // hlimbs: hash-group sums in 2 limbs (re-run with 3 when a group's range
  // check fails)
  bool run(Ctx& c, std::vector<std::optional<Tensor>>* slots, const TableSet& tables, Partial* po,
           RunOpts o = RunOpts{}, UnitPending* pend = nullptr) const {
    const bool narrow = o.narrow, weighted = o.weighted, fullsort = o.fullsort, special = o.special;
    const int qfrac = o.qfrac, hlimbs = o.hlimbs;
    // sharded phase 1 (execute_sharded): the communicator and table layout
    const ShardEnv* env = po ? po->env : nullptr;
    Comm* comm = env ? env->comm : nullptr;
    auto is_rows = [&](const std::string& t) { return comm && env->kind_of(t) == SHARD_ROWS; };
    if (comm && !o.shuffled) {
      // row-shard build sides the scan reads root rows of (the group build,
      // operand / key columns) are re-aligned to the fact shards by key
      // range first; the others exchange presence / flag bitmaps below
      std::vector<std::pair<int, int>> sh;  // (build, fact probe)
      for (size_t p = 0; p < P.probes.size(); ++p) {
        const int bi = P.probes[p].build;
        bool rid = P.builds[bi].assign_groups;
        for (const auto& a : P.accs)
          for (const auto& f : a.f) rid = rid || (f.kind != FK_CONST && f.x.probe == static_cast<int>(p));
        for (const auto& k : P.hkeys) rid = rid || k.probe == static_cast<int>(p);
        if (rid && is_rows(P.builds[bi].table)) sh.push_back({bi, static_cast<int>(p)});
      }
      if (!sh.empty()) {
        const Table* fact = bind_table(tables, P.fact_table);
        if (!fact) return nofuse(__LINE__);
        std::vector<std::pair<const Column*, long long>> fcols;
        for (auto [bi, p] : sh) {
          const Column* fc = fact->find(P.probes[p].fact_column);
          if (!fc || fc->t.dtype != TQP_I64) return nofuse(__LINE__);
          fcols.push_back({fc, fact->rows});
        }
        ensure_key_info(c, fcols, std::vector<bool>(fcols.size(), false));
        std::vector<long long> mine;
        for (auto& [fc, rows] : fcols) {
          mine.push_back(rows ? fc->range->mn : 1);
          mine.push_back(rows ? fc->range->mx : 0);  // empty shard: an empty range
        }
        const std::vector<long long> all = allgather_host(c, *comm, mine);
        TableSet t2 = tables;
        ShardEnv env2 = *env;
        std::vector<std::shared_ptr<Table>> hold;
        for (size_t i = 0; i < sh.size(); ++i) {
          const BuildDesc& B = P.builds[sh[i].first];
          std::vector<long long> lo(comm->size), hi(comm->size);
          for (int r = 0; r < comm->size; ++r) {
            lo[r] = all[r * mine.size() + 2 * i];
            hi[r] = all[r * mine.size() + 2 * i + 1];
          }
          const Table* bt = bind_table(tables, B.table);
          if (!bt) return nofuse(__LINE__);
          hold.push_back(shuffle_table(c, *comm, *bt, B.key_column, lo, hi));
          env->shuffled_tables += 1;
          for (auto& [name, tp] : t2)
            if (iequals(name, B.table)) tp = hold.back().get();
          std::string lower = B.table;
          for (auto& ch : lower) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
          env2.kinds[lower] = SHARD_COPARTITIONED;
        }
        const ShardEnv* saved = po->env;
        po->env = &env2;
        RunOpts r = o;
        r.shuffled = true;
        const bool ok = run(c, slots, t2, po, r, pend);
        po->env = saved;
        return ok;
      }
    }
    // build sides, children first (builds[] is in post-order by construction)
    // err[0]: precondition flag; err[2]: result rows counted on the device
    HostProf hp;
    std::vector<Probe> built(P.builds.size());
    std::vector<std::shared_ptr<DevBuf>> keep;
    std::vector<long long> build_range(P.builds.size(), 0);
    const unsigned long long* group_table = nullptr;
    bool row_rec_grp = false;
    const unsigned* group_present = nullptr;
    unsigned long long* grec_p = nullptr;
    int grec_words = 0;
    const int nacc_all = static_cast<int>(P.accs.size());
    // key ranges of every build side: cached with the column after the first
    // query that keys on it; otherwise one launch per column and one host
    // round trip for all of them
    const size_t nb = P.builds.size();
    std::vector<long long> mm(2 * std::max<size_t>(1, nb));
    std::vector<size_t> todo;
    for (size_t bi = 0; bi < nb; ++bi) {
      const BuildDesc& B = P.builds[bi];
      const Table* tab = bind_table(tables, B.table);
      const Column* key = tab ? tab->find(B.key_column) : nullptr;
      if (!key || key->t.dtype != TQP_I64) return nofuse(__LINE__);
      std::lock_guard<std::mutex> lk(key->range->mu);
      if (key->range->ready) {
        mm[2 * bi] = key->range->mn;
        mm[2 * bi + 1] = key->range->mx;
      } else {
        mm[2 * bi] = 0x7fffffffffffffffLL;
        mm[2 * bi + 1] = static_cast<long long>(0x8000000000000000ULL);
        todo.push_back(bi);
      }
    }
    std::shared_ptr<DevBuf> mmb;
    if (!todo.empty()) {
      mmb = c.alloc_bytes(sizeof(long long) * 2 * nb);
      const bool pinned = nb <= static_cast<size_t>(Ctx::kPinnedMinMaxPairs);
      TQP_CUDA(cudaMemcpyAsync(mmb->ptr, pinned ? c.h_err + Ctx::kPinnedMinMax : mm.data(), sizeof(long long) * 2 * nb,
                               cudaMemcpyHostToDevice, c.stream));
      for (size_t bi : todo) {
        const BuildDesc& B = P.builds[bi];
        const Table* tab = bind_table(tables, B.table);
        const Column* key = tab->find(B.key_column);
        if (tab->rows) {
          k_minmax<false><<<c.grid_for(tab->rows, 256, 8, 16), 256, 0, c.stream>>>(
              key->t.ptr<long long>(), tab->rows, static_cast<long long*>(mmb->ptr) + 2 * bi);
          c.count_launch();
        }
      }
      std::vector<long long> fresh(2 * nb);
      long long* rd = pinned ? c.h_err + Ctx::kPinnedRead : fresh.data();
      TQP_CUDA(cudaMemcpyAsync(rd, mmb->ptr, sizeof(long long) * 2 * nb, cudaMemcpyDeviceToHost, c.stream));
      c.sync();
      for (size_t bi : todo) {
        mm[2 * bi] = rd[2 * bi];
        mm[2 * bi + 1] = rd[2 * bi + 1];
        const Column* key = bind_table(tables, P.builds[bi].table)->find(P.builds[bi].key_column);
        std::lock_guard<std::mutex> lk(key->range->mu);
        key->range->mn = mm[2 * bi];
        key->range->mx = mm[2 * bi + 1];
        key->range->ready = true;
      }
    }
    hp.mark("ranges");
    // row-shard build sides: the global key range and row count (one
    // all-gather for all of them; every rank then makes the same table shape)
    std::vector<long long> gn(nb, -1);
    bool exchange = false;
    if (comm) {
      std::vector<long long> mine;
      for (size_t bi = 0; bi < nb; ++bi) {
        if (!is_rows(P.builds[bi].table)) continue;
        if (P.builds[bi].assign_groups) return nofuse(__LINE__);  // (re-aligned above)
        mine.push_back(bind_table(tables, P.builds[bi].table)->rows);
        mine.push_back(mm[2 * bi]);
        mine.push_back(mm[2 * bi + 1]);
      }
      if (!mine.empty()) {
        exchange = true;
        const std::vector<long long> all = allgather_host(c, *comm, mine);
        size_t j = 0;
        for (size_t bi = 0; bi < nb; ++bi) {
          if (!is_rows(P.builds[bi].table)) continue;
          long long n = 0, mn = 0x7fffffffffffffffLL, mx = static_cast<long long>(0x8000000000000000ULL);
          for (int r = 0; r < comm->size; ++r) {
            const long long* v = &all[r * mine.size() + j];
            if (v[0] <= 0) continue;
            n += v[0];
            mn = std::min(mn, v[1]);
            mx = std::max(mx, v[2]);
          }
          gn[bi] = n;
          mm[2 * bi] = n ? mn : 0;
          mm[2 * bi + 1] = n ? mx : 0;
          j += 3;
        }
      }
    }
    // one zeroed arena for the unit's small state - the error words, every
    // build's presence bitmap and the touched-group bitmap - so one memset
    // replaces one per buffer (each is host time between the unit's kernels)
    // a build whose key range is too wide for direct addressing (or would
    // overflow the range arithmetic) is an open-addressing table of `cap`
    // slots; the group of a group-assigning hashed build is its slot
    std::vector<size_t> bm_off(nb, 0);
    std::vector<char> hashed(nb, 0);
    std::vector<long long> slots_of(nb, 0);  // direct: key range; hashed: capacity
    size_t arena = 256, touched_off = 0;
    bool generic_only = weighted;  // the NVRTC kernels address dense, unweighted builds only
    for (size_t bi = 0; bi < nb; ++bi) {
      const long long n = gn[bi] >= 0 ? gn[bi] : bind_table(tables, P.builds[bi].table)->rows;
      const long long mn = mm[2 * bi], mx = mm[2 * bi + 1];
      const unsigned long long span = static_cast<unsigned long long>(mx) - static_cast<unsigned long long>(mn);
      const bool wide = n && (span > static_cast<unsigned long long>(16LL * n + (1LL << 22)) || span >= (1ULL << 31));
      long long range = n ? static_cast<long long>(span) + 1 : 1;
      if (wide) {
        if (gn[bi] >= 0) return nofuse(__LINE__);  // a row-shard build side exchanges direct-address bitmaps only
        if (mn == static_cast<long long>(0x8000000000000000ULL)) return nofuse(__LINE__);  // no empty-slot marker
        if (n >= (1LL << 31)) return nofuse(__LINE__);
        long long cap = 1024;
        while (cap < 2 * n) cap <<= 1;
        hashed[bi] = 1;
        range = cap;
        generic_only = true;
      }
      slots_of[bi] = range;
      bm_off[bi] = arena;
      if (!wide) arena += (sizeof(unsigned) * static_cast<size_t>((range + 31) / 32) + 255) & ~size_t(255);
      if (P.mode == MODE_BUILDGRP && P.group_probe >= 0 && P.group_probe < static_cast<int>(P.probes.size()) &&
          P.probes[P.group_probe].build == static_cast<int>(bi)) {
        touched_off = arena;
        arena += (sizeof(unsigned) * static_cast<size_t>((range + 31) / 32 + 1) + 255) & ~size_t(255);
      }
    }
    // does a direct-addressed build's key column repeat a value? Checked once
    // per column (one bitmap pass and one host round trip for all of them)
    // and cached with its range: a build over a unique key sets its presence
    // bits fire-and-forget (presence_insert_unique) instead of checking every
    // returned word for a repeated key
    {
      std::vector<size_t> uq;
      for (size_t bi = 0; bi < nb; ++bi) {
        if (hashed[bi] || gn[bi] >= 0) continue;
        const Table* tab = bind_table(tables, P.builds[bi].table);
        if (!tab->rows) continue;
        const Column* key = tab->find(P.builds[bi].key_column);
        std::lock_guard<std::mutex> lk(key->range->mu);
        if (key->range->unique < 0) uq.push_back(bi);
      }
      if (!uq.empty()) {
        size_t bytes = 256;
        std::vector<size_t> off;
        for (size_t bi : uq) {
          off.push_back(bytes);
          bytes += (sizeof(unsigned) * static_cast<size_t>((slots_of[bi] + 31) / 32) + 255) & ~size_t(255);
        }
        if (uq.size() > 64) return nofuse(__LINE__);
        auto ub = c.alloc_bytes(bytes);
        TQP_CUDA(cudaMemsetAsync(ub->ptr, 0, bytes, c.stream));
        unsigned char* up = static_cast<unsigned char*>(ub->ptr);
        for (size_t j = 0; j < uq.size(); ++j) {
          const Table* tab = bind_table(tables, P.builds[uq[j]].table);
          const Column* key = tab->find(P.builds[uq[j]].key_column);
          k_key_unique<<<c.grid_for(tab->rows, 256, 4, 16), 256, 0, c.stream>>>(
              key->t.ptr<long long>(), tab->rows, mm[2 * uq[j]], reinterpret_cast<unsigned*>(up + off[j]),
              reinterpret_cast<int*>(up) + j);
          c.count_launch();
        }
        std::vector<int> dupf(uq.size());
        TQP_CUDA(cudaMemcpyAsync(dupf.data(), up, sizeof(int) * uq.size(), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        for (size_t j = 0; j < uq.size(); ++j) {
          const Column* key = bind_table(tables, P.builds[uq[j]].table)->find(P.builds[uq[j]].key_column);
          std::lock_guard<std::mutex> lk(key->range->mu);
          key->range->unique = dupf[j] ? 0 : 1;
        }
      }
    }
    auto err_buf = c.alloc_bytes(arena);
    TQP_CUDA(cudaMemsetAsync(err_buf->ptr, 0, arena, c.stream));
    long long* err = static_cast<long long*>(err_buf->ptr);
    unsigned char* arena_p = static_cast<unsigned char*>(err_buf->ptr);
    for (size_t bi = 0; bi < P.builds.size(); ++bi) {
      const BuildDesc& B = P.builds[bi];
      const Table* tab = bind_table(tables, B.table);
      const Column* key = tab->find(B.key_column);
      long long n = tab->rows;
      const long long range = slots_of[bi];
      BuildSpec bs;
      zero_padding(bs);  // its bytes key the kernel memo
      bs.n = n;
      bs.kmin = (n || gn[bi] > 0) ? mm[2 * bi] : 0;
      bs.range = range;
      if (!hashed[bi] && gn[bi] < 0 && n) {
        std::lock_guard<std::mutex> lk(key->range->mu);
        bs.unique = key->range->unique == 1 ? 1 : 0;
      }
      // a flagless group-assigning direct build keeps its rows in the group
      // records (BuildSpec::row_rec): no table at all
      const bool row_rec = B.assign_groups && B.flags.empty() && !hashed[bi] && gn[bi] < 0;
      auto table = c.alloc_bytes(row_rec ? 0 : sizeof(unsigned long long) * range);
      // a filtered build's table is only read where its presence bit is set
      // (probe_lookup and every generated probe check the bitmap first), so
      // only an unfiltered one, read as `entry != 0`, needs zeroed slots -
      // and not even that when its n unique keys fill all n slots of the
      // range (a repeated key leaves a slot unwritten, but it is flagged as
      // a duplicate and the unit is discarded). A hashed table's entries are
      // only read where the slot's key matched (written by the claiming row).
      if (!row_rec && !hashed[bi] && ((!build_filtered(B) && range != n) || weighted))
        TQP_CUDA(cudaMemsetAsync(table->ptr, 0, sizeof(unsigned long long) * range, c.stream));
      if (hashed[bi]) {
        auto hk = c.alloc_bytes(sizeof(long long) * range);
        keep.push_back(hk);
        fill_u64(c, static_cast<unsigned long long*>(hk->ptr), range, static_cast<unsigned long long>(bs.kmin - 1));
        bs.hkeys = static_cast<long long*>(hk->ptr);
        bs.hmask = static_cast<unsigned long long>(range - 1);
      }
      if (weighted) {
        auto mu = c.alloc_bytes(sizeof(unsigned) * range);
        keep.push_back(mu);
        TQP_CUDA(cudaMemsetAsync(mu->ptr, 0, mu->bytes, c.stream));
        bs.mult = static_cast<unsigned*>(mu->ptr);
      }
      keep.push_back(table);
      bs.table = row_rec ? nullptr : static_cast<unsigned long long*>(table->ptr);
      bs.row_rec = row_rec ? 1 : 0;
      build_range[bi] = range;
      bs.bitmap = reinterpret_cast<unsigned*>(arena_p + bm_off[bi]);
      bs.err = err;
      bool ok = true;
      bs.key = {key->t.data(), OT_I64, -1};
      for (const auto& t : B.terms) {
        Term nt;
        StrTerm st;
        bool is_str;
        if (!make_term(tables, B.table, t, &nt, &st, &is_str)) return nofuse(__LINE__);
        if (is_str) {
          if (bs.nstr >= kMaxStrTerms) return nofuse(__LINE__);
          bs.str[bs.nstr++] = st;
        } else {
          if (bs.nterms >= kMaxTerms) return nofuse(__LINE__);
          bs.terms[bs.nterms++] = nt;
        }
      }
      for (const auto& t : B.flags) {
        Term nt;
        StrTerm st;
        bool is_str;
        if (!make_term(tables, B.table, t, &nt, &st, &is_str) || !is_str) return nofuse(__LINE__);
        bs.flags[bs.nflags++] = st;
      }
      for (const auto& ch : B.children) {
        const Column* kc = tab->find(ch.fact_column);
        if (!kc || kc->t.dtype != TQP_I64) return nofuse(__LINE__);
        Probe p = built[ch.build];
        p.key = {kc->t.data(), OT_I64, -1};
        bs.probes[bs.nprobes++] = p;
      }
      if (B.assign_groups) {
        // the group is the key slot: one record per slot [count, limbs per
        // accumulator], whole 32-byte sectors, written only for inserted slots
        grec_words = (1 + kLimbWords * std::max(1, nacc_all) + 3) & ~3;
        auto grec = c.alloc_bytes(sizeof(unsigned long long) * grec_words * (range + 1));
        keep.push_back(grec);
        group_table = bs.table;  // nullptr for a row_rec build (rows in the records)
        row_rec_grp = row_rec;
        group_present = bs.bitmap;
        grec_p = static_cast<unsigned long long*>(grec->ptr);
        bs.assign_groups = 1;
        bs.zrec = grec_p;
        bs.zrec_words = grec_words;
      }
      if (!ok) return nofuse(__LINE__);
      if (n) {
        // kBuildRows rows per thread: the per-row dependent loads (term,
        // probe, insert) need many warps in flight
        const void* bk = reinterpret_cast<const void*>(&k_build);
        int rows_per_thread = kBuildRows;
        if (jit_wanted(n) && build_tile_wanted(n) && !generic_only) {
          // large build side: TMA-staged scan of its columns (jit_build_tile.cuh)
          TileSpec bt;
          bt.p.n = n;
          std::vector<int> offs;
          bool stageable = true;
          auto stage_col = [&](const Operand& o) {
            const int w = o.type == OT_U8 ? 1 : 8;
            if (!o.ptr || reinterpret_cast<uintptr_t>(o.ptr) % 16) stageable = false;
            for (int i = 0; i < bt.ncols; ++i)
              if (bt.col_ptr[i] == o.ptr) {
                offs.push_back(bt.col_off[i]);
                return;
              }
            if (bt.ncols >= kMaxCols) {
              stageable = false;
              return;
            }
            bt.col_ptr[bt.ncols] = static_cast<const unsigned char*>(o.ptr);
            bt.col_w[bt.ncols] = w;
            bt.col_off[bt.ncols] = bt.stage_bytes;
            offs.push_back(bt.stage_bytes);
            bt.stage_bytes += (build_tile_rows() * w + 127) & ~127;
            ++bt.ncols;
          };
          stage_col(bs.key);
          for (int t = 0; t < bs.nterms; ++t)
            if (bs.terms[t].kind == TK_INT || bs.terms[t].kind == TK_F64) stage_col(bs.terms[t].x);
          for (int p = 0; p < bs.nprobes; ++p) stage_col(bs.probes[p].key);
          if (stageable) {
            bt.rows = build_tile_rows();
            const void* kfn = jit_kernel(gen_build(bs, true, offs, build_tile_cw(), build_tile_rows()), "q_build_tile");
            int optin = 0;
            TQP_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device));
            cudaFuncAttributes fa{};
            TQP_CUDA(cudaFuncGetAttributes(&fa, kfn));
            const size_t budget = static_cast<size_t>(optin) - fa.sharedSizeBytes - 1024 - 256;
            bt.stages = static_cast<int>(std::min<size_t>(kMaxStages, budget / bt.stage_bytes));
            if (bt.stages >= 2) {
              const size_t smem = 256 + static_cast<size_t>(bt.stages) * bt.stage_bytes;
              cudaError_t e = c.ensure_smem(kfn, static_cast<int>(smem));
              if (e != cudaSuccess) throw Error(TQP_ERR_CUDA, std::string("cuda: ") + cudaGetErrorString(e));
              void* targs[] = {&bt, &bs};
              cudaEvent_t ev = c.kernel_begin();
              TQP_CUDA(cudaLaunchKernel(kfn, dim3(c.num_sms), dim3(build_tile_cw() * 32 + 32), targs, smem, c.stream));
              c.kernel_end("q_build_tile", ev);
              c.count_launch();
              bk = nullptr;
            }
          }
        }
        if (bk && jit_wanted(n) && !generic_only) {
          rows_per_thread = jit_build_rows();
          hp.mark("bprep");
          std::string key = build_key(bs);
          append_bytes(key, rows_per_thread);
          bk = memo->get(static_cast<int>(bi), key, [&] { return jit_kernel(gen_build(bs), "q_build"); });
          hp.mark("bjit");
        }
        if (bk) {
          void* args[] = {&bs};
          cudaEvent_t ev = c.kernel_begin();
          TQP_CUDA(cudaLaunchKernel(bk, dim3(c.grid_for(n, kThreads, rows_per_thread, 1 << 20)), dim3(kThreads), args, 0,
                                    c.stream));
          c.kernel_end(bk == reinterpret_cast<const void*>(&k_build) ? "k_build" : "q_build", ev);
          c.count_launch();
          hp.mark("blaunch");
        }
      }
      if (gn[bi] >= 0) {
        // row-shard build side: all-gather every rank's presence and flag
        // bitmaps over the global key range and merge them into this rank's
        // bitmap and table entries (the north star's "part build side
        // all-gathered": 2.5 MB of bits at SF100 instead of the table)
        const long long nw = (range + 31) / 32;
        const int nf = bs.nflags;
        auto mine = c.alloc_bytes(sizeof(unsigned) * nw * (1 + nf));
        auto all = c.alloc_bytes(sizeof(unsigned) * nw * (1 + nf) * comm->size);
        TQP_CUDA(cudaMemcpyAsync(mine->ptr, bs.bitmap, sizeof(unsigned) * nw, cudaMemcpyDeviceToDevice, c.stream));
        if (nf && nw) {
          k_flag_bits<<<c.grid_for(nw, 256), 256, 0, c.stream>>>(bs.table, bs.bitmap, range, nf,
                                                                 static_cast<unsigned*>(mine->ptr) + nw);
          c.count_launch();
        }
        comm->allgather(c, mine->ptr, all->ptr, sizeof(unsigned) * nw * (1 + nf));
        env->bitmap_merges += 1;
        env->exchange_bytes += static_cast<long long>(sizeof(unsigned) * nw * (1 + nf) * comm->size);
        if (nw) {
          k_merge_build_bits<<<c.grid_for(nw, 256), 256, 0, c.stream>>>(static_cast<const unsigned*>(all->ptr), comm->size,
                                                                        nw, nf, range, bs.bitmap, bs.table, err);
          c.count_launch();
        }
        keep.push_back(mine);
        keep.push_back(all);
      }
      Probe pr;
      pr.kmin = bs.kmin;
      pr.range = range;
      pr.table = bs.table;
      if (bs.row_rec) {
        pr.rowrec = bs.zrec;
        pr.rstride = bs.zrec_words;
      }
      pr.bitmap = hashed[bi] ? nullptr : bs.bitmap;
      pr.hkeys = bs.hkeys;
      pr.hmask = bs.hmask;
      pr.mult = bs.mult;
      built[bi] = pr;
    }
    hp.mark("builds");
    // fact probe
    const Table* fact = bind_table(tables, P.fact_table);
    if (!fact) return nofuse(__LINE__);
    ProbeSpec ps;
    zero_padding(ps);
    ps.n = fact->rows;
    ps.err = err;
    bool ok = true;
    // conjuncts on the same column merge into one lo <= x <= hi range
    std::vector<Term> raw_terms;
    for (const auto& t : P.terms) {
      Term nt;
      StrTerm st;
      bool is_str;
      if (!make_term(tables, P.fact_table, t, &nt, &st, &is_str) || is_str) return nofuse(__LINE__);
      if (nt.kind <= TK_F64 && reinterpret_cast<uintptr_t>(nt.x.ptr) % 16) return nofuse(__LINE__);
      raw_terms.push_back(nt);
    }
    std::vector<Operand> term_cols;
    if (!merge_range_terms(raw_terms, ps, term_cols)) return nofuse(__LINE__);
    for (const auto& p : P.probes) {
      Probe pr = built[p.build];
      pr.key = make_operand(tables, P, {-1, p.fact_column}, &ok);
      if (pr.key.type != OT_I64) return nofuse(__LINE__);
      ps.probes[ps.nprobes++] = pr;
    }
    for (const auto& a : P.accs) {
      Acc& d = ps.acc[ps.nacc++];
      d.is_int = a.is_int;
      d.nf = static_cast<int>(a.f.size());
      if (!a.is_int && a.f.size() > static_cast<size_t>(kFixedFactors)) return nofuse(__LINE__);
      for (size_t i = 0; i < a.f.size(); ++i) {
        if (a.f[i].kind != FK_CONST) d.f[i].x = make_operand(tables, P, a.f[i].x, &ok);
        d.f[i].kind = a.f[i].kind;
        d.f[i].k = a.f[i].k;
        const double k = a.f[i].k;
        switch (a.f[i].kind) {  // factor = fa + fb * x
          case FK_X: d.f[i].fa = 0.0; d.f[i].fb = 1.0; break;
          case FK_K_MINUS_X: d.f[i].fa = k; d.f[i].fb = -1.0; break;
          case FK_K_PLUS_X: d.f[i].fa = k; d.f[i].fb = 1.0; break;
          case FK_X_MINUS_K: d.f[i].fa = -k; d.f[i].fb = 1.0; break;
          case FK_X_PLUS_K: d.f[i].fa = k; d.f[i].fb = 1.0; break;
          case FK_X_TIMES_K: d.f[i].fa = 0.0; d.f[i].fb = k; break;
          default: d.f[i].fa = k; d.f[i].fb = 0.0; d.f[i].x = Operand{}; break;  // constant
        }
      }
      for (int i = static_cast<int>(a.f.size()); i < kFixedFactors; ++i) {
        d.f[i] = Factor{};  // 1 + 0 * 0
        d.f[i].kind = FK_CONST;
      }
      d.gate_probe = a.gate_probe;
      d.gate_bit = a.gate_bit;
      d.gate_else = a.gate_else;
    }
    for (const auto& kcol : P.key_columns) ps.keys[ps.nkeys++] = make_operand(tables, P, {-1, kcol}, &ok);
    ps.group_probe = P.mode == MODE_BUILDGRP ? P.group_probe : -1;
    // small-group keys are 1-byte strings; wider ones (or an accumulator
    // count without a small-group kernel) run as the hash-group unit
    if (P.mode == MODE_SMALL && alt && (!ok || !tile_kernel(MODE_SMALL, ps.nacc)))
      return alt->run(c, slots, tables, po, o.with_narrow(false), pend);
    if (!ok) return nofuse(__LINE__);
    // probes whose matched root row is read: with repeated build keys such a
    // probe must match exactly one row (checked per row in a weighted run)
    ps.weighted = weighted ? 1 : 0;
    ps.root_mask = 0;
    for (int a = 0; a < ps.nacc; ++a) {
      if (ps.acc[a].gate_probe >= 0) ps.root_mask |= 1u << ps.acc[a].gate_probe;
      for (int i = 0; i < ps.acc[a].nf; ++i)
        if (ps.acc[a].f[i].kind != FK_CONST && ps.acc[a].f[i].x.src >= 0) ps.root_mask |= 1u << ps.acc[a].f[i].x.src;
    }
    if (P.mode == MODE_BUILDGRP && P.group_probe >= 0) ps.root_mask |= 1u << P.group_probe;
    for (const auto& hk : P.hkeys)
      if (hk.probe >= 0) ps.root_mask |= 1u << hk.probe;
    // MODE_HASH: key digits from the key columns' ranges, the code's mixed
    // radix, and the table shape (private / direct / open addressing)
    std::shared_ptr<DevBuf> htag_buf, hrec_buf;
    std::vector<const long long*> hdict_vals(kMaxKeys, nullptr);
    unsigned long long hcap = 0;
    int hrec_words = 0;
    if (P.mode == MODE_HASH) {
      const int nk = static_cast<int>(P.hkeys.size());
      if (nk < 1 || nk > kMaxKeys) return nofuse(__LINE__);
      std::vector<const Column*> kc(nk);
      std::vector<std::pair<const Column*, long long>> icols;
      std::vector<bool> iday;
      for (int i = 0; i < nk; ++i) {
        const OperandDesc& o = P.hkeys[i];
        const std::string& tname = o.probe < 0 ? P.fact_table : P.builds[P.probes[o.probe].build].table;
        const Table* tab = bind_table(tables, tname);
        kc[i] = tab ? tab->find(o.column) : nullptr;
        if (!kc[i]) return nofuse(__LINE__);
        GKey& K = ps.hkeys[i];
        K.x.ptr = kc[i]->t.data();
        K.x.src = o.probe;
        K.x.col = -1;
        if (P.hkey_lt[i] == TQP_LT_UTF8) {
          if (kc[i]->t.dtype != TQP_STR8 || kc[i]->t.cols < 1 || kc[i]->t.cols > 7) return nofuse(__LINE__);
          K.x.type = OT_U8;
          K.width = static_cast<int>(kc[i]->t.cols);
          K.range = 1ULL << (8 * K.width);
        } else {
          if (kc[i]->t.dtype != TQP_I64 || kc[i]->t.cols != 1) return nofuse(__LINE__);
          if (reinterpret_cast<uintptr_t>(K.x.ptr) % 16) return nofuse(__LINE__);
          K.x.type = OT_I64;
          icols.push_back({kc[i], tab->rows});
          iday.push_back(P.hkey_lt[i] == TQP_LT_DATE);
        }
      }
      ensure_key_info(c, icols, iday);
      // int keys whose ranges multiply past 2^62: the widest ones take
      // dictionary digits (rank among the column's distinct values)
      std::vector<char> use_dict(nk, 0);
      {
        auto range_of = [&](int i) -> long double {
          const GKey& K = ps.hkeys[i];
          if (K.width) return use_dict[i] ? static_cast<long double>(std::max<long long>(1, kc[i]->dict->d))
                                          : static_cast<long double>(K.range);
          const KeyRange& r = *kc[i]->range;
          if (r.mn > r.mx) return 1.0L;
          if (use_dict[i]) return static_cast<long double>(std::max<long long>(1, kc[i]->dict->d));
          const long double step = (P.hkey_lt[i] == TQP_LT_DATE && r.day == 1) ? 86400000000000.0L : 1.0L;
          return (static_cast<long double>(r.mx) - static_cast<long double>(r.mn)) / step + 1.0L;
        };
        for (;;) {
          long double prod = 1.0L;
          for (int i = 0; i < nk; ++i) prod *= range_of(i);
          if (prod <= 4.0e18L) break;  // < 2^62
          int widest = -1;
          for (int i = 0; i < nk; ++i)
            if (!use_dict[i] && (widest < 0 || range_of(i) > range_of(widest))) widest = i;
          if (widest < 0) break;
          const std::string& tname = P.hkeys[widest].probe < 0 ? P.fact_table : P.builds[P.probes[P.hkeys[widest].probe].build].table;
          if (!ensure_dict(c, kc[widest], bind_table(tables, tname)->rows, ps.hkeys[widest].width ? 0 : kc[widest]->range->mn))
            return nofuse(__LINE__);
          use_dict[widest] = 1;
        }
      }
      unsigned __int128 total = 1;
      for (int i = 0; i < nk; ++i) {
        GKey& K = ps.hkeys[i];
        if (K.width) {
          if (use_dict[i]) {
            const KeyDict& D = *kc[i]->dict;
            K.range = static_cast<unsigned long long>(std::max<long long>(1, D.d));
            K.dkeys = static_cast<const long long*>(D.hkeys->ptr);
            K.dranks = static_cast<const unsigned*>(D.hranks->ptr);
            K.dmask = D.mask;
            K.dempty = D.empty;
            hdict_vals[i] = D.vals.ptr<long long>();
          }
          total *= K.range;
          continue;
        }
        const KeyRange& r = *kc[i]->range;
        if (r.mn > r.mx) {  // empty key column: no row reaches the table
          K.kmin = 0;
          K.range = 1;
        } else if (use_dict[i]) {
          const KeyDict& D = *kc[i]->dict;
          K.kmin = 0;
          K.range = static_cast<unsigned long long>(std::max<long long>(1, D.d));
          K.dkeys = static_cast<const long long*>(D.hkeys->ptr);
          K.dranks = static_cast<const unsigned*>(D.hranks->ptr);
          K.dmask = D.mask;
          K.dempty = D.empty;
          hdict_vals[i] = D.vals.ptr<long long>();
        } else {
          K.kmin = r.mn;
          K.step = (P.hkey_lt[i] == TQP_LT_DATE && r.day == 1) ? 86400000000000LL : 1;
          K.range = (static_cast<unsigned long long>(r.mx) - static_cast<unsigned long long>(r.mn)) /
                        static_cast<unsigned long long>(K.step) + 1ULL;
          if (K.range == 0) return nofuse(__LINE__);  // the full 2^64 span
        }
        total *= K.range;
        if (total > (static_cast<unsigned __int128>(1) << 62)) return nofuse(__LINE__);
      }
      if (total > (static_cast<unsigned __int128>(1) << 62)) return nofuse(__LINE__);
      unsigned long long stride = 1;
      for (int i = nk - 1; i >= 0; --i) {
        ps.hkeys[i].stride = stride;
        stride *= ps.hkeys[i].range;
      }
      ps.nhkeys = nk;
      const unsigned long long R = static_cast<unsigned long long>(total);
      // special: one more word per record, NaN / +Inf / -Inf bits per accumulator;
      // 3-limb records are padded to whole 32-byte sectors, 2-limb ones are
      // kept dense (an L2-resident table is worth more than aligned records)
      const int L = (hlimbs == 2 && !po) ? 2 : kLimbWords;  // sharded partials: 3 limbs (no per-group fmax check)
      int W = 0;  // accumulator words per record (ProbeSpec::hoff)
      for (int a = 0; a < ps.nacc; ++a) {
        ps.hoff[a] = W;
        W += (L == 2 && ps.acc[a].is_int) ? 1 : L;
      }
      W = std::max(W, L * std::max(0, 1 - ps.nacc));  // no accumulator: one (unused) slot
      hrec_words = 1 + W + (special ? 1 : 0);
      if (L == kLimbWords) hrec_words = (hrec_words + 3) & ~3;
      ps.hflags = special ? 1 + W : -1;
      ps.hlimbs = L;
      const size_t priv_bytes = static_cast<size_t>(R) * (1 + kLimbWords * nacc_all) * sizeof(unsigned long long);
      ps.hpriv = priv_bytes <= kHashPrivBytes && !std::getenv("TQP_HASH_NOPRIV");
      ps.hdirect = ps.hpriv || (R <= kHashDirectMax && R <= 4ULL * static_cast<unsigned long long>(ps.n) + (1ULL << 20));
      if (ps.hdirect) {
        hcap = R;
      } else {
        const unsigned long long want = 2ULL * std::min<unsigned long long>(static_cast<unsigned long long>(std::max<long long>(ps.n, 1)), R);
        hcap = 1024;
        while (hcap < want) hcap <<= 1;
      }
      if (static_cast<double>(hcap) * (8.0 + 8.0 * hrec_words) > static_cast<double>(kHashMaxBytes)) return nofuse(__LINE__);
      // direct tables are indexed by code (hmask + 1 slots) and zeroed up
      // front: no tags; open-addressing tables claim slots by tag and the
      // claiming row zeroes the record
      ps.hmask = hcap - 1;
      hrec_buf = c.alloc_bytes(sizeof(unsigned long long) * hrec_words * hcap);
      if (ps.hdirect) {
        TQP_CUDA(cudaMemsetAsync(hrec_buf->ptr, 0, hrec_buf->bytes, c.stream));
        ps.htag = nullptr;
      } else {
        htag_buf = c.alloc_bytes(sizeof(unsigned long long) * hcap);
        TQP_CUDA(cudaMemsetAsync(htag_buf->ptr, 0, htag_buf->bytes, c.stream));
        ps.htag = static_cast<unsigned long long*>(htag_buf->ptr);
      }
      ps.fmax_out = po ? nullptr : err + 7;
      ps.absmax_out = po ? nullptr : err + 5;  // sharded partials keep the whole-scan bound
      ps.qfrac = qfrac;
      ps.qstats = po ? nullptr : err + 6;
      ps.gcnt = static_cast<unsigned long long*>(hrec_buf->ptr);
      ps.gacc = ps.gcnt + 1;
      ps.gstride = hrec_words;
    }
    // prefix sharing: an fp64 accumulator whose leading factors equal another
    // (earlier, ungated) accumulator's whole product starts from that value:
    // ((p*(1-d))*(1+t)) reuses p*(1-d) with identical rounding
    for (int a = 0; a < ps.nacc; ++a) {
      Acc& A = ps.acc[a];
      A.base = -1;
      if (A.is_int) continue;
      for (int b = a - 1; b >= 0 && A.base < 0; --b) {
        const Acc& B = ps.acc[b];
        if (B.is_int || B.gate_probe >= 0 || B.base >= 0 || B.nf >= A.nf || B.nf == 0) continue;
        bool same = true;
        for (int i = 0; i < B.nf && same; ++i) {
          const Factor &x = A.f[i], &y = B.f[i];
          same = x.kind == y.kind && x.k == y.k && x.x.ptr == y.x.ptr && x.x.src == y.x.src;
        }
        if (!same) continue;
        A.base = b;
        const int rest = A.nf - B.nf;
        for (int i = 0; i < kFixedFactors; ++i) {
          if (i < rest) {
            A.f[i] = A.f[i + B.nf];
          } else {
            A.f[i] = Factor{};
            A.f[i].kind = FK_CONST;
          }
        }
        A.nf = rest;
      }
    }

    if (ps.nacc > max_acc_for(P.mode)) return nofuse(__LINE__);
    // the tile kernels read accumulator operands from the staged fact tile;
    // MODE_HASH (generic kernel) also reads probe-root columns at the match
    for (int a = 0; a < ps.nacc; ++a)
      for (int i = 0; i < kFixedFactors; ++i)
        if (ps.acc[a].f[i].kind != FK_CONST && ps.acc[a].f[i].x.src >= 0 && P.mode != MODE_HASH) return nofuse(__LINE__);
    // distinct fact columns staged per tile; operands address them by index
    TileSpec ts;
    zero_padding(ts);
    auto col_index = [&](Operand& o) {
      if (o.src >= 0 || !o.ptr) return true;
      const int w = o.type == OT_U8 ? 1 : 8;
      for (int i = 0; i < ts.ncols; ++i) {
        if (ts.col_ptr[i] == o.ptr) {
          o.col = i;
          return true;
        }
      }
      if (ts.ncols >= kMaxCols) return nofuse(__LINE__);
      ts.col_ptr[ts.ncols] = static_cast<const unsigned char*>(o.ptr);
      ts.col_w[ts.ncols] = w;
      o.col = ts.ncols++;
      return true;
    };
    for (int i = 0; i < ps.nterms; ++i) {
      if (ps.terms[i].kind >= RK_TRUE) continue;
      if (!col_index(term_cols[i])) return nofuse(__LINE__);
      ps.terms[i].col = term_cols[i].col;
    }
    for (int i = 0; i < ps.nprobes; ++i)
      if (!col_index(ps.probes[i].key)) return nofuse(__LINE__);
    for (int a = 0; a < ps.nacc; ++a)
      for (int i = 0; i < ps.acc[a].nf; ++i)
        if (ps.acc[a].f[i].kind != FK_CONST && !col_index(ps.acc[a].f[i].x)) return nofuse(__LINE__);
    for (int i = 0; i < ps.nkeys; ++i)
      if (!col_index(ps.keys[i])) return nofuse(__LINE__);
    for (int i = 0; i < ps.nhkeys; ++i)  // int64 fact keys come from the staged tile
      if (!ps.hkeys[i].width && ps.hkeys[i].x.src < 0 && !col_index(ps.hkeys[i].x)) return nofuse(__LINE__);
    // the common hash-group shape runs the lean instance (fused_kernels.cuh)
    bool lean = P.mode == MODE_HASH && !ps.hpriv && !ps.htag && ps.hlimbs == 2 && ps.hflags < 0 && ps.nprobes == 0 &&
                !ps.weighted && !std::getenv("TQP_HASH_NOLEAN");
    for (int i = 0; lean && i < ps.nhkeys; ++i) {
      const GKey& K = ps.hkeys[i];
      lean = K.x.src < 0 && K.x.col >= 0 && !K.width && !K.dkeys;
    }
    for (int a = 0; lean && a < ps.nacc; ++a) {
      lean = ps.acc[a].gate_probe < 0;
      for (int i = 0; lean && i < kFixedFactors; ++i) lean = ps.acc[a].f[i].x.src < 0;
    }
    ts.rows = P.mode == MODE_SMALL ? TileShape<MODE_SMALL>::ROWS : lean ? TileShape<MODE_HASH, true>::ROWS : kTileRows;
    ts.aux_bytes = static_cast<int>(P.mode == MODE_SMALL    ? aux_bytes_for<MODE_SMALL>(ps.nacc)
                                    : P.mode == MODE_SCALAR ? aux_bytes_for<MODE_SCALAR>(ps.nacc)
                                                            : aux_bytes_for<MODE_BUILDGRP>(ps.nacc));
    ts.evict_first = (P.mode == MODE_HASH && !ps.hpriv && !std::getenv("TQP_NO_EVICT_FIRST")) ? 1 : 0;
    if (P.mode == MODE_HASH && ps.hpriv)  // the CTA's records [code][count, limbs per accumulator]
      ts.aux_bytes = static_cast<int>(((ps.hmask + 1) * (1 + kLimbWords * ps.nacc) * sizeof(unsigned long long) + 15) & ~15ULL);
    const bool wide = P.mode == MODE_SMALL && !narrow && jit_wanted(ps.n) && small_wide_wanted() && !generic_only;
    int small_threads = TileShape<MODE_SMALL>::THREADS;
    const bool regacc = wide && small_regacc();
    const int wide_cw = regacc ? small_reg_cw() : kWideCW;
    if (regacc) {  // register accumulators: no cells, taller tiles, more consumer warps
      ts.aux_bytes = 0;
      ts.rows = small_reg_rows();
      small_threads = wide_cw * 32 + 32;
    } else if (wide) {  // per-thread cells for kWideSlots slots, kWideCW consumer warps
      ts.aux_bytes = static_cast<int>(sizeof(unsigned long long) * kWideSlots * (ps.nacc + 1) * kWideCW * 32);
      small_threads = kWideCW * 32 + 32;
    }
    for (int i = 0; i < ts.ncols; ++i) {
      ts.col_off[i] = ts.stage_bytes;
      ts.stage_bytes += (ts.rows * ts.col_w[i] + 127) & ~127;  // 128 B aligned columns
    }
    if (ts.stage_bytes == 0) ts.stage_bytes = 128;
    // as many stages as fit next to the fixed (static + staging) parts
    const int optin = c.smem_optin();
    cudaFuncAttributes fa{};
    const size_t fixed = 256 + static_cast<size_t>(ts.aux_bytes);
    const void* kfn = lean ? tile_kernel_lean(ps.nacc) : tile_kernel(P.mode, ps.nacc);
    if (!kfn) return nofuse(__LINE__);
    const bool jit = jit_wanted(ps.n) && (P.mode != MODE_HASH || lean) && !generic_only && ps.nacc > 0;
    if (jit) {
      std::vector<int> bm;
      for (const auto& pd : P.probes) bm.push_back(probe_mode_of(P.builds[pd.build]));
      ts.p = ps;
      const int cw = wide ? wide_cw : P.mode == MODE_SMALL ? TileShape<MODE_SMALL>::CW : TileShape<MODE_SCALAR>::CW;
      hp.mark("tprep");
      const int slots = wide ? kWideSlots : kGroups;
      std::string key = tile_key(ts);
      for (int v : {static_cast<int>(P.mode), cw, slots, regacc ? 1 : 0}) append_bytes(key, v);
      for (int v : bm) append_bytes(key, v);
      kfn = memo->get(-1, key, [&] { return jit_kernel(gen_pipeline(ts, P.mode, cw, bm, slots, regacc), "q_tile"); });
      hp.mark("tgen");
    }
    hp.mark("gen");
    fa.sharedSizeBytes = c.static_smem(kfn);
    const size_t budget = static_cast<size_t>(optin) - fa.sharedSizeBytes - 1024;
    if (fixed + 2 * static_cast<size_t>(ts.stage_bytes) > budget) return nofuse(__LINE__);
    ts.stages = static_cast<int>(std::min<size_t>(kMaxStages, (budget - fixed) / ts.stage_bytes));
    const size_t smem = fixed + static_cast<size_t>(ts.stages) * ts.stage_bytes;
    const std::string tile_name = std::string(jit ? "q_tile<" : "k_tile<") +
                                  (P.mode == MODE_SCALAR  ? "scalar"
                                   : P.mode == MODE_SMALL ? "small"
                                   : P.mode == MODE_HASH  ? (ps.hpriv ? "hash-priv" : lean ? "hash-lean" : ps.hdirect ? "hash-direct" : "hash")
                                                          : "buildgrp") + "," +
                                  std::to_string(ps.nacc) + ">";
    auto launch_tile = [&](const void* kernel, int threads, int grid_) -> void {
      cudaError_t e = c.ensure_smem(kernel, static_cast<int>(smem));
      if (e != cudaSuccess) {
        throw Error(TQP_ERR_CUDA, std::string("cuda: ") + cudaGetErrorString(e) + " setting " + std::to_string(smem) +
                                      " B dynamic smem (static " + std::to_string(fa.sharedSizeBytes) + ", optin " +
                                      std::to_string(optin) + ", stages " + std::to_string(ts.stages) + ")");
      }
      ts.p = ps;
      void* args[] = {&ts};
      cudaEvent_t ev = c.kernel_begin(true);
      TQP_CUDA(cudaLaunchKernel(kernel, dim3(grid_), dim3(threads), args, smem, c.stream));
      c.kernel_end(tile_name, ev);
      TQP_CUDA(cudaGetLastError());
      c.count_launch();
    };

    FinalSpec fs;
    if (!final_spec(P, fs)) return nofuse(__LINE__);
    const int grid = c.num_sms;  // persistent: one CTA per SM
    std::vector<Tensor> outs(P.outs.size());
    long long nrows = 0;
    // phase 1 of a sharded run writes its partial state straight after the
    // header; the local run merges it with the same phase-2 kernels (one part)
    std::shared_ptr<DevBuf> part_keep;  // alive until the merge has read it
    auto part_buf = [&](long long nrec, int words) {
      auto buf = c.alloc_bytes(sizeof(unsigned long long) * (kHdrWords + nrec * words));
      part_keep = buf;
      if (po) {
        unsigned long long h[kHdrWords] = {kPartMagic,
                                           static_cast<unsigned long long>(P.mode),
                                           static_cast<unsigned long long>(nrec),
                                           static_cast<unsigned long long>(words),
                                           static_cast<unsigned long long>(fs.nacc),
                                           static_cast<unsigned long long>(fs.nouts),
                                           static_cast<unsigned long long>(P.mode == MODE_HASH ? ps.nhkeys : static_cast<int>(P.key_columns.size())),
                                           hash_key_widths(ps)};
        TQP_CUDA(cudaMemcpyAsync(buf->ptr, h, sizeof(h), cudaMemcpyHostToDevice, c.stream));
        po->buf = buf;
        po->words = kHdrWords + nrec * words;
      }
      return static_cast<unsigned long long*>(buf->ptr) + kHdrWords;
    };

    if (P.mode == MODE_SCALAR) {
      ps.part = part_buf(grid, kMaxAcc + 1);
      launch_tile(kfn, TileShape<MODE_SCALAR>::THREADS, grid);
      if (!po) final_scalar(c, ps.part, grid, fs, err, outs);
      nrows = 1;
    } else if (P.mode == MODE_SMALL) {
      ps.part = part_buf(grid, kSmallPartWords);
      launch_tile(kfn, small_threads, grid);
      if (!po) nrows = final_small(c, reinterpret_cast<const SmallPart*>(ps.part), grid, fs, err, outs);
    } else if (P.mode == MODE_HASH) {
      launch_tile(kfn, lean ? TileShape<MODE_HASH, true>::THREADS : TileShape<MODE_HASH>::THREADS, grid);
      auto pres = c.alloc_bytes(sizeof(unsigned) * ((hcap + 31) / 32 + 1));
      keep.push_back(pres);
      keep.push_back(htag_buf);
      keep.push_back(hrec_buf);
      // a direct table's presence bits say no more than its count words:
      // only the top-k walk reads them
      const bool want_present = ps.htag || (P.topk && !fullsort);
      if (ps.htag)
        k_hash_present<<<c.grid_for(static_cast<long long>(hcap), 256), 256, 0, c.stream>>>(
            ps.htag, static_cast<long long>(hcap), static_cast<unsigned*>(pres->ptr));
      else if (want_present)
        k_count_present<<<c.grid_for(static_cast<long long>(hcap), 256), 256, 0, c.stream>>>(
            ps.gcnt, ps.gstride, static_cast<long long>(hcap), static_cast<unsigned*>(pres->ptr));
      if (want_present) c.count_launch();
      GroupSpec gs = hash_group_spec(ps, fs, want_present ? static_cast<const unsigned*>(pres->ptr) : nullptr, hdict_vals);
      if (po) {
        Tensor gids = touched_groups(c, ps.gcnt, ps.gstride, static_cast<long long>(hcap), gs.present);
        const long long n = gids.rows;
        const int words = record_words(gs.nkeyc, fs.nacc);
        unsigned long long* rec = part_buf(n, words);
        if (n) {
          k_fill_records<<<c.grid_for(n, 256), 256, 0, c.stream>>>(gs, gids.ptr<long long>(), n, nullptr, words, rec, err);
          c.count_launch();
        }
      } else if (!emit_groups(c, gs, static_cast<long long>(hcap), reinterpret_cast<const long long*>(ps.htag), err, outs,
                              nrows, fullsort, !ps.htag)) {
        return nofuse(__LINE__);
      }
    } else {
      // MODE_BUILDGRP
      long long ngroups = build_range[P.probes[P.group_probe].build];
      if (!grec_p || !group_present) return nofuse(__LINE__);  // the group build assigns the groups
      ps.gcnt = grec_p;
      ps.gacc = grec_p + 1;
      ps.gstride = grec_words;
      ps.group_probe = P.group_probe;
      if (!touched_off) return nofuse(__LINE__);
      ps.touched = reinterpret_cast<unsigned*>(arena_p + touched_off);
      launch_tile(kfn, TileShape<MODE_BUILDGRP>::THREADS, grid);
      GroupSpec gs;
      gs.f = fs;
      gs.gacc = ps.gacc;
      gs.gcnt = ps.gcnt;
      gs.group_table = group_table;
      gs.row_in_cnt = row_rec_grp ? 1 : 0;
      gs.cnt_stride = grec_words;
      gs.acc_stride = grec_words;
      gs.present = ps.touched;  // groups with rows (a subset of the inserted slots)
      gs.acc_words = kLimbWords;
      const BuildDesc& gb = P.builds[P.probes[P.group_probe].build];
      const Table* groot = bind_table(tables, gb.table);
      gs.nkeyc = static_cast<int>(P.group_key_root_columns.size());
      for (int i = 0; i < gs.nkeyc; ++i) {
        const Column* kc = groot->find(P.group_key_root_columns[i]);
        if (!kc || kc->t.dtype != TQP_I64) return nofuse(__LINE__);
        gs.key_cols[i] = kc->t.ptr<long long>();
      }
      const Column* bk = groot->find(gb.key_column);
      if (po) {
        // the touched groups as self-describing records, keyed by the unique
        // build key: shards may split a group (the merge adds exactly)
        Tensor gids = touched_groups(c, ps.gcnt, ps.gstride, ngroups, ps.touched, row_rec_grp ? 0xffffffffULL : ~0ULL);
        const long long n = gids.rows;
        const int words = record_words(gs.nkeyc, fs.nacc);
        unsigned long long* rec = part_buf(n, words);
        if (n) {
          k_fill_records<<<c.grid_for(n, 256), 256, 0, c.stream>>>(gs, gids.ptr<long long>(), n, bk->t.ptr<long long>(),
                                                                  words, rec, err);
          c.count_launch();
        }
      } else if (!emit_groups(c, gs, ngroups, bk->t.ptr<long long>(), err, outs, nrows, fullsort)) {
        return nofuse(__LINE__);
      }
    }
    long long herr[4] = {0, 0, 0, 0};
    hp.mark("launched");
    if (pend && !po) {
      // deferred: the word travels with the outputs and is checked at the
      // result's synchronisation; rows are patched there when device-side
      TQP_CUDA(cudaMemcpyAsync(pend->host ? pend->host : c.h_err + Ctx::kPinnedUnitErr, err, 32, cudaMemcpyDeviceToHost,
                               c.stream));
      pend->active = true;
      pend->nrows = nrows;
      pend->err = err_buf;
      pend->outs.clear();
      for (auto& o : outs) pend->outs.push_back(o.data());
      for (size_t i = 0; i < P.final_slots.size(); ++i) (*slots)[P.final_slots[i]] = outs[P.final_cols[i]];
      return true;
    }
    TQP_CUDA(cudaMemcpyAsync(c.h_err + Ctx::kPinnedRead, err, 32, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    hp.mark("sync");
    std::memcpy(herr, c.h_err + Ctx::kPinnedRead, 32);
    if (exchange && (herr[0] || herr[1])) {
      // a re-run would repeat this rank's collectives alone: the caller
      // agrees across ranks and gathers the tables instead
      if (po) *po = Partial{};
      return nofuse(__LINE__);
    }
    if (wide && herr[1] && !herr[0]) return run(c, slots, tables, po, o.with_narrow(true));  // a fifth key in a CTA
    if (herr[0] && herr[3] == FR_DUP_KEY && !weighted) {
      if (std::getenv("TQP_DEBUG_FALLBACK")) std::fprintf(stderr, "tqp: repeated build keys: unit reruns weighted\n");
      { RunOpts r = o; r.weighted = true; return run(c, slots, tables, po, r); }
    }
    if (herr[0] && (herr[3] == FR_TOPK_BLOCK || herr[3] == FR_TOPK_FINAL) && !fullsort && P.topk && !po) {
      if (std::getenv("TQP_DEBUG_FALLBACK")) std::fprintf(stderr, "tqp: top-k ties overflow: unit reruns with a full group sort\n");
      { RunOpts r = o; r.fullsort = true; return run(c, slots, tables, po, r); }
    }
    if (herr[0] && (herr[3] == FR_LIMB2 || herr[3] == FR_GROUP_VALUE) && P.mode == MODE_HASH && hlimbs == 2) {
      if (std::getenv("TQP_DEBUG_FALLBACK")) std::fprintf(stderr, "tqp: 2-limb group sums out of range: unit reruns with 3 limbs\n");
      { RunOpts r = o; r.hlimbs = 3; return run(c, slots, tables, po, r); }
    }
    if (herr[0] && herr[3] == FR_Q64_CONVERT && P.mode == MODE_HASH && !po && (!special || qfrac == 64)) {
      // NaN / Inf values: flagged per group; finite values with bits below
      // 2^-64: more fraction bits (exact while the sums' range allows)
      long long lowneg = 0;
      TQP_CUDA(cudaMemcpyAsync(&lowneg, err + 6, sizeof(lowneg), cudaMemcpyDeviceToHost, c.stream));
      c.sync();
      const int F = std::max<long long>(64, lowneg) > 120 ? -1 : static_cast<int>(std::max<long long>(64, lowneg));
      if (F > 0 && (!special || F > qfrac)) {
        if (std::getenv("TQP_DEBUG_FALLBACK"))
          std::fprintf(stderr, "tqp: NaN/Inf or fine fp64 group values: unit reruns with special flags, %d fraction bits\n", F);
        { RunOpts r = o; r.special = true; r.qfrac = F; return run(c, slots, tables, po, r); }
      }
    }
    if (herr[0] && alt && (P.mode == MODE_SMALL || P.mode == MODE_BUILDGRP)) {
      if (std::getenv("TQP_DEBUG_FALLBACK")) std::fprintf(stderr, "tqp: unit reruns as hash-group (reason %lld)\n", herr[3]);
      return alt->run(c, slots, tables, po, o.with_narrow(false));
    }
    if (herr[0] && std::getenv("TQP_DEBUG_FALLBACK"))
      std::fprintf(stderr, "tqp: fused unit left the fused path (reason %lld)\n", herr[3]);
    if (herr[0]) {  // preconditions violated: exact per-instruction path
      if (po) *po = Partial{};
      return nofuse(__LINE__);
    }
    if (po) return true;
    if (nrows < 0) nrows = herr[2];
    for (size_t j = 0; j < outs.size(); ++j) outs[j].rows = nrows;
    for (size_t i = 0; i < P.final_slots.size(); ++i) (*slots)[P.final_slots[i]] = outs[P.final_cols[i]];
    return true;
  }

  // ---- shared phase-2 pieces -----------------------------------------------------
  static int out_dtype(const PipeDesc& P, const OutDesc& o) {
    if (o.fn >= 10) return P.mode == MODE_SMALL ? TQP_STR8 : TQP_I64;
    if (o.fn == 1) return TQP_I64;
    if (o.fn == 2) return TQP_F64;
    return o.is_int ? TQP_I64 : TQP_F64;
  }

  bool final_spec(const PipeDesc& P_, FinalSpec& fs) const {
    fs.nacc = static_cast<int>(P_.accs.size());
    if (fs.nacc > kMaxAcc) return false;
    for (int a = 0; a < fs.nacc; ++a) fs.acc_is_int[a] = P_.accs[a].is_int;
    fs.nouts = static_cast<int>(P_.outs.size());
    if (fs.nouts > 16) return false;
    for (int j = 0; j < fs.nouts; ++j) {
      const OutDesc& d = P_.outs[j];
      fs.outs[j] = {d.fn, d.acc, d.is_int ? 1 : 0, d.op, d.a, d.b};
    }
    if (P_.konst.size() > static_cast<size_t>(kMaxEpiConst)) return false;
    for (size_t i = 0; i < P_.konst.size(); ++i) fs.konst[i] = P_.konst[i];
    return true;
  }

  void final_scalar(Ctx& c, const unsigned long long* part, long long nparts, FinalSpec fs, long long* err,
                    std::vector<Tensor>& outs) const {
    for (size_t j = 0; j < outs.size(); ++j) {
      outs[j] = c.alloc(out_dtype(P, P.outs[j]), 1, 1);
      fs.out_ptr[j] = outs[j].data();
    }
    k_final_scalar<<<1, kThreads, 0, c.stream>>>(part, nparts, fs, err);
    c.count_launch();
  }

  long long final_small(Ctx& c, const SmallPart* parts, long long nparts, FinalSpec fs, long long* err,
                        std::vector<Tensor>& outs) const {
    auto rank = c.alloc_bytes(sizeof(int) * nparts * kGroups);
    for (size_t j = 0; j < outs.size(); ++j) {
      outs[j] = c.alloc(out_dtype(P, P.outs[j]), kMerged, 1);
      fs.out_ptr[j] = outs[j].data();
    }
    void* kp[4] = {nullptr, nullptr, nullptr, nullptr};
    for (size_t j = 0; j < P.outs.size(); ++j)
      if (P.outs[j].fn >= 10) kp[P.outs[j].fn - 10] = outs[j].data();
    const size_t staged = nparts * (sizeof(SmallPart) + sizeof(int) * kGroups);
    static_assert(sizeof(SmallPart) % 16 == 0, "staged copy moves 16-byte vectors");
    const bool stage = staged <= kFinalSmallStageMax && reinterpret_cast<uintptr_t>(parts) % 16 == 0 &&
                       c.ensure_smem(reinterpret_cast<const void*>(&k_final_small<true>), static_cast<int>(staged)) ==
                           cudaSuccess;
    if (stage)
      k_final_small<true><<<1, kFinalSmallThreads, staged, c.stream>>>(
          parts, static_cast<int>(nparts), fs, static_cast<int>(P.key_columns.size()), kp[0], kp[1], kp[2], kp[3],
          static_cast<int*>(rank->ptr), err + 2, err);
    else
      k_final_small<false><<<1, kFinalSmallThreads, 0, c.stream>>>(
          parts, static_cast<int>(nparts), fs, static_cast<int>(P.key_columns.size()), kp[0], kp[1], kp[2], kp[3],
          static_cast<int*>(rank->ptr), err + 2, err);
    c.count_launch();
    return -1;  // on the device (err[2]); read with the error flag
  }

  // cmask: the count bits of a count word (row_in_cnt: the low 32)
  // ascending slots whose count word is nonzero, in one pass (k_nonzero_slots)
  static Tensor nonzero_slots(Ctx& c, const unsigned long long* gcnt, long long cnt_stride, long long ngroups) {
    if (!ngroups) return c.alloc(TQP_I64, 0, 1);
    const long long tiles = (ngroups + kSlotTile - 1) / kSlotTile;
    auto scratch = c.alloc_bytes(sizeof(longlong2) * (tiles + 1) + 16);
    TQP_CUDA(cudaMemsetAsync(scratch->ptr, 0, scratch->bytes, c.stream));
    auto* desc = static_cast<longlong2*>(scratch->ptr);
    Tensor o = c.alloc(TQP_I64, ngroups, 1);
    k_nonzero_slots<<<static_cast<unsigned>(tiles), kSlotThreads, 0, c.stream>>>(
        gcnt, cnt_stride, ngroups, o.ptr<long long>(), desc, reinterpret_cast<int*>(desc + tiles + 1));
    c.count_launch();
    long long* h = c.h_err + Ctx::kPinnedRead;
    TQP_CUDA(cudaMemcpyAsync(h, desc + tiles - 1, sizeof(longlong2), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    const long long total = h[1];
    if (total * 2 < ngroups) {
      Tensor t = c.alloc(TQP_I64, total, 1);
      if (total) TQP_CUDA(cudaMemcpyAsync(t.data(), o.data(), t.bytes(), cudaMemcpyDeviceToDevice, c.stream));
      return t;
    }
    o.rows = total;
    return o;
  }

  static Tensor touched_groups(Ctx& c, const unsigned long long* gcnt, long long cnt_stride, long long ngroups,
                               const unsigned* present, unsigned long long cmask = ~0ULL) {
    if (!present && cmask == ~0ULL) return nonzero_slots(c, gcnt, cnt_stride, ngroups);
    Tensor mask = c.alloc(TQP_BOOL, ngroups, 1);
    if (ngroups) {
      k_nonzero_groups<<<c.grid_for(ngroups, 256), 256, 0, c.stream>>>(gcnt, cnt_stride, ngroups, present, cmask,
                                                                       mask.ptr<uint8_t>());
      c.count_launch();
    }
    return k::compact(c, k::iota(c, ngroups), mask);
  }

  // a group output column: STR8 (rows, width) for a string key of a hash
  // unit, else per out_dtype
  Tensor alloc_out(Ctx& c, const GroupSpec& gs, size_t j, long long rows) const {
    const OutDesc& o = P.outs[j];
    if (o.fn >= 10 && gs.key_w[o.fn - 10]) return c.alloc(TQP_STR8, rows, gs.key_w[o.fn - 10]);
    return c.alloc(out_dtype(P, o), rows, 1);
  }

  // group outputs: top-k in the reference's tie order, or every group
  // ascending by the (unique) build key `bk` (indexed like the key columns)
  // fullsort: the top-k kernel met more ties than it keeps candidates for;
  // every group is emitted in ascending key order and the ORDER BY + LIMIT
  // run as the reference lowers them (stable SortPermRows per key, last key
  // first, then the first k rows), on the device
  // gids_sorted: slot order is key order (direct hash-group tables)
  bool emit_groups(Ctx& c, GroupSpec gs, long long ngroups, const long long* bk, long long* err,
                   std::vector<Tensor>& outs, long long& nrows, bool fullsort = false, bool gids_sorted = false) const {
    if (P.topk && fullsort) {
      GroupSpec all = gs;
      std::vector<Tensor> rows(outs.size());
      if (!emit_all_groups(c, all, ngroups, bk, err, rows, nrows, gids_sorted)) return false;
      Tensor perm = k::iota(c, nrows);
      for (int i = static_cast<int>(P.sort_outs.size()) - 1; i >= 0; --i)
        perm = k::sort_perm_rows(c, rows[P.sort_outs[i].first], perm, P.sort_outs[i].second);
      const long long m = std::min<long long>(nrows, P.k);
      perm.rows = m;
      for (size_t j = 0; j < outs.size(); ++j) outs[j] = k::gather(c, rows[j], perm);
      nrows = m;
      return true;
    }
    if (P.topk) {
      gs.nsort = static_cast<int>(P.sort_outs.size());
      for (int i = 0; i < gs.nsort; ++i) {
        gs.sort_out[i] = P.sort_outs[i].first;
        gs.sort_asc[i] = P.sort_outs[i].second;
      }
      const int k = static_cast<int>(P.k);
      for (size_t j = 0; j < outs.size(); ++j) {
        outs[j] = alloc_out(c, gs, j, std::max(1, k));
        gs.f.out_ptr[j] = outs[j].data();
      }
      nrows = 0;
      if (k == 0 || ngroups == 0) return true;
      const int nk = gs.nsort + gs.nkeyc;
      TopkKernel kern = topk_kernel(nk);
      if (!kern || k > kTopkMaxK || gs.nsort < 1) return false;
      // one wave: as many blocks as are resident at once, up to topk_bps()
      // per SM (the last block reads one value list per block)
      const int per_sm = c.blocks_per_sm(reinterpret_cast<const void*>(kern), kTopkThreads);
      const int blocks = static_cast<int>(std::max<long long>(
          1, std::min<long long>({static_cast<long long>(std::max(1, std::min(per_sm, topk_bps()))) * c.num_sms,
                                  (ngroups + 8191) / 8192, static_cast<long long>(kTopkMaxBlocks)})));
      auto bck = c.alloc_bytes(sizeof(unsigned long long) * blocks * kTopkBlkCand);
      auto bcg = c.alloc_bytes(sizeof(unsigned) * blocks * kTopkBlkCand);
      auto bn = c.alloc_bytes(sizeof(int) * blocks + 16);
      int* bnc = static_cast<int*>(bn->ptr);
      // the last-block ticket lives after the error words (zeroed with them)
      unsigned* ticket = reinterpret_cast<unsigned*>(err + 4);
      static const bool tracing = std::getenv("TQP_TOPK_TRACE") != nullptr;
      std::shared_ptr<DevBuf> tb;
      if (tracing) {
        tb = c.alloc_bytes(sizeof(unsigned long long) * (8 * blocks + 12));
        TQP_CUDA(cudaMemsetAsync(tb->ptr, 0, tb->bytes, c.stream));
      }
      kern<<<blocks, kTopkThreads, 0, c.stream>>>(gs, ngroups, k, static_cast<unsigned long long*>(bck->ptr),
                                                  static_cast<unsigned*>(bcg->ptr), bnc, ticket, err + 2, err,
                                                  tb ? static_cast<unsigned long long*>(tb->ptr) : nullptr);
      c.count_launch();
      if (tracing) topk_trace_report(c, tb, blocks);
      nrows = -1;  // on the device (err[2]); read with the error flag
      return true;
    }
    return emit_all_groups(c, gs, ngroups, bk, err, outs, nrows, gids_sorted);
  }

  // every group with rows, ascending by its (unique) key `bk`
  bool emit_all_groups(Ctx& c, GroupSpec gs, long long ngroups, const long long* bk, long long* err,
                       std::vector<Tensor>& outs, long long& nrows, bool gids_sorted = false) const {
    Tensor gids = touched_groups(c, gs.gcnt, gs.cnt_stride, ngroups, gs.present,
                                 gs.row_in_cnt ? 0xffffffffULL : ~0ULL);
    const long long n = gids.rows;
    Tensor order;
    if (!gids_sorted) {
      Tensor keys = c.alloc(TQP_I64, n, 1);
      if (n) {
        k_group_keys<<<c.grid_for(n, 256), 256, 0, c.stream>>>(gs.group_table, gs.row_in_cnt ? gs.gcnt : nullptr,
                                                                gs.cnt_stride, gids.ptr<long long>(), n, bk,
                                                                keys.ptr<long long>());
        c.count_launch();
      }
      // positions of the touched groups in ascending build-key order
      order = k::radix_sort_payload(c, keys, nullptr, false);
    }
    for (size_t j = 0; j < outs.size(); ++j) {
      outs[j] = alloc_out(c, gs, j, n);
      gs.f.out_ptr[j] = outs[j].data();
    }
    if (n) {
      k_group_rows<<<c.grid_for(n, 256), 256, 0, c.stream>>>(gs, gids.ptr<long long>(),
                                                              gids_sorted ? nullptr : order.ptr<long long>(), n, err);
      c.count_launch();
    }
    nrows = n;
    return true;
  }

  // ---- phase 2 of a sharded run: merge the parts (in the given order) ----------
  void finish(Ctx& c, std::vector<std::optional<Tensor>>& slots, const std::vector<PartRef>& parts,
              const std::string& where) const {
    FinalSpec fs;
    if (!final_spec(P, fs)) throw Error(TQP_ERR_EXEC, where + ": unit has no partial form");
    const int nkeyc = static_cast<int>(P.mode == MODE_HASH ? P.hkeys.size() : P.group_key_root_columns.size());
    const size_t hdr_keys = P.mode == MODE_HASH ? P.hkeys.size() : P.key_columns.size();
    unsigned long long key_widths = 0;
    const long long want_words = P.mode == MODE_SCALAR  ? kMaxAcc + 1
                                 : P.mode == MODE_SMALL ? kSmallPartWords
                                                        : record_words(nkeyc, fs.nacc);
    if (parts.empty()) throw Error(TQP_ERR_ARG, where + ": no partials to merge");
    if (alt && (P.mode == MODE_SMALL || P.mode == MODE_BUILDGRP) && parts[0].ptr && parts[0].words >= kHdrWords) {
      // shards whose small-group run overflowed produced hash-group partials
      unsigned long long h[kHdrWords];
      TQP_CUDA(cudaMemcpyAsync(h, parts[0].ptr, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
      c.sync();
      if (h[0] == kPartMagic && h[1] == static_cast<unsigned long long>(MODE_HASH)) return alt->finish(c, slots, parts, where);
    }
    long long total = 0;
    std::vector<long long> nrec(parts.size());
    for (size_t i = 0; i < parts.size(); ++i) {
      unsigned long long h[kHdrWords];
      if (!parts[i].ptr || parts[i].words < kHdrWords) throw Error(TQP_ERR_ARG, where + ": partial " + std::to_string(i) + " is truncated");
      TQP_CUDA(cudaMemcpyAsync(h, parts[i].ptr, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
      c.sync();
      if (h[0] != kPartMagic || h[1] != static_cast<unsigned long long>(P.mode) ||
          h[3] != static_cast<unsigned long long>(want_words) || h[4] != static_cast<unsigned long long>(fs.nacc) ||
          h[5] != static_cast<unsigned long long>(fs.nouts) || h[6] != hdr_keys || (i > 0 && h[7] != key_widths)) {
        throw Error(TQP_ERR_ARG, where + ": partial " + std::to_string(i) + " was not produced by this plan");
      }
      key_widths = h[7];
      nrec[i] = static_cast<long long>(h[2]);
      if (kHdrWords + nrec[i] * want_words > parts[i].words)
        throw Error(TQP_ERR_ARG, where + ": partial " + std::to_string(i) + " is truncated");
      total += nrec[i];
    }
    auto cat = c.alloc_bytes(sizeof(unsigned long long) * std::max<long long>(1, total * want_words));
    unsigned long long* catp = static_cast<unsigned long long*>(cat->ptr);
    long long off = 0;
    for (size_t i = 0; i < parts.size(); ++i) {
      if (nrec[i])
        TQP_CUDA(cudaMemcpyAsync(catp + off * want_words, static_cast<const unsigned long long*>(parts[i].ptr) + kHdrWords,
                                 sizeof(unsigned long long) * nrec[i] * want_words, cudaMemcpyDeviceToDevice, c.stream));
      off += nrec[i];
    }
    auto err_buf = c.alloc_bytes(64);  // error words + the top-k ticket
    long long* err = static_cast<long long*>(err_buf->ptr);
    TQP_CUDA(cudaMemsetAsync(err, 0, 64, c.stream));
    std::vector<Tensor> outs(P.outs.size());
    long long nrows = 0;
    bool ok = true;
    std::vector<std::shared_ptr<DevBuf>> keep;
    if (P.mode == MODE_SCALAR) {
      final_scalar(c, catp, total, fs, err, outs);
      nrows = 1;
    } else if (P.mode == MODE_SMALL) {
      nrows = final_small(c, reinterpret_cast<const SmallPart*>(catp), total, fs, err, outs);
    } else {
      // open-addressing table keyed by the build key, at most half full
      long long cap = 1024;
      while (cap < 2 * total) cap <<= 1;
      const int nacc = std::max(1, fs.nacc);
      auto htag = c.alloc_bytes(sizeof(unsigned long long) * cap);
      auto hbk = c.alloc_bytes(sizeof(long long) * cap);
      auto hkeys = c.alloc_bytes(sizeof(long long) * cap * std::max(1, nkeyc));
      auto hcnt = c.alloc_bytes(sizeof(unsigned long long) * cap);
      auto hacc = c.alloc_bytes(sizeof(unsigned long long) * 2 * nacc * cap);
      keep = {htag, hbk, hkeys, hcnt, hacc};
      for (auto& b : {htag, hcnt, hacc}) TQP_CUDA(cudaMemsetAsync(b->ptr, 0, b->bytes, c.stream));
      if (total) {
        k_merge_records<<<c.grid_for(total, 256), 256, 0, c.stream>>>(
            catp, total, static_cast<int>(want_words), nkeyc, fs.nacc, cap - 1,
            static_cast<unsigned long long*>(htag->ptr), static_cast<long long*>(hbk->ptr),
            static_cast<long long*>(hkeys->ptr), static_cast<unsigned long long*>(hcnt->ptr),
            static_cast<unsigned long long*>(hacc->ptr), err);
        c.count_launch();
      }
      GroupSpec gs;
      gs.f = fs;
      gs.gacc = static_cast<unsigned long long*>(hacc->ptr);
      gs.gcnt = static_cast<unsigned long long*>(hcnt->ptr);
      gs.group_table = nullptr;
      gs.cnt_stride = 1;
      gs.acc_stride = 2LL * fs.nacc;
      gs.nkeyc = nkeyc;
      for (int i = 0; i < nkeyc; ++i) gs.key_cols[i] = static_cast<const long long*>(hkeys->ptr) + i * cap;
      for (int i = 0; i < nkeyc; ++i) gs.key_w[i] = static_cast<int>((key_widths >> (8 * i)) & 0xff);
      ok = emit_groups(c, gs, cap, static_cast<const long long*>(hbk->ptr), err, outs, nrows);
    }
    long long herr[4] = {0, 0, 0, 0};
    TQP_CUDA(cudaMemcpyAsync(c.h_err + Ctx::kPinnedRead, err, 32, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    std::memcpy(herr, c.h_err + Ctx::kPinnedRead, 32);
    if (nrows < 0) nrows = herr[2];
    if (herr[0] && (herr[3] == kReasonEpiDivZero || herr[3] == kReasonEpiOverflow))
      throw Error(TQP_ERR_EXEC, P.epi_step + (herr[3] == kReasonEpiDivZero ? ": arith: division by zero at row 0"
                                                                            : ": arith: integer overflow at row 0"),
                  0);
    if (!ok || herr[0]) {
      // the local path would re-run these steps per instruction; merged
      // partials cannot, so report what the exact path raises
      throw Error(TQP_ERR_EXEC, where + ": merged partials violate the fused preconditions "
                                        "(AVG over zero rows, more than 256 groups, or an int64 overflow)");
    }
    for (size_t j = 0; j < outs.size(); ++j) outs[j].rows = nrows;
    for (size_t i = 0; i < P.final_slots.size(); ++i) slots[P.final_slots[i]] = outs[P.final_cols[i]];
  }
};

}  // namespace

std::vector<FusedUnit> plan_fusion(Ctx& ctx, const Plan& plan) {
  (void)ctx;
  std::vector<FusedUnit> units;
  Analysis A(plan);
  A.analyse();
  // live-out check helper: slots produced in [a, b] read after b or output
  std::map<int, int> last_read_step;
  for (size_t s = 0; s < plan.steps.size(); ++s)
    for (const auto& in : plan.steps[s].instrs)
      for (int x : in.inputs) last_read_step[x] = static_cast<int>(s);
  std::set<int> plan_outputs;
  for (const auto& o : plan.outputs) plan_outputs.insert(o.slot);
  int next_free = 0;
  for (size_t s = 0; s < plan.steps.size(); ++s) {
    if (A.rels[s].kind != Rel::AGG || static_cast<int>(s) < next_free) continue;
    Planner pl(A, plan);
    if (!pl.plan_agg(static_cast<int>(s))) {
      if (std::getenv("TQP_FUSION_DEBUG")) std::fprintf(stderr, "[tqp] no fusion at %s: %s\n", plan.steps[s].id.c_str(), pl.why.c_str());
      continue;
    }
    PipeDesc& P = pl.P;
    if (P.first_step < next_free) continue;
    // every slot produced inside the unit and needed later must be produced
    // by the unit
    std::set<int> provided(P.final_slots.begin(), P.final_slots.end());
    bool ok = true;
    for (int q = P.first_step; q <= P.last_step && ok; ++q) {
      for (const auto& in : plan.steps[q].instrs) {
        int x = in.output;
        bool needed = plan_outputs.count(x) || (last_read_step.count(x) && last_read_step[x] > P.last_step);
        if (needed && !provided.count(x)) ok = false;
      }
      // project steps without instructions pass slots through
      for (int x : plan.steps[q].output_slots) {
        bool needed = plan_outputs.count(x) || (last_read_step.count(x) && last_read_step[x] > P.last_step);
        if (needed && !provided.count(x)) ok = false;
      }
    }
    if (!ok) continue;
    std::ostringstream ex;
    const char* mode = P.mode == MODE_SCALAR  ? "scalar"
                       : P.mode == MODE_SMALL ? "small-group"
                       : P.mode == MODE_HASH  ? "hash-group"
                                              : "build-group";
    ex << "fact=" << P.fact_table << " terms=" << P.terms.size() << " probes=" << P.probes.size()
       << " builds=" << P.builds.size() << " accumulators=" << P.accs.size() << " mode=" << mode
       << (P.topk ? " topk=" + std::to_string(P.k) : std::string());
    FusedUnit u;
    u.first_step = P.first_step;
    u.last_step = P.last_step;
    u.name = std::string("fused_") + (P.probes.empty() ? "scan_" : "probe_") + mode + (P.topk ? "_topk" : "");
    u.explain = ex.str();
    auto R = std::make_shared<Runner>(Runner{P});
    if ((P.mode == MODE_SMALL && P.hash_alt) || (P.mode == MODE_BUILDGRP && !P.hkeys.empty())) {
      // the hash-group unit a small-group overflow or a build-group unit whose
      // group build meets repeated keys (or unconvertible values) reruns as
      PipeDesc H = P;
      H.mode = MODE_HASH;
      H.key_columns.clear();
      H.group_key_root_columns.clear();
      if (P.mode == MODE_BUILDGRP) H.builds[H.probes[H.group_probe].build].assign_groups = false;
      H.group_probe = -1;
      R->alt = std::make_shared<const Runner>(Runner{H});
    }
    u.run = [R](Ctx& c, std::vector<std::optional<Tensor>>& slots, const TableSet& t, UnitPending* pend) {
      return (*R)(c, slots, t, pend);
    };
    u.partial = [R](Ctx& c, const TableSet& t, Partial* out) { return R->run(c, nullptr, t, out); };
    const std::string where = plan.steps[P.last_step].id;
    u.finish = [R, where](Ctx& c, std::vector<std::optional<Tensor>>& slots, const std::vector<PartRef>& parts) {
      R->finish(c, slots, parts, where);
    };
    units.push_back(std::move(u));
    next_free = P.last_step + 1;
  }
  return units;
}

}  // namespace tqp
