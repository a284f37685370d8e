// Fused relational pipelines on B200 (sm_100a), HBM-bound.
//
// One pass over the fact table evaluates a conjunctive predicate in
// registers, probes unique-key build sides through dense direct-address
// tables (L2-resident), evaluates the aggregate expressions and accumulates:
//   MODE_SCALAR  : no group keys (Q6, Q14) - per-thread fp64/int64 registers,
//                  fixed-order warp/CTA trees, per-CTA partials merged in CTA
//                  order (run-to-run deterministic);
//   MODE_SMALL   : <= 64 groups keyed by up to four 1-byte string columns (Q1)
//                  - warp-aggregated per-warp shared-memory tables
//                  (__match_any-free ballot loop, deterministic order),
//                  per-CTA partials merged by key in CTA order;
//   MODE_BUILDGRP: the group is the matched build row (Q3: l_orderkey =
//                  o_orderkey, o_orderdate/o_shippriority functionally
//                  dependent) - global atomics on exact Q64.64 fixed-point
//                  sums (two u64 atomics with carry; order-independent, so
//                  deterministic and GPU-count invariant).
// Loads are 128-bit (two consecutive rows per thread) and go through the
// read-only path; an operand repeated across terms/aggregates hits L1.
#pragma once

#include "device.cuh"

namespace tqp {
namespace fz {

constexpr int kMaxTerms = 8;
constexpr int kMaxProbes = 3;
constexpr int kMaxAcc = 8;
constexpr int kMaxFactors = 4;
constexpr int kMaxKeys = 4;
constexpr int kMaxStrTerms = 4;
constexpr int kMaxFlags = 7;
constexpr int kGroups = 64;  // MODE_SMALL per-CTA slot capacity
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

enum OperandType : int { OT_I64 = 0, OT_F64 = 1, OT_U8 = 2 };
enum TermKind : int { TK_INT = 0, TK_F64 = 1, TK_TRUE = 2, TK_FALSE = 3 };
enum FactorKind : int { FK_X = 0, FK_K_MINUS_X, FK_K_PLUS_X, FK_X_MINUS_K, FK_X_PLUS_K, FK_X_TIMES_K, FK_CONST };
enum Mode : int { MODE_SCALAR = 0, MODE_SMALL = 1, MODE_BUILDGRP = 2 };

// A per-row operand: fact column (src = -1) or a column of the build-side
// root row matched by probe `src`.
struct Operand {
  const void* ptr = nullptr;
  int type = OT_I64;
  int src = -1;
};

struct Term {
  Operand x;
  int kind = TK_TRUE;
  int op = TQP_EQ;
  long long ik = 0;
  double fk = 0.0;
};

// string predicate over STR8 rows: compare with a literal (zero-extended, as
// string_compare_rows, executor.cpp:72-108) or LIKE (substring_match,
// kernels.cpp:692-728)
struct StrTerm {
  const uint8_t* ptr = nullptr;
  int width = 1;
  int is_like = 0;
  int op = TQP_EQ;      // compare op when !is_like
  int anchor = TQP_START;
  int litlen = 0;
  unsigned char lit[48];
};

struct Factor {
  Operand x;
  int kind = FK_X;
  double k = 0.0;
};

struct Acc {
  int is_int = 0;
  int nf = 0;
  Factor f[kMaxFactors];
  int gate_probe = -1;  // value counts only if flag bit of probe is set
  int gate_bit = 0;
  double gate_else = 0.0;
};

// dense direct-address build table: entry 0 = empty, else
//   bits 0-31 rowid+1 | bits 32-56 group id | bits 57-63 flags
struct Probe {
  Operand key;
  long long kmin = 0;
  long long range = 0;
  const unsigned long long* table = nullptr;
};

struct ProbeSpec {
  long long n = 0;
  int nterms = 0;
  Term terms[kMaxTerms];
  int nprobes = 0;
  Probe probes[kMaxProbes];
  int nacc = 0;
  Acc acc[kMaxAcc];
  int nkeys = 0;
  Operand keys[kMaxKeys];  // MODE_SMALL: 1-byte string columns (fact)
  int group_probe = -1;    // MODE_BUILDGRP
  // outputs
  unsigned long long* part;  // SCALAR: [cta][nacc+1]; SMALL: per-CTA tables
  unsigned long long* gacc;  // BUILDGRP: [group][nacc] x 2 words (Q64.64 or int64)
  unsigned long long* gcnt;  // BUILDGRP: [group]
  long long* err;            // [0] != 0: data violates the fused preconditions
};

struct BuildSpec {
  long long n = 0;
  int nterms = 0;
  Term terms[kMaxTerms];
  int nstr = 0;
  StrTerm str[kMaxStrTerms];
  int nprobes = 0;
  Probe probes[kMaxProbes];
  int nflags = 0;
  StrTerm flags[kMaxFlags];
  Operand key;  // root key column (int64)
  long long kmin = 0;
  long long range = 0;
  unsigned long long* table = nullptr;
  int assign_groups = 0;
  unsigned int* group_counter = nullptr;
  int* group_row = nullptr;
  long long* err = nullptr;
};

// ---- operand access ----------------------------------------------------------
__device__ __forceinline__ long long ld_i64(const void* p, long long r) {
  return __ldg(static_cast<const long long*>(p) + r);
}
__device__ __forceinline__ double ld_f64(const void* p, long long r) {
  return __ldg(static_cast<const double*>(p) + r);
}

// two consecutive fact rows (row0 even) with one 128-bit load
__device__ __forceinline__ void ld_pair(const Operand& o, long long row0, unsigned long long& a,
                                        unsigned long long& b) {
  if (o.type == OT_U8) {
    unsigned short v = __ldg(reinterpret_cast<const unsigned short*>(static_cast<const uint8_t*>(o.ptr) + row0));
    a = v & 0xff;
    b = v >> 8;
  } else {
    ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(static_cast<const unsigned long long*>(o.ptr) + row0));
    a = v.x;
    b = v.y;
  }
}

__device__ __forceinline__ unsigned long long ld_row(const Operand& o, long long row) {
  if (o.type == OT_U8) return __ldg(static_cast<const uint8_t*>(o.ptr) + row);
  return __ldg(static_cast<const unsigned long long*>(o.ptr) + row);
}

template <typename T>
__device__ __forceinline__ bool cmp_op(T x, T y, int op) {
  switch (op) {
    case TQP_EQ: return x == y;
    case TQP_NE: return x != y;
    case TQP_LT: return x < y;
    case TQP_LE: return x <= y;
    case TQP_GT: return x > y;
    default: return x >= y;
  }
}

__device__ __forceinline__ bool eval_term(const Term& t, unsigned long long raw) {
  switch (t.kind) {
    case TK_INT: return cmp_op<long long>(static_cast<long long>(raw), t.ik, t.op);
    case TK_F64: return cmp_op<double>(__longlong_as_double(static_cast<long long>(raw)), t.fk, t.op);
    case TK_TRUE: return true;
    default: return false;
  }
}

__device__ __forceinline__ bool eval_str(const StrTerm& s, long long row) {
  const uint8_t* p = s.ptr + row * s.width;
  int len = 0;
  while (len < s.width && p[len] != 0) ++len;
  if (s.is_like) {
    int pl = s.litlen;
    if (pl > len) return false;
    auto at = [&](int off) {
      for (int j = 0; j < pl; ++j)
        if (p[off + j] != s.lit[j]) return false;
      return true;
    };
    switch (s.anchor) {
      case TQP_START: return at(0);
      case TQP_END: return at(len - pl);
      case TQP_ANY:
        for (int o = 0; o + pl <= len; ++o)
          if (at(o)) return true;
        return false;
      default: return len == pl && at(0);
    }
  }
  int m = s.width > s.litlen ? s.width : s.litlen;
  int c = 0;
  for (int j = 0; j < m && c == 0; ++j) {
    int x = j < s.width ? p[j] : 0;
    int y = j < s.litlen ? s.lit[j] : 0;
    if (x != y) c = x < y ? -1 : 1;
  }
  return cmp_op<int>(c, 0, s.op);
}

__device__ __forceinline__ double apply_factor(const Factor& f, double x) {
  switch (f.kind) {
    case FK_X: return x;
    case FK_K_MINUS_X: return __dsub_rn(f.k, x);
    case FK_K_PLUS_X: return __dadd_rn(f.k, x);
    case FK_X_MINUS_K: return __dsub_rn(x, f.k);
    case FK_X_PLUS_K: return __dadd_rn(x, f.k);
    case FK_X_TIMES_K: return __dmul_rn(x, f.k);
    default: return f.k;
  }
}

struct RowCtx {
  long long rid[kMaxProbes];
  unsigned flags[kMaxProbes];
  unsigned gid[kMaxProbes];
};

__device__ __forceinline__ bool probe_lookup(const Probe& p, long long key, long long& rid, unsigned& flags,
                                             unsigned& gid) {
  long long idx = key - p.kmin;
  if (idx < 0 || idx >= p.range) return false;
  unsigned long long e = __ldg(p.table + idx);
  if (!e) return false;
  rid = static_cast<long long>(e & 0xffffffffULL) - 1;
  gid = static_cast<unsigned>((e >> 32) & 0x1ffffffULL);
  flags = static_cast<unsigned>(e >> 57);
  return true;
}

__device__ __forceinline__ unsigned long long operand_value(const Operand& o, unsigned long long fact_raw,
                                                            const RowCtx& rc) {
  if (o.src < 0) return fact_raw;
  return ld_row(o, rc.rid[o.src]);
}

// value of accumulator a for one row; fact operands already loaded in fv[]
__device__ __forceinline__ unsigned long long eval_acc(const Acc& a, const unsigned long long* fv, const RowCtx& rc) {
  if (a.is_int) return operand_value(a.f[0].x, fv[0], rc);
  double v = 0.0;
#pragma unroll
  for (int i = 0; i < kMaxFactors; ++i) {
    if (i < a.nf) {
      double x = __longlong_as_double(static_cast<long long>(operand_value(a.f[i].x, fv[i], rc)));
      double y = apply_factor(a.f[i], x);
      v = i == 0 ? y : __dmul_rn(v, y);
    }
  }
  if (a.gate_probe >= 0 && !((rc.flags[a.gate_probe] >> a.gate_bit) & 1u)) v = a.gate_else;
  return static_cast<unsigned long long>(__double_as_longlong(v));
}

// ---- exact Q64.64 fixed point ----------------------------------------------------
// x -> round-toward-zero(x * 2^64) as int128. Exact for |x| >= 2^-11 (every
// money value); false for |x| >= 2^62, NaN, Inf.
__device__ __forceinline__ bool f64_to_q64(double x, __int128& out) {
  long long bits = __double_as_longlong(x);
  int ex = static_cast<int>((bits >> 52) & 0x7ff);
  if (ex == 0x7ff) return false;
  unsigned long long mant = static_cast<unsigned long long>(bits) & ((1ULL << 52) - 1);
  if (ex == 0) {
    ex = 1;
  } else {
    mant |= 1ULL << 52;
  }
  int shift = ex - 1075 + 64;
  unsigned __int128 v;
  if (shift >= 0) {
    if (shift > 73) return false;
    v = static_cast<unsigned __int128>(mant) << shift;
  } else if (shift > -64) {
    v = static_cast<unsigned __int128>(mant >> (-shift));
  } else {
    v = 0;
  }
  out = bits < 0 ? -static_cast<__int128>(v) : static_cast<__int128>(v);
  return true;
}

__device__ __forceinline__ double q64_to_f64(unsigned long long lo, unsigned long long hi) {
  __int128 v = static_cast<__int128>((static_cast<unsigned __int128>(hi) << 64) | lo);
  bool neg = v < 0;
  unsigned __int128 u = neg ? static_cast<unsigned __int128>(-v) : static_cast<unsigned __int128>(v);
  double ip = static_cast<double>(static_cast<unsigned long long>(u >> 64));
  double fp = static_cast<double>(static_cast<unsigned long long>(u)) * 5.421010862427522e-20;  // 2^-64
  double r = ip + fp;
  return neg ? -r : r;
}

__device__ __forceinline__ void atomic_add_q64(unsigned long long* p, __int128 v) {
  unsigned long long lo = static_cast<unsigned long long>(v);
  unsigned long long hi = static_cast<unsigned long long>(static_cast<unsigned __int128>(v) >> 64);
  unsigned long long old = atomicAdd(p, lo);
  unsigned long long carry = (old + lo < old) ? 1ULL : 0ULL;
  atomicAdd(p + 1, hi + carry);
}

// ---- build kernel ------------------------------------------------------------
__global__ void k_minmax(const long long* __restrict__ k, long long n, long long* out) {
  long long mn = 0x7fffffffffffffffLL, mx = static_cast<long long>(0x8000000000000000ULL);
  for (long long i = gtid(); i < n; i += gstride()) {
    long long v = k[i];
    mn = v < mn ? v : mn;
    mx = v > mx ? v : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    long long a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, mn);
    atomicMax(out + 1, mx);
  }
}

__global__ void __launch_bounds__(kThreads) k_build(const BuildSpec s) {
  for (long long r = gtid(); r < s.n; r += gstride()) {
    bool pass = true;
#pragma unroll
    for (int t = 0; t < kMaxTerms; ++t)
      if (t < s.nterms && pass) pass = eval_term(s.terms[t], ld_row(s.terms[t].x, r));
#pragma unroll
    for (int t = 0; t < kMaxStrTerms; ++t)
      if (t < s.nstr && pass) pass = eval_str(s.str[t], r);
#pragma unroll
    for (int p = 0; p < kMaxProbes; ++p) {
      if (p < s.nprobes && pass) {
        long long rid;
        unsigned fl, g;
        pass = probe_lookup(s.probes[p], static_cast<long long>(ld_row(s.probes[p].key, r)), rid, fl, g);
      }
    }
    if (!pass) continue;
    unsigned flags = 0;
#pragma unroll
    for (int f = 0; f < kMaxFlags; ++f)
      if (f < s.nflags && eval_str(s.flags[f], r)) flags |= 1u << f;
    long long key = static_cast<long long>(ld_row(s.key, r));
    long long idx = key - s.kmin;
    if (idx < 0 || idx >= s.range) {
      atomicExch(reinterpret_cast<unsigned long long*>(s.err), 1ULL);
      continue;
    }
    unsigned gid = 0;
    if (s.assign_groups) {
      gid = atomicAdd(s.group_counter, 1u);
      if (gid >= (1u << 25)) {
        atomicExch(reinterpret_cast<unsigned long long*>(s.err), 1ULL);
        continue;
      }
      s.group_row[gid] = static_cast<int>(r);
    }
    unsigned long long e = static_cast<unsigned long long>(r + 1) | (static_cast<unsigned long long>(gid) << 32) |
                           (static_cast<unsigned long long>(flags) << 57);
    if (atomicCAS(s.table + idx, 0ULL, e) != 0ULL) {
      // duplicate build key: the join is 1:N, outside the fused contract
      atomicExch(reinterpret_cast<unsigned long long*>(s.err), 1ULL);
    }
  }
}

// ---- probe + aggregate kernel ------------------------------------------------
// per row: predicate, probes; returns pass and fills rc
__device__ __forceinline__ void row_filter_probe(const ProbeSpec& s, const unsigned long long (*tv)[2], long long row0,
                                                 bool pass[2], RowCtx rc[2]) {
#pragma unroll
  for (int t = 0; t < kMaxTerms; ++t) {
    if (t < s.nterms) {
      pass[0] = pass[0] && eval_term(s.terms[t], tv[t][0]);
      pass[1] = pass[1] && eval_term(s.terms[t], tv[t][1]);
    }
  }
#pragma unroll
  for (int p = 0; p < kMaxProbes; ++p) {
    if (p < s.nprobes && (pass[0] || pass[1])) {
      unsigned long long k0, k1;
      ld_pair(s.probes[p].key, row0, k0, k1);
      if (pass[0]) pass[0] = probe_lookup(s.probes[p], static_cast<long long>(k0), rc[0].rid[p], rc[0].flags[p], rc[0].gid[p]);
      if (pass[1]) pass[1] = probe_lookup(s.probes[p], static_cast<long long>(k1), rc[1].rid[p], rc[1].flags[p], rc[1].gid[p]);
    }
  }
}

__device__ __forceinline__ void load_terms(const ProbeSpec& s, long long row0, unsigned long long (*tv)[2]) {
#pragma unroll
  for (int t = 0; t < kMaxTerms; ++t)
    if (t < s.nterms && s.terms[t].kind <= TK_F64) ld_pair(s.terms[t].x, row0, tv[t][0], tv[t][1]);
}

// fact operands of accumulator a for both rows
__device__ __forceinline__ void load_acc_operands(const Acc& a, long long row0, unsigned long long (*fv)[kMaxFactors]) {
#pragma unroll
  for (int i = 0; i < kMaxFactors; ++i) {
    if (i < (a.is_int ? 1 : a.nf) && a.f[i].x.src < 0 && a.f[i].kind != FK_CONST) {
      ld_pair(a.f[i].x, row0, fv[0][i], fv[1][i]);
    } else {
      fv[0][i] = fv[1][i] = 0;
    }
  }
}

template <typename T>
__device__ __forceinline__ T shfl_xor_u64(T v, int o) {
  return __shfl_xor_sync(0xffffffffu, v, o);
}

__global__ void __launch_bounds__(kThreads) k_probe_scalar(const ProbeSpec s) {
  __shared__ unsigned long long s_part[kWarps][kMaxAcc + 1];
  unsigned long long acc[kMaxAcc];
  long long absmax[kMaxAcc];
#pragma unroll
  for (int a = 0; a < kMaxAcc; ++a) {
    acc[a] = 0;  // 0.0 and 0 share the bit pattern
    absmax[a] = 0;
  }
  long long cnt = 0;
  const long long npairs = (s.n + 1) / 2;
  for (long long q = gtid(); q < npairs; q += gstride()) {
    const long long row0 = 2 * q;
    bool pass[2] = {true, row0 + 1 < s.n};
    unsigned long long tv[kMaxTerms][2];
    load_terms(s, row0, tv);
    RowCtx rc[2];
    row_filter_probe(s, tv, row0, pass, rc);
    if (!pass[0] && !pass[1]) continue;
#pragma unroll
    for (int a = 0; a < kMaxAcc; ++a) {
      if (a < s.nacc) {
        unsigned long long fv[2][kMaxFactors];
        load_acc_operands(s.acc[a], row0, fv);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          if (!pass[r]) continue;
          unsigned long long v = eval_acc(s.acc[a], fv[r], rc[r]);
          if (s.acc[a].is_int) {
            long long iv = static_cast<long long>(v);
            acc[a] = static_cast<unsigned long long>(static_cast<long long>(acc[a]) + iv);
            long long av = iv < 0 ? -iv : iv;
            absmax[a] = av > absmax[a] ? av : absmax[a];
          } else {
            acc[a] = static_cast<unsigned long long>(
                __double_as_longlong(__dadd_rn(__longlong_as_double(static_cast<long long>(acc[a])),
                                               __longlong_as_double(static_cast<long long>(v)))));
          }
        }
      }
    }
    cnt += (pass[0] ? 1 : 0) + (pass[1] ? 1 : 0);
  }
  // fixed-order warp tree, then warps in order
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int a = 0; a < kMaxAcc; ++a) {
    if (a < s.nacc) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        unsigned long long y = shfl_xor_u64(acc[a], o);
        long long am = shfl_xor_u64(absmax[a], o);
        absmax[a] = am > absmax[a] ? am : absmax[a];
        if (s.acc[a].is_int) {
          acc[a] = static_cast<unsigned long long>(static_cast<long long>(acc[a]) + static_cast<long long>(y));
        } else {
          acc[a] = static_cast<unsigned long long>(__double_as_longlong(
              __dadd_rn(__longlong_as_double(static_cast<long long>(acc[a])), __longlong_as_double(static_cast<long long>(y)))));
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) {
#pragma unroll
    for (int a = 0; a < kMaxAcc; ++a)
      if (a < s.nacc) s_part[warp][a] = acc[a];
    s_part[warp][kMaxAcc] = static_cast<unsigned long long>(cnt);
    // int64 sums may not be exact if |v| * count can reach 2^63 (the
    // reference errors on the first overflowing prefix): hand over to the
    // exact per-instruction path
#pragma unroll
    for (int a = 0; a < kMaxAcc; ++a) {
      if (a < s.nacc && s.acc[a].is_int && absmax[a] > 0 && cnt > 0 &&
          static_cast<double>(absmax[a]) * static_cast<double>(s.n) >= 9.0e18) {
        atomicExch(reinterpret_cast<unsigned long long*>(s.err), 1ULL);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long* out = s.part + static_cast<long long>(blockIdx.x) * (kMaxAcc + 1);
    for (int a = 0; a < s.nacc; ++a) {
      unsigned long long t = s_part[0][a];
      for (int w = 1; w < kWarps; ++w) {
        if (s.acc[a].is_int) {
          t = static_cast<unsigned long long>(static_cast<long long>(t) + static_cast<long long>(s_part[w][a]));
        } else {
          t = static_cast<unsigned long long>(__double_as_longlong(__dadd_rn(
              __longlong_as_double(static_cast<long long>(t)), __longlong_as_double(static_cast<long long>(s_part[w][a])))));
        }
      }
      out[a] = t;
    }
    unsigned long long c = 0;
    for (int w = 0; w < kWarps; ++w) c += s_part[w][kMaxAcc];
    out[kMaxAcc] = c;
  }
}

// MODE_SMALL: per-CTA hash of group codes -> slot, per-warp accumulators.
struct SmallPart {  // per CTA, in global memory
  unsigned int ncodes;
  unsigned int codes[kGroups];
  unsigned long long cnt[kGroups];
  unsigned long long acc[kGroups][kMaxAcc];
};

__device__ __forceinline__ unsigned hash_code(unsigned c) { return (c * 2654435761u) >> 26; }  // 6 bits

__global__ void __launch_bounds__(kThreads) k_probe_small(const ProbeSpec s) {
  __shared__ unsigned int s_codes[kGroups];
  __shared__ unsigned long long s_acc[kWarps][kGroups][kMaxAcc];
  __shared__ unsigned long long s_cnt[kWarps][kGroups];
  __shared__ int s_overflow;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kGroups; i += blockDim.x) s_codes[i] = 0xffffffffu;
  for (int i = threadIdx.x; i < kWarps * kGroups * kMaxAcc; i += blockDim.x) (&s_acc[0][0][0])[i] = 0;
  for (int i = threadIdx.x; i < kWarps * kGroups; i += blockDim.x) (&s_cnt[0][0])[i] = 0;
  if (threadIdx.x == 0) s_overflow = 0;
  __syncthreads();
  long long absmax[kMaxAcc];
#pragma unroll
  for (int a = 0; a < kMaxAcc; ++a) absmax[a] = 0;

  const long long npairs = (s.n + 1) / 2;
  const long long wstride = gstride();
  // warp-uniform trip count
  for (long long base = (gtid() & ~31LL); base < npairs; base += wstride) {
    const long long q = base + lane;
    const long long row0 = 2 * q;
    bool pass[2] = {q < npairs, q < npairs && row0 + 1 < s.n};
    unsigned long long tv[kMaxTerms][2];
    RowCtx rc[2];
    if (pass[0]) {
      load_terms(s, row0, tv);
      row_filter_probe(s, tv, row0, pass, rc);
    }
    // group codes (big-endian over the key bytes: numeric order = key order)
    unsigned code[2] = {0, 0};
#pragma unroll
    for (int k = 0; k < kMaxKeys; ++k) {
      if (k < s.nkeys && (pass[0] || pass[1])) {
        unsigned long long b0, b1;
        ld_pair(s.keys[k], row0, b0, b1);
        code[0] = (code[0] << 8) | static_cast<unsigned>(b0);
        code[1] = (code[1] << 8) | static_cast<unsigned>(b1);
      }
    }
    unsigned long long val[2][kMaxAcc];
#pragma unroll
    for (int a = 0; a < kMaxAcc; ++a) {
      if (a < s.nacc) {
        unsigned long long fv[2][kMaxFactors];
        if (pass[0] || pass[1]) load_acc_operands(s.acc[a], row0, fv);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          val[r][a] = pass[r] ? eval_acc(s.acc[a], fv[r], rc[r]) : 0ULL;
          if (pass[r] && s.acc[a].is_int) {
            long long iv = static_cast<long long>(val[r][a]);
            iv = iv < 0 ? -iv : iv;
            absmax[a] = iv > absmax[a] ? iv : absmax[a];
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      // slot lookup / insert
      int slot = -1;
      if (pass[r]) {
        unsigned h = hash_code(code[r]);
        for (int probe = 0; probe < kGroups; ++probe) {
          unsigned cur = s_codes[h];
          if (cur == code[r]) {
            slot = static_cast<int>(h);
            break;
          }
          if (cur == 0xffffffffu) {
            unsigned prev = atomicCAS(&s_codes[h], 0xffffffffu, code[r]);
            if (prev == 0xffffffffu || prev == code[r]) {
              slot = static_cast<int>(h);
              break;
            }
          }
          h = (h + 1) & (kGroups - 1);
        }
        if (slot < 0) s_overflow = 1;
      }
      // ballot loop over the distinct slots present in this warp batch
      unsigned todo = __ballot_sync(0xffffffffu, slot >= 0);
      while (todo) {
        const int leader = __ffs(todo) - 1;
        const int sl = __shfl_sync(0xffffffffu, slot, leader);
        const bool mine = slot == sl;
        const unsigned members = __ballot_sync(0xffffffffu, mine);
#pragma unroll
        for (int a = 0; a < kMaxAcc; ++a) {
          if (a < s.nacc) {
            unsigned long long x = mine ? val[r][a] : 0ULL;  // 0.0 == bits 0
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              unsigned long long y = __shfl_xor_sync(0xffffffffu, x, o);
              if (s.acc[a].is_int) {
                x = static_cast<unsigned long long>(static_cast<long long>(x) + static_cast<long long>(y));
              } else {
                x = static_cast<unsigned long long>(__double_as_longlong(
                    __dadd_rn(__longlong_as_double(static_cast<long long>(x)), __longlong_as_double(static_cast<long long>(y)))));
              }
            }
            if (lane == 0) {
              unsigned long long& dst = s_acc[warp][sl][a];
              if (s.acc[a].is_int) {
                dst = static_cast<unsigned long long>(static_cast<long long>(dst) + static_cast<long long>(x));
              } else {
                dst = static_cast<unsigned long long>(__double_as_longlong(
                    __dadd_rn(__longlong_as_double(static_cast<long long>(dst)), __longlong_as_double(static_cast<long long>(x)))));
              }
            }
          }
        }
        if (lane == 0) s_cnt[warp][sl] += __popc(members);
        todo &= ~members;
      }
    }
  }
  // int64 exactness guard (see k_probe_scalar)
#pragma unroll
  for (int a = 0; a < kMaxAcc; ++a) {
    if (a < s.nacc && s.acc[a].is_int && static_cast<double>(absmax[a]) * static_cast<double>(s.n) >= 9.0e18) {
      atomicExch(reinterpret_cast<unsigned long long*>(s.err), 1ULL);
    }
  }
  __syncthreads();
  if (s_overflow && threadIdx.x == 0) atomicExch(reinterpret_cast<unsigned long long*>(s.err), 1ULL);
  // CTA partial: warps merged in warp order
  SmallPart* out = reinterpret_cast<SmallPart*>(s.part) + blockIdx.x;
  for (int sl = threadIdx.x; sl < kGroups; sl += blockDim.x) {
    out->codes[sl] = s_codes[sl];
    unsigned long long c = 0;
    for (int w = 0; w < kWarps; ++w) c += s_cnt[w][sl];
    out->cnt[sl] = c;
    for (int a = 0; a < s.nacc; ++a) {
      unsigned long long t = s_acc[0][sl][a];
      for (int w = 1; w < kWarps; ++w) {
        if (s.acc[a].is_int) {
          t = static_cast<unsigned long long>(static_cast<long long>(t) + static_cast<long long>(s_acc[w][sl][a]));
        } else {
          t = static_cast<unsigned long long>(__double_as_longlong(__dadd_rn(
              __longlong_as_double(static_cast<long long>(t)), __longlong_as_double(static_cast<long long>(s_acc[w][sl][a])))));
        }
      }
      out->acc[sl][a] = t;
    }
  }
}

// MODE_BUILDGRP: exact fixed-point atomics per matched build row
__global__ void __launch_bounds__(kThreads) k_probe_buildgrp(const ProbeSpec s) {
  const long long npairs = (s.n + 1) / 2;
  for (long long q = gtid(); q < npairs; q += gstride()) {
    const long long row0 = 2 * q;
    bool pass[2] = {true, row0 + 1 < s.n};
    unsigned long long tv[kMaxTerms][2];
    load_terms(s, row0, tv);
    RowCtx rc[2];
    row_filter_probe(s, tv, row0, pass, rc);
    if (!pass[0] && !pass[1]) continue;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (!pass[r]) continue;
      const unsigned g = rc[r].gid[s.group_probe];
      atomicAdd(s.gcnt + g, 1ULL);
#pragma unroll
      for (int a = 0; a < kMaxAcc; ++a) {
        if (a < s.nacc) {
          unsigned long long fv[kMaxFactors];
#pragma unroll
          for (int i = 0; i < kMaxFactors; ++i) {
            fv[i] = (i < (s.acc[a].is_int ? 1 : s.acc[a].nf) && s.acc[a].f[i].x.src < 0 && s.acc[a].f[i].kind != FK_CONST)
                        ? ld_row(s.acc[a].f[i].x, row0 + r)
                        : 0ULL;
          }
          unsigned long long v = eval_acc(s.acc[a], fv, rc[r]);
          unsigned long long* dst = s.gacc + (static_cast<long long>(g) * s.nacc + a) * 2;
          if (s.acc[a].is_int) {
            long long iv = static_cast<long long>(v);
            atomic_add_q64(dst, static_cast<__int128>(iv));
          } else {
            __int128 qv;
            if (!f64_to_q64(__longlong_as_double(static_cast<long long>(v)), qv)) {
              atomicExch(reinterpret_cast<unsigned long long*>(s.err), 1ULL);
              qv = 0;
            }
            atomic_add_q64(dst, qv);
          }
        }
      }
    }
  }
}

}  // namespace fz
}  // namespace tqp
