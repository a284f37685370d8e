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
#include "fz_layout.cuh"
#include "scan.cuh"

namespace tqp {
namespace fz {

// ---- build kernel ------------------------------------------------------------
// Does a key column repeat a value? One pass setting a bit per key over its
// (known) range; a bit already set flags the column (*dup = 1). Run once per
// column, the first time a direct-addressed build keys on it (KeyRange::unique).
__global__ void __launch_bounds__(256) k_key_unique(const long long* __restrict__ k, long long n, long long kmin,
                                                    unsigned* __restrict__ bits, int* __restrict__ dup) {
  bool rep = false;
  for (long long i = gtid(); i < n; i += gstride()) {
    const unsigned long long idx = static_cast<unsigned long long>(__ldg(k + i) - kmin);
    const unsigned b = 1u << (idx & 31);
    rep = rep || (atomicOr(bits + (idx >> 5), b) & b) != 0u;
  }
  if (__any_sync(0xffffffffu, rep) && (threadIdx.x & 31) == 0) atomicExch(dup, 1);
}

// key range of a build side: 128-bit loads, warp then block reduction, one
// atomic pair per block (a per-warp atomic on one address serialises at L2)
// DAY: also out[2] |= 1 if a value is not a whole number of days in ns (a
// Date column keyed by day digits, MODE_HASH)
template <bool DAY = false>
__global__ void __launch_bounds__(256) k_minmax(const long long* __restrict__ k, long long n, long long* out) {
  __shared__ long long s_mn[8], s_mx[8];
  long long mn = 0x7fffffffffffffffLL, mx = static_cast<long long>(0x8000000000000000ULL);
  bool odd = false;
  constexpr long long kDay = 86400000000000LL;
  const bool aligned = (reinterpret_cast<uintptr_t>(k) & 15) == 0;
  const long long npair = aligned ? n / 2 : 0;
  const longlong2* k2 = reinterpret_cast<const longlong2*>(k);
  for (long long i = gtid(); i < npair; i += gstride()) {
    const longlong2 v = __ldg(k2 + i);
    mn = min(mn, min(v.x, v.y));
    mx = max(mx, max(v.x, v.y));
    if (DAY) odd = odd || (v.x % kDay) != 0 || (v.y % kDay) != 0;
  }
  for (long long i = 2 * npair + gtid(); i < n; i += gstride()) {
    const long long v = __ldg(k + i);
    mn = min(mn, v);
    mx = max(mx, v);
    if (DAY) odd = odd || (v % kDay) != 0;
  }
  if (DAY && __any_sync(0xffffffffu, odd) && (threadIdx.x & 31) == 0) atomicOr(reinterpret_cast<unsigned long long*>(out + 2), 1ULL);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    s_mn[warp] = mn;
    s_mx[warp] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
      mn = min(mn, s_mn[w]);
      mx = max(mx, s_mx[w]);
    }
    atomicMin(out, mn);
    atomicMax(out + 1, mx);
  }
}

constexpr int kBuildRows = 4;
__global__ void __launch_bounds__(kThreads) k_build(const BuildSpec s) {
  unsigned dup = 0;
  // kBuildRows rows per thread (stride blockDim) with every independent column
  // load issued before any dependent work: the per-row chain (filter ->
  // child probe -> insert) is latency-bound otherwise
  const long long span = static_cast<long long>(blockDim.x) * kBuildRows;
  for (long long base0 = static_cast<long long>(blockIdx.x) * span; base0 < s.n; base0 += static_cast<long long>(gridDim.x) * span) {
    bool pass[kBuildRows];
    long long key[kBuildRows], pk[kBuildRows][kMaxProbes];
#pragma unroll
    for (int j = 0; j < kBuildRows; ++j) {
      const long long r = base0 + j * blockDim.x + threadIdx.x;
      pass[j] = r < s.n;
      key[j] = pass[j] ? static_cast<long long>(ld_row(s.key, r)) : 0;
#pragma unroll
      for (int p = 0; p < kMaxProbes; ++p)
        pk[j][p] = (p < s.nprobes && pass[j]) ? static_cast<long long>(ld_row(s.probes[p].key, r)) : 0;
    }
#pragma unroll
    for (int t = 0; t < kMaxTerms; ++t) {
      if (t < s.nterms) {
        unsigned long long v[kBuildRows];
#pragma unroll
        for (int j = 0; j < kBuildRows; ++j) {
          const long long r = base0 + j * blockDim.x + threadIdx.x;
          // constant terms (TK_TRUE / TK_FALSE) have no column
          v[j] = pass[j] && s.terms[t].kind <= TK_F64 ? ld_row(s.terms[t].x, r) : 0ULL;
        }
#pragma unroll
        for (int j = 0; j < kBuildRows; ++j) pass[j] = pass[j] && eval_term(s.terms[t], v[j]);
      }
    }
    for (int t = 0; t < s.nstr; ++t)
#pragma unroll
      for (int j = 0; j < kBuildRows; ++j)
        if (pass[j]) pass[j] = eval_str(s.str[t], base0 + j * blockDim.x + threadIdx.x);
    unsigned wgt[kBuildRows];  // row weight: product of the child probes' multiplicities
#pragma unroll
    for (int j = 0; j < kBuildRows; ++j) wgt[j] = 1u;
#pragma unroll
    for (int p = 0; p < kMaxProbes; ++p) {
      if (p < s.nprobes) {
#pragma unroll
        for (int j = 0; j < kBuildRows; ++j) {
          long long rid;
          unsigned fl, g, m = 1u;
          if (pass[j]) pass[j] = probe_lookup(s.probes[p], pk[j][p], rid, fl, g, &m);
          wgt[j] *= m;
        }
      }
    }
    unsigned old[kBuildRows], set[kBuildRows];
#pragma unroll
    for (int j = 0; j < kBuildRows; ++j) {
      old[j] = set[j] = 0u;
      if (!__any_sync(0xffffffffu, pass[j])) continue;  // warp-uniform: nothing to insert
      const long long r = base0 + j * blockDim.x + threadIdx.x;
      long long idx = -1;
      if (pass[j]) {
        unsigned flags = 0;
        for (int f = 0; f < s.nflags; ++f)
          if (eval_str(s.flags[f], r)) flags |= 1u << f;
        const unsigned long long entry = static_cast<unsigned long long>(r + 1) | (static_cast<unsigned long long>(flags) << 57);
        if (s.hkeys) {
          // open addressing: the first row with a key claims its slot
          bool seen = false;
          const long long sl = build_hash_insert(s, key[j], seen);
          if (sl < 0) {
            set_fallback(s.err, FR_HASH_FULL);
          } else {
            if (!seen) {
              if (s.assign_groups)  // the group is the slot: zero its record
                for (int w = 0; w < s.zrec_words; ++w) s.zrec[sl * s.zrec_words + w] = 0ULL;
              s.table[sl] = entry;
            } else if (!s.mult) {
              dup = 1u;  // a repeated key: the unit reruns weighted
            }
            if (s.mult) atomicAdd(s.mult + sl, wgt[j]);
          }
          idx = -1;  // no presence bits
        } else {
          idx = key[j] - s.kmin;
          if (idx < 0 || idx >= s.range) {
            atomicExch(reinterpret_cast<unsigned long long*>(s.err), 1ULL);
            idx = -1;
          } else {
            if (s.assign_groups)  // the group is the key slot: zero its record
              for (int w = 0; w < s.zrec_words; ++w) s.zrec[idx * s.zrec_words + w] = 0ULL;
            if (s.row_rec) s.zrec[idx * s.zrec_words] = static_cast<unsigned long long>(entry & 0xffffffffULL) << 32;
            else s.table[idx] = entry;
            if (s.mult) atomicAdd(s.mult + idx, wgt[j]);
          }
        }
      }
      if (!s.hkeys) {
        if (s.unique) presence_insert_unique(s.bitmap, idx);
        else presence_insert(s.bitmap, idx, old[j], set[j], dup);
      }
    }
    if (!s.mult) {
#pragma unroll
      for (int j = 0; j < kBuildRows; ++j) dup |= old[j] & set[j];
    } else {
      dup = 0u;  // weighted: repeated keys are summed, not flagged
    }
  }
  build_dup_check(dup, s.err);
}

// value of accumulator `ac` for rows k0..k0+N-1 of this thread (row index
// k * CT + ct inside the tile); operands from the staged tile
template <int CT, int N>
__device__ __forceinline__ void acc_rows(const TileSpec& t, const unsigned char* stage, const Acc& ac, const bool* pass,
                                         const RowCtx* rc, int ct, int k0, unsigned long long* v) {
  if (ac.is_int) {
    const Operand& o = ac.f[0].x;
    const unsigned long long* col = reinterpret_cast<const unsigned long long*>(stage + t.col_off[o.col < 0 ? 0 : o.col]);
    if (o.src < 0) {
#pragma unroll
      for (int k = 0; k < N; ++k) v[k] = pass[k0 + k] ? col[(k0 + k) * CT + ct] : 0ULL;
    } else {
#pragma unroll
      for (int k = 0; k < N; ++k) v[k] = pass[k0 + k] ? ld_row(o, rc[k0 + k].rid[o.src]) : 0ULL;
    }
    return;
  }
  double d[N];
#pragma unroll
  for (int i = 0; i < kFixedFactors; ++i) {
    const Factor& f = ac.f[i];
    double xs[N];
    if (f.x.col >= 0 && f.x.src < 0) {
      // fact operand: every row reads the staged tile (masked rows are
      // discarded later, so no per-row branch)
      const unsigned long long* col = reinterpret_cast<const unsigned long long*>(stage + t.col_off[f.x.col]);
#pragma unroll
      for (int k = 0; k < N; ++k) xs[k] = __longlong_as_double(static_cast<long long>(col[(k0 + k) * CT + ct]));
    } else if (f.x.src >= 0) {
#pragma unroll
      for (int k = 0; k < N; ++k)
        xs[k] = pass[k0 + k] ? __longlong_as_double(static_cast<long long>(ld_row(f.x, rc[k0 + k].rid[f.x.src]))) : 0.0;
    } else {
#pragma unroll
      for (int k = 0; k < N; ++k) xs[k] = 0.0;
    }
    const double fa = f.fa, fb = f.fb;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const double y = __dadd_rn(fa, __dmul_rn(fb, xs[k]));
      d[k] = i == 0 ? y : __dmul_rn(d[k], y);
    }
  }
#pragma unroll
  for (int k = 0; k < N; ++k) {
    if (pass[k0 + k] && ac.gate_probe >= 0 && !((rc[k0 + k].flags[ac.gate_probe] >> ac.gate_bit) & 1u))
      d[k] = ac.gate_else;
    v[k] = pass[k0 + k] ? static_cast<unsigned long long>(__double_as_longlong(d[k])) : 0ULL;
  }
}

// Descriptors pre-resolved once per CTA into shared memory: stage-relative
// byte offsets and affine factor coefficients, read with static indices by
// fully unrolled loops (no dynamic param-space indexing in the tile loop).
constexpr unsigned kNoCol = 0xffffffffu;
// accumulator slots the tile kernels unroll (register budget per mode)
__host__ __device__ constexpr int max_acc_for(int mode) { return mode == MODE_SMALL ? kMaxAccSmall : 4; }
enum FactorMode : int { FM_SKIP = 0, FM_X = 1, FM_A_PLUS_X = 2, FM_A_MINUS_X = 3, FM_AFFINE = 4 };
struct TileDesc {
  int nterms, nacc, nkeys, nprobes;
  int t_kind[kMaxTerms];
  unsigned t_off[kMaxTerms];
  unsigned long long t_lo[kMaxTerms], t_hi[kMaxTerms];
  int a_int[kMaxAcc], a_gate_probe[kMaxAcc], a_gate_bit[kMaxAcc];
  double a_gate_else[kMaxAcc];
  unsigned a_off[kMaxAcc][kFixedFactors];
  int a_src[kMaxAcc][kFixedFactors];
  int a_mode[kMaxAcc][kFixedFactors];  // FM_* (uniform fast forms)
  int a_base[kMaxAcc];                 // earlier accumulator whose product is a prefix, or -1
  const void* a_ptr[kMaxAcc][kFixedFactors];  // MODE_HASH: probe-root operand columns (a_src >= 0)
  double a_fa[kMaxAcc][kFixedFactors], a_fb[kMaxAcc][kFixedFactors];
  unsigned k_off[kMaxKeys];
  unsigned p_off[kMaxProbes];
};

__device__ void load_desc(const TileSpec& t, TileDesc& d) {
  const ProbeSpec& s = t.p;
  d.nterms = s.nterms;
  d.nacc = s.nacc;
  d.nkeys = s.nkeys;
  d.nprobes = s.nprobes;
  for (int i = 0; i < s.nterms; ++i) {
    d.t_kind[i] = s.terms[i].kind;
    d.t_off[i] = s.terms[i].col >= 0 ? static_cast<unsigned>(t.col_off[s.terms[i].col]) : 0u;
    d.t_lo[i] = s.terms[i].lo;
    d.t_hi[i] = s.terms[i].hi;
  }
  for (int a = 0; a < s.nacc; ++a) {
    const Acc& ac = s.acc[a];
    d.a_int[a] = ac.is_int;
    d.a_gate_probe[a] = ac.gate_probe;
    d.a_gate_bit[a] = ac.gate_bit;
    d.a_gate_else[a] = ac.gate_else;
    for (int i = 0; i < kFixedFactors; ++i) {
      const Factor& f = ac.f[i];
      d.a_src[a][i] = f.x.src;
      d.a_ptr[a][i] = f.x.ptr;
      d.a_off[a][i] = (f.x.src < 0 && f.x.col >= 0) ? static_cast<unsigned>(t.col_off[f.x.col]) : kNoCol;
      d.a_fa[a][i] = ac.is_int ? 0.0 : f.fa;
      d.a_fb[a][i] = ac.is_int ? 0.0 : f.fb;
      // fast forms are exact restatements: 0 + 1*x == x (up to the sign of
      // a zero, which never survives the +0.0-seeded sums), a + 1*x == a + x,
      // a + (-1)*x == a - x; padding factors 1 + 0*0 are skipped
      int m = FM_AFFINE;
      if (d.a_off[a][i] == kNoCol && f.x.src < 0 && f.fa == 1.0 && f.fb == 0.0) m = FM_SKIP;
      else if (f.fa == 0.0 && f.fb == 1.0) m = FM_X;
      else if (f.fb == 1.0) m = FM_A_PLUS_X;
      else if (f.fb == -1.0) m = FM_A_MINUS_X;
      d.a_mode[a][i] = m;
    }
    d.a_base[a] = ac.base;
  }
  for (int q = 0; q < s.nkeys; ++q) d.k_off[q] = static_cast<unsigned>(t.col_off[s.keys[q].col]);
  for (int p = 0; p < s.nprobes; ++p) d.p_off[p] = static_cast<unsigned>(t.col_off[s.probes[p].key.col]);
}

// LEAN (MODE_HASH only): the common hash-group shape compiled without the
// general features - fact-column int keys (no dictionary, no string bytes),
// a direct table of 2-limb records, no probes, weights, gates or special-value
// flags. Same operation order as the general instance (same bits); the
// general kernel is ~14 k instructions and its hot loop missed the
// instruction cache (ncu: 40 % of warp stalls were no_instructions).
template <int MODE, int NA_, bool LEAN = false>
__global__ void __launch_bounds__(TileShape<MODE, LEAN>::THREADS, 1) k_tile(const TileSpec t) {
  using S = TileShape<MODE, LEAN>;
  constexpr bool LN = LEAN && MODE == MODE_HASH;
  constexpr int CW = S::CW, CT = S::CT, R = S::R, SUB = S::SUB;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned long long s_wred[MODE == MODE_SMALL ? kGroups : 1][kMaxAcc + 1][CW];
  __shared__ unsigned int s_codes[kGroups];
  __shared__ int s_overflow;
  __shared__ TileDesc d;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem);
  unsigned long long* empty = full + kMaxStages;
  // per-thread staging (SCALAR: running sums; SMALL: row values), then stages
  unsigned long long* s_stage_val = reinterpret_cast<unsigned long long*>(smem + 256);
  unsigned char* stages = smem + 256 + t.aux_bytes;
  const ProbeSpec& s = t.p;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long ntiles = (s.n + S::ROWS - 1) / S::ROWS;
  const int nst = t.stages;

  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_overflow = 0;
    load_desc(t, d);
  }
  if (threadIdx.x < kGroups) s_codes[threadIdx.x] = 0xffffffffu;
  for (int i = threadIdx.x; i < t.aux_bytes / 8; i += blockDim.x) s_stage_val[i] = 0;
  __syncthreads();

  if (warp == 0) {
    // ---- producer: one lane streams tiles into the ring ----
    if (lane == 0) {
      long long it = 0;
      for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = static_cast<int>(it % nst);
        if (it >= nst) mbar_wait(&empty[st], static_cast<unsigned>(((it / nst) - 1) & 1));
        if (MODE == MODE_HASH && t.evict_first) issue_tile<true>(t, stages + static_cast<size_t>(st) * t.stage_bytes, &full[st], tile);
        else issue_tile(t, stages + static_cast<size_t>(st) * t.stage_bytes, &full[st], tile);
      }
    }
  } else {
    // ---- consumers ----
    const int ct = threadIdx.x - 32;
    const int cw = warp - 1;
    constexpr int NA = kMaxAcc;
    constexpr int NAX = NA_;  // accumulators: exact count, fully unrolled
    constexpr int NG = 1;
    unsigned long long acc[NG][NA];
    unsigned int gcnt_local[NG];
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      gcnt_local[g] = 0;
#pragma unroll
      for (int a = 0; a < NA; ++a) acc[g][a] = 0;  // 0.0 and 0 share bits
    }
    long long absmax = 0;  // int accumulators: exactness guard
    double fabsmax = 0.0;  // build-group fp64 values: Q64.64 range guard
    long long it = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int st = static_cast<int>(it % nst);
      const unsigned char* stage = stages + static_cast<size_t>(st) * t.stage_bytes;
      mbar_wait(&full[st], static_cast<unsigned>((it / nst) & 1));
      const long long row0 = tile * S::ROWS;
      bool pass[R];
#pragma unroll
      for (int k = 0; k < R; ++k) pass[k] = row0 + k * CT + ct < s.n;
      // predicate: unrolled over the term slots, uniform dispatch per term,
      // straight-line over this thread's rows
#pragma unroll
      for (int i = 0; i < kMaxTerms; ++i) {
        if (i < d.nterms) {
          const int kind = d.t_kind[i];
          const unsigned long long* col = reinterpret_cast<const unsigned long long*>(stage + d.t_off[i]);
          const unsigned long long lo = d.t_lo[i], hi = d.t_hi[i];
          if (kind == RK_INT) {
            const unsigned long long span = hi - lo;
#pragma unroll
            for (int k = 0; k < R; ++k) pass[k] = pass[k] && (col[k * CT + ct] - lo <= span);
          } else if (kind == RK_F64) {
            const double flo = __longlong_as_double(static_cast<long long>(lo));
            const double fhi = __longlong_as_double(static_cast<long long>(hi));
#pragma unroll
            for (int k = 0; k < R; ++k) {
              const double x = __longlong_as_double(static_cast<long long>(col[k * CT + ct]));
              pass[k] = pass[k] && x >= flo && x <= fhi;
            }
          } else {
            RTerm tm;
            tm.kind = kind;
            tm.lo = lo;
            tm.hi = hi;
#pragma unroll
            for (int k = 0; k < R; ++k) pass[k] = pass[k] && eval_rterm(tm, kind <= RK_F64_NE ? col[k * CT + ct] : 0ULL);
          }
        }
      }
      RowCtx rc[R];
#pragma unroll
      for (int p = 0; p < kMaxProbes; ++p) {
        if (!LN && p < d.nprobes) {
          const Probe& pr = s.probes[p];
          const unsigned long long* col = reinterpret_cast<const unsigned long long*>(stage + d.p_off[p]);
#pragma unroll
          for (int k = 0; k < R; ++k)
            if (pass[k]) pass[k] = probe_lookup(pr, static_cast<long long>(col[k * CT + ct]), rc[k].rid[p], rc[k].flags[p], rc[k].gid[p], &rc[k].mult[p]);
        }
      }
      // weighted run (repeated build keys): the row counts prod(mult) times;
      // a probe whose root row is read must have matched exactly one row
      unsigned wt[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        wt[k] = 1u;
        if (!LN && s.weighted && pass[k]) {
#pragma unroll
          for (int p = 0; p < kMaxProbes; ++p) {
            if (p < d.nprobes) {
              wt[k] *= rc[k].mult[p];
              if (((s.root_mask >> p) & 1u) && rc[k].mult[p] != 1u) set_fallback(s.err, FR_DUP_KEY);
            }
          }
        }
      }
      bool any = MODE == MODE_SMALL;  // small-group runs warp-collective slot claims: no per-thread skip
#pragma unroll
      for (int k = 0; k < R; ++k) any = any || pass[k];
      if (any) {
        int slot[R];
        if constexpr (MODE == MODE_SMALL) {
          // the CTA's <= kGroups codes in registers: branch-free match
          unsigned cr[kGroups];
#pragma unroll
          for (int j = 0; j < kGroups; ++j) cr[j] = s_codes[j];
          unsigned code[R];
          bool miss = false;
#pragma unroll
          for (int k = 0; k < R; ++k) {
            code[k] = 0;
#pragma unroll
            for (int q = 0; q < kMaxKeys; ++q)
              if (q < d.nkeys) code[k] = (code[k] << 8) | stage[d.k_off[q] + k * CT + ct];
            slot[k] = -1;
#pragma unroll
            for (int j = 0; j < kGroups; ++j) slot[k] = cr[j] == code[k] ? j : slot[k];
            if (!pass[k]) slot[k] = -1;
            miss = miss || (pass[k] && slot[k] < 0);
          }
          if (__any_sync(0xffffffffu, miss)) {
            // first sighting of a code in this CTA: claim a free slot (rare)
#pragma unroll
            for (int k = 0; k < R; ++k) {
              if (!pass[k] || slot[k] >= 0) continue;
              for (int j = 0; j < kGroups; ++j) {
                const unsigned prev = atomicCAS(&s_codes[j], 0xffffffffu, code[k]);
                if (prev == 0xffffffffu || prev == code[k]) {
                  slot[k] = j;
                  break;
                }
              }
              if (slot[k] < 0) {
                s_overflow = 1;
                pass[k] = false;
              }
            }
          }
#pragma unroll
          for (int k = 0; k < R; ++k)
            if (pass[k]) s_stage_val[(slot[k] * (NA_ + 1) + NA_) * CT + ct] += wt[k];
        } else {
#pragma unroll
          for (int k = 0; k < R; ++k) gcnt_local[0] += pass[k] ? wt[k] : 0u;
        }
        unsigned g[R];
        if constexpr (MODE == MODE_HASH) {
          // group code per row (mixed radix over the key digits), then its
          // slot: the CTA's shared-memory records (hpriv) or the global table
#pragma unroll
          for (int k = 0; k < R; ++k) {
            g[k] = 0u;
            if (!pass[k]) continue;
            const long long row = row0 + k * CT + ct;
            unsigned long long code = 0;
            bool bad = false;
#pragma unroll
            for (int q = 0; q < kMaxKeys; ++q) {
              if (q < s.nhkeys) {
                const GKey& K = s.hkeys[q];
                long long rid = rc[k].rid[0];  // static select keeps rc in registers
#pragma unroll
                for (int p = 1; p < kMaxProbes; ++p) rid = K.x.src == p ? rc[k].rid[p] : rid;
                const long long krow = (LN || K.x.src < 0) ? row : rid;
                unsigned long long raw = 0;
                if (LN || !K.width)
                  raw = (LN || K.x.src < 0) ? reinterpret_cast<const unsigned long long*>(stage + t.col_off[K.x.col])[k * CT + ct]
                                            : ld_row(K.x, rid);
                unsigned long long dg;
                if constexpr (LN) {
                  dg = raw - static_cast<unsigned long long>(K.kmin);
                  if (K.step != 1) dg /= static_cast<unsigned long long>(K.step);
                } else {
                  dg = gkey_digit(K, raw, krow);
                }
                bad = bad || dg >= K.range;
                code += dg * K.stride;
              }
            }
            long long slot = -1;
            if (bad) {
              set_fallback(s.err, FR_KEY_RANGE);
            } else if (!LN && s.hpriv) {
              slot = static_cast<long long>(code);
              atomicAdd(s_stage_val + slot * (1 + kLimbWords * NA_), static_cast<unsigned long long>(wt[k]));
            } else {
              // direct tables are zeroed up front (no tag, no claim)
              slot = (!LN && s.htag) ? hash_claim(s, code) : static_cast<long long>(code);
              if (slot < 0) set_fallback(s.err, FR_HASH_FULL);
              else red_add_hint(s.gcnt + slot * s.gstride, static_cast<unsigned long long>(wt[k]) + kCntAdd, l2_policy_evict_last());
            }
            if (slot < 0) pass[k] = false;
            g[k] = static_cast<unsigned>(slot < 0 ? 0 : slot);
          }
        }
        if constexpr (MODE == MODE_BUILDGRP) {
#pragma unroll
          for (int k = 0; k < R; ++k) {
            unsigned gg = rc[k].gid[0];
#pragma unroll
            for (int p = 1; p < kMaxProbes; ++p) gg = s.group_probe == p ? rc[k].gid[p] : gg;
            g[k] = pass[k] ? gg : 0u;
            if (pass[k]) {
              atomicAdd(s.gcnt + static_cast<long long>(g[k]) * s.gstride, static_cast<unsigned long long>(wt[k]));
              atomicOr(s.touched + (g[k] >> 5), 1u << (g[k] & 31));
            }
          }
        }
        // values, fully unrolled (NA is a template parameter) and branch-free:
        // product = start * (fa0 + fb0 x0) * (fa1 + fb1 x1) * (fa2 + fb2 x2),
        // start = 1.0 (1 * f0 == f0 exactly) or an earlier accumulator's
        // product (prefix sharing); a missing operand reads as 0 and a
        // padding factor is 1 + 0 * 0, so every slot runs the same code
        double dvals[NAX > 0 ? NAX : 1][R];
#pragma unroll
        for (int a = 0; a < NAX; ++a) {
          const bool is_int = d.a_int[a];
          unsigned long long v[R];
          if (is_int) {
            const unsigned long long* col = reinterpret_cast<const unsigned long long*>(stage + d.a_off[a][0]);
            const int isrc = MODE == MODE_HASH ? d.a_src[a][0] : -1;
#pragma unroll
            for (int k = 0; k < R; ++k) {
              if (MODE == MODE_HASH && !LN && isrc >= 0) {  // a probe's root column at the matched row
                long long rid = rc[k].rid[0];
#pragma unroll
                for (int p = 1; p < kMaxProbes; ++p) rid = isrc == p ? rc[k].rid[p] : rid;
                v[k] = pass[k] ? static_cast<unsigned long long>(ld_i64(d.a_ptr[a][0], rid)) : 0ULL;
              } else {
                v[k] = pass[k] ? col[k * CT + ct] : 0ULL;
              }
              if (!LN && s.weighted && wt[k] != 1u) {  // v * weight, exactly or the exact path
                const __int128 pw = static_cast<__int128>(static_cast<long long>(v[k])) * wt[k];
                if (pw != static_cast<__int128>(static_cast<long long>(pw))) set_fallback(s.err, FR_INT_RANGE);
                v[k] = static_cast<unsigned long long>(static_cast<long long>(pw));
              }
              long long iv = static_cast<long long>(v[k]);
              iv = iv < 0 ? -iv : iv;
              absmax = iv > absmax ? iv : absmax;
              dvals[a][k] = 1.0;
            }
          } else {
            const int base = d.a_base[a];
            double dv[R];
#pragma unroll
            for (int k = 0; k < R; ++k) {
              dv[k] = 1.0;
#pragma unroll
              for (int b = 0; b < a; ++b) dv[k] = base == b ? dvals[b][k] : dv[k];
            }
#pragma unroll
            for (int i = 0; i < kFixedFactors; ++i) {
              const unsigned off = d.a_off[a][i];
              const bool has = off != kNoCol;
              const unsigned long long* col = reinterpret_cast<const unsigned long long*>(stage + (has ? off : 0u));
              const double fa = d.a_fa[a][i], fb = d.a_fb[a][i];
              const int fsrc = MODE == MODE_HASH ? d.a_src[a][i] : -1;
#pragma unroll
              for (int k = 0; k < R; ++k) {
                double x = has ? __longlong_as_double(static_cast<long long>(col[k * CT + ct])) : 0.0;
                if (MODE == MODE_HASH && !LN && fsrc >= 0) {  // a probe's root column at the matched row
                  long long rid = rc[k].rid[0];
#pragma unroll
                  for (int p = 1; p < kMaxProbes; ++p) rid = fsrc == p ? rc[k].rid[p] : rid;
                  x = pass[k] ? ld_f64(d.a_ptr[a][i], rid) : 0.0;
                }
                dv[k] = __dmul_rn(dv[k], __dadd_rn(fa, __dmul_rn(fb, x)));
              }
            }
#pragma unroll
            for (int k = 0; k < R; ++k) dvals[a][k] = dv[k];
            const int gp = d.a_gate_probe[a];
            if (!LN && gp >= 0) {
              const int gb = d.a_gate_bit[a];
              const double ge = d.a_gate_else[a];
#pragma unroll
              for (int k = 0; k < R; ++k) {
                unsigned fl = rc[k].flags[0];  // static select keeps rc in registers
#pragma unroll
                for (int p = 1; p < kMaxProbes; ++p) fl = gp == p ? rc[k].flags[p] : fl;
                if (pass[k] && !((fl >> gb) & 1u)) dv[k] = ge;
              }
            }
#pragma unroll
            for (int k = 0; k < R; ++k) v[k] = pass[k] ? static_cast<unsigned long long>(__double_as_longlong(dv[k])) : 0ULL;
          }
          if ((MODE == MODE_SCALAR || MODE == MODE_SMALL) && !is_int && s.weighted) {
#pragma unroll
            for (int k = 0; k < R; ++k)
              if (wt[k] != 1u)
                v[k] = static_cast<unsigned long long>(__double_as_longlong(
                    __dmul_rn(__longlong_as_double(static_cast<long long>(v[k])), static_cast<double>(wt[k]))));
          }
          if constexpr (MODE == MODE_SCALAR) {
#pragma unroll
            for (int k = 0; k < R; ++k) acc[0][a] = add_acc(is_int, acc[0][a], v[k]);  // masked rows add 0
          } else if constexpr (MODE == MODE_SMALL) {
            // per-thread accumulator slot [group][a][thread]; masked rows add
            // 0 to slot 0 (x + 0 == x), so no per-row branch
#pragma unroll
            for (int k = 0; k < R; ++k) {
              const int sl = slot[k] < 0 ? 0 : slot[k];
              unsigned long long* cell = s_stage_val + (sl * (NAX + 1) + a) * CT + ct;
              *cell = add_acc(is_int, *cell, v[k]);
            }
          } else {
#pragma unroll
            for (int k = 0; k < R; ++k) {
              if (!pass[k]) continue;
              __int128 qv;
              if (is_int) {
                qv = static_cast<__int128>(static_cast<long long>(v[k]));
              } else {
                const double dv = __longlong_as_double(static_cast<long long>(v[k]));
                if (!f64_to_qf(dv, MODE == MODE_HASH ? s.qfrac : 64, qv)) {
                  qv = 0;
                  if (MODE == MODE_HASH && !LN && s.hflags >= 0 && (isnan(dv) || isinf(dv))) {
                    const unsigned long long bit = isnan(dv) ? 1ULL : dv > 0 ? 2ULL : 4ULL;
                    atomicOr(s.gcnt + static_cast<long long>(g[k]) * s.gstride + s.hflags, bit << (3 * a));
                  } else {
                    set_fallback(s.err, FR_Q64_CONVERT);
                    if (MODE == MODE_HASH && s.qstats && !isnan(dv) && !isinf(dv))
                      atomicMax(s.qstats, static_cast<long long>(-lowbit_exp(dv)));
                  }
                } else {
                  fabsmax = fmax(fabsmax, fabs(dv));
                }
                if (!LN && wt[k] != 1u) {  // exact: the weight multiplies the fixed-point value
                  qv *= static_cast<__int128>(wt[k]);
                  fabsmax = fmax(fabsmax, fabs(dv) * static_cast<double>(wt[k]));
                }
              }
              if (MODE == MODE_HASH && !LN && s.hpriv) {
                atomic_add_limbs(s_stage_val + static_cast<long long>(g[k]) * (1 + kLimbWords * NA_) + 1 + a * kLimbWords, qv);
              } else if (MODE == MODE_HASH && (LN || s.hlimbs == 2)) {
                unsigned long long* w = s.gacc + static_cast<long long>(g[k]) * s.gstride + s.hoff[a];
                if (is_int) red_add_hint(w, static_cast<unsigned long long>(static_cast<long long>(qv)), l2_policy_evict_last());
                else if (!atomic_add_limbs2(w, qv, l2_policy_evict_last())) set_fallback(s.err, FR_LIMB2);
              } else {
                atomic_add_limbs(s.gacc + static_cast<long long>(g[k]) * s.gstride + a * kLimbWords, qv);
              }
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    // int64 sums are exact only while |v| * rows < 2^63 (the reference
    // errors on the first overflowing prefix): otherwise the exact path
    if (MODE == MODE_HASH && s.absmax_out) {
      if (absmax) atomicMax(s.absmax_out, absmax);
    } else if (static_cast<double>(absmax) * static_cast<double>(s.n) >= 9.0e18) {
      set_fallback(s.err, FR_INT_RANGE);
    }
    if constexpr (MODE == MODE_BUILDGRP || MODE == MODE_HASH) q64_range_check(fabsmax, s.n, s.err, MODE == MODE_HASH ? s.qfrac : 64);
    if (MODE == MODE_HASH && s.fmax_out && fabsmax > 0.0) atomicMax(s.fmax_out, __double_as_longlong(fabsmax));
    if constexpr (MODE == MODE_SMALL) {
      for (int gg = 0; gg < kGroups; ++gg) {
        for (int a = 0; a <= s.nacc; ++a) {
          unsigned long long x = s_stage_val[(gg * (NA_ + 1) + a) * CT + ct];
          const bool is_int = a == s.nacc || s.acc[a].is_int;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) x = add_acc(is_int, x, __shfl_xor_sync(0xffffffffu, x, o));
          if (lane == 0) s_wred[gg][a == s.nacc ? kMaxAcc : a][cw] = x;
        }
      }
    }
    if constexpr (MODE == MODE_SCALAR) {
      // fixed-order warp trees, one slot per (accumulator, warp)
#pragma unroll
      for (int gg = 0; gg < NG; ++gg) {
#pragma unroll
        for (int a = 0; a < NA; ++a) {
          if (a < s.nacc) {
            unsigned long long x = acc[gg][a];
            const bool is_int = s.acc[a].is_int;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x = add_acc(is_int, x, __shfl_xor_sync(0xffffffffu, x, o));
            if (lane == 0) s_wred[gg][a][cw] = x;
          }
        }
        unsigned long long c = gcnt_local[gg];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) s_wred[gg][kMaxAcc][cw] = c;
      }
    }
  }
  __syncthreads();
  if constexpr (MODE == MODE_SCALAR) {
    if (threadIdx.x == 0) {
      unsigned long long* out = s.part + static_cast<long long>(blockIdx.x) * (kMaxAcc + 1);
      for (int a = 0; a < s.nacc; ++a) {
        unsigned long long tot = s_wred[0][a][0];
        for (int w = 1; w < CW; ++w) tot = add_acc(s.acc[a].is_int, tot, s_wred[0][a][w]);
        out[a] = tot;
      }
      unsigned long long c = 0;
      for (int w = 0; w < CW; ++w) c += s_wred[0][kMaxAcc][w];
      out[kMaxAcc] = c;
    }
  } else if constexpr (MODE == MODE_HASH) {
    if (!LN && s.hpriv) {
      // flush the CTA's records into the (direct) global table: one add per
      // word per CTA, limbs re-split so every added limb is < 2^42; the
      // packed count carries the adds for the reader's limb bound
      constexpr int RW = 1 + kLimbWords * NA_;
      const long long ncode = static_cast<long long>(s.hmask) + 1;
      for (long long code = threadIdx.x; code < ncode; code += blockDim.x) {
        const unsigned long long* r = s_stage_val + code * RW;
        const unsigned long long c = r[0];
        if (!c) continue;
        if (c >= static_cast<unsigned long long>(kLimbMaxRows)) set_fallback(s.err, FR_LIMB_ROWS);
        atomicAdd(s.gcnt + code * s.gstride, c + kCntAdd);
#pragma unroll
        for (int a = 0; a < NA_; ++a) {
          const __int128 v = limbs_to_i128(r + 1 + a * kLimbWords);
          if (s.hlimbs == 2) {
            unsigned long long* w = s.gacc + code * s.gstride + s.hoff[a];
            if (s.acc[a].is_int) red_add_hint(w, static_cast<unsigned long long>(static_cast<long long>(v)), l2_policy_evict_last());
            else if (!atomic_add_limbs2(w, v, l2_policy_evict_last())) set_fallback(s.err, FR_LIMB2);
          } else {
            atomic_add_limbs(s.gacc + code * s.gstride + a * kLimbWords, v);
          }
        }
      }
    }
  } else if constexpr (MODE == MODE_SMALL) {
    if (s_overflow && threadIdx.x == 0) atomicExch(reinterpret_cast<unsigned long long*>(s.err), 1ULL);
    SmallPart* out = reinterpret_cast<SmallPart*>(s.part) + blockIdx.x;
    for (int sl = threadIdx.x; sl < kGroups; sl += blockDim.x) {
      out->codes[sl] = s_codes[sl];
      unsigned long long c = 0;
      for (int w = 0; w < CW; ++w) c += s_wred[sl][kMaxAcc][w];
      out->cnt[sl] = c;
      for (int a = 0; a < s.nacc; ++a) {
        unsigned long long tot = s_wred[sl][a][0];
        for (int w = 1; w < CW; ++w) tot = add_acc(s.acc[a].is_int, tot, s_wred[sl][a][w]);
        out->acc[sl][a] = tot;
      }
    }
  }
}

}  // namespace fz
}  // namespace tqp
