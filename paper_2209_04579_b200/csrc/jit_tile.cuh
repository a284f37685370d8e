// Skeleton of a specialised fused fact-scan kernel, compiled at run time by
// NVRTC (jit.cu) after the generated pipeline hooks:
//
//   Q_MODE, Q_NA, Q_ROWS, Q_CW, Q_INT_MASK       constants of the pipeline
//   bool q_row(t, stage, ri, valid, v, code, gid, absmax)
//        predicate + probes + accumulator values of tile row `ri`, straight-
//        line code with every constant folded (fused.cu's generator)
//
// The pipeline is the one of k_tile (fused_kernels.cuh): a persistent CTA per
// SM, warp 0 streams tiles into a shared-memory ring with cp.async.bulk +
// mbarrier transaction counts, Q_CW consumer warps evaluate their rows and
// release the stage. Outputs use the same partial layouts as k_tile, so the
// finalize / merge kernels are shared.
#pragma once

namespace tqp {
namespace fz {

constexpr int Q_CT = Q_CW * 32;
constexpr int Q_R = Q_ROWS / Q_CT;
#ifndef Q_SLOTS
#define Q_SLOTS kGroups  // small-group slots per CTA (<= kGroups)
#endif
#ifndef Q_REGACC
#define Q_REGACC 0  // small-group accumulators in registers instead of shared-memory cells
#endif
__device__ __forceinline__ bool q_is_int(int a) { return (Q_INT_MASK >> a) & 1; }

extern "C" __global__ void __launch_bounds__(Q_CT + 32, 1) q_tile(const TileSpec t) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned long long s_wred[Q_MODE == MODE_SMALL ? Q_SLOTS : 1][Q_NA + 1][Q_CW];
  __shared__ unsigned int s_codes[kGroups];
  __shared__ int s_ncodes;
  __shared__ int s_overflow;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem);
  unsigned long long* empty = full + kMaxStages;
  unsigned long long* s_cell = reinterpret_cast<unsigned long long*>(smem + 256);
  unsigned char* stages = smem + 256 + t.aux_bytes;
  const ProbeSpec& s = t.p;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long ntiles = (s.n + Q_ROWS - 1) / Q_ROWS;
  const int nst = t.stages;

  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], Q_CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_overflow = 0;
    s_ncodes = 0;
  }
  if (threadIdx.x < kGroups) s_codes[threadIdx.x] = 0xffffffffu;
  for (int i = threadIdx.x; i < t.aux_bytes / 8; i += blockDim.x) s_cell[i] = 0;
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      long long it = 0;
      for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = static_cast<int>(it % nst);
        if (it >= nst) mbar_wait(&empty[st], static_cast<unsigned>(((it / nst) - 1) & 1));
        if (Q_MODE == MODE_HASH && t.evict_first) issue_tile<true>(t, stages + static_cast<size_t>(st) * t.stage_bytes, &full[st], tile);
        else issue_tile(t, stages + static_cast<size_t>(st) * t.stage_bytes, &full[st], tile);
      }
    }
  } else {
    const int ct = threadIdx.x - 32;
    const int cw = warp - 1;
    unsigned long long acc[Q_NA > 0 ? Q_NA : 1];
#pragma unroll
    for (int a = 0; a < Q_NA; ++a) acc[a] = 0;  // 0.0 and 0 share bits
    unsigned long long cnt = 0;
    long long absmax = 0;
    double fabsmax = 0.0;  // build-group fp64 values: Q64.64 range guard
    // MODE_SMALL with Q_REGACC: per-thread [slot][acc + count] accumulators in
    // registers. A row adds to its slot only (predicated), in the same order
    // as the shared-memory cells, so the sums are bit-identical to them; the
    // cells' shared-memory traffic (a load and a store of 8 B per accumulator
    // per row, twice the staged column bytes) is gone.
    unsigned long long racc[Q_REGACC ? Q_SLOTS : 1][Q_NA + 1];
#pragma unroll
    for (int j = 0; j < (Q_REGACC ? Q_SLOTS : 1); ++j)
#pragma unroll
      for (int a = 0; a <= Q_NA; ++a) racc[j][a] = 0;
    long long it = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int st = static_cast<int>(it % nst);
      const unsigned char* stage = stages + static_cast<size_t>(st) * t.stage_bytes;
      mbar_wait(&full[st], static_cast<unsigned>((it / nst) & 1));
      const long long row0 = tile * Q_ROWS;
      bool pass[Q_R];
      unsigned long long v[Q_R][Q_NA > 0 ? Q_NA : 1];
      unsigned code[Q_R], gid[Q_R];
#pragma unroll
      for (int k = 0; k < Q_R; ++k) {
        const int ri = k * Q_CT + ct;
        pass[k] = q_row(t, stage, ri, row0 + ri < s.n, v[k], code[k], gid[k], absmax);
      }
      if constexpr (Q_MODE == MODE_SCALAR) {
#pragma unroll
        for (int k = 0; k < Q_R; ++k) {
          cnt += pass[k] ? 1u : 0u;
#pragma unroll
          for (int a = 0; a < Q_NA; ++a) acc[a] = add_acc(q_is_int(a), acc[a], v[k][a]);  // masked rows add 0
        }
      } else if constexpr (Q_MODE == MODE_SMALL) {
        // slot of each row's code among the CTA's claimed codes
        const int ncl = *reinterpret_cast<volatile int*>(&s_ncodes);
        unsigned cr[Q_SLOTS];
#pragma unroll
        for (int j = 0; j < Q_SLOTS; ++j) cr[j] = s_codes[j];
        int slot[Q_R];
        bool miss = false;
#pragma unroll
        for (int k = 0; k < Q_R; ++k) {
          slot[k] = -1;
          if (Q_SLOTS <= 4 || ncl <= 4) {
#pragma unroll
            for (int j = 0; j < (Q_SLOTS < 4 ? Q_SLOTS : 4); ++j) slot[k] = cr[j] == code[k] ? j : slot[k];
          } else {
#pragma unroll
            for (int j = 0; j < Q_SLOTS; ++j) slot[k] = cr[j] == code[k] ? j : slot[k];
          }
          miss = miss || (pass[k] && slot[k] < 0);
        }
        if (__any_sync(0xffffffffu, miss)) {
          // first sighting of a code in this CTA: claim a free slot (rare)
#pragma unroll
          for (int k = 0; k < Q_R; ++k) {
            if (!pass[k] || slot[k] >= 0) continue;
            for (int j = 0; j < Q_SLOTS; ++j) {
              const unsigned prev = atomicCAS(&s_codes[j], 0xffffffffu, code[k]);
              if (prev == 0xffffffffu || prev == code[k]) {
                slot[k] = j;
                if (prev == 0xffffffffu) atomicMax(&s_ncodes, j + 1);
                break;
              }
            }
            if (slot[k] < 0) {
              s_overflow = 1;
              pass[k] = false;
#pragma unroll
              for (int a = 0; a < Q_NA; ++a) v[k][a] = 0;
            }
          }
        }
        // per-thread cells [slot][acc + count][thread]; masked rows add 0 to
        // slot 0 (x + 0 == x), so there is no per-row branch
#if Q_REGACC
#pragma unroll
        for (int k = 0; k < Q_R; ++k) {
          const int tgt = slot[k] < 0 ? 0 : slot[k];
#pragma unroll
          for (int j = 0; j < Q_SLOTS; ++j) {
            if (tgt == j) {
#pragma unroll
              for (int a = 0; a < Q_NA; ++a) racc[j][a] = add_acc(q_is_int(a), racc[j][a], v[k][a]);
              racc[j][Q_NA] += pass[k] ? 1u : 0u;
            }
          }
        }
#else
#pragma unroll
        for (int k = 0; k < Q_R; ++k) {
          unsigned long long* cell = s_cell + (slot[k] < 0 ? 0 : slot[k]) * (Q_NA + 1) * Q_CT + ct;
#pragma unroll
          for (int a = 0; a < Q_NA; ++a) cell[a * Q_CT] = add_acc(q_is_int(a), cell[a * Q_CT], v[k][a]);
          cell[Q_NA * Q_CT] += pass[k] ? 1u : 0u;
        }
#endif
      } else if constexpr (Q_MODE == MODE_HASH) {
        // k_tile<MODE_HASH, NA, LEAN>'s row update: packed count, then the
        // exact 2-limb sums (Q(128-F).F fixed point, F = s.qfrac)
        const unsigned long long pol = l2_policy_evict_last();
#pragma unroll
        for (int k = 0; k < Q_R; ++k) {
          if (!pass[k]) continue;
          unsigned long long* rec = s.gcnt + static_cast<long long>(gid[k]) * s.gstride;
          red_add_hint(rec, 1ULL + kCntAdd, pol);
#pragma unroll
          for (int a = 0; a < Q_NA; ++a) {
            __int128 qv;
            if (q_is_int(a)) {
              qv = static_cast<__int128>(static_cast<long long>(v[k][a]));
            } else {
              const double dv = __longlong_as_double(static_cast<long long>(v[k][a]));
              if (!f64_to_qf(dv, s.qfrac, qv)) {
                qv = 0;
                set_fallback(s.err, FR_Q64_CONVERT);
                if (s.qstats && !isnan(dv) && !isinf(dv)) atomicMax(s.qstats, static_cast<long long>(-lowbit_exp(dv)));
              } else {
                fabsmax = fmax(fabsmax, fabs(dv));
              }
            }
            if (q_is_int(a)) red_add_hint(rec + 1 + s.hoff[a], static_cast<unsigned long long>(static_cast<long long>(qv)), pol);
            else if (!atomic_add_limbs2(rec + 1 + s.hoff[a], qv, pol)) set_fallback(s.err, FR_LIMB2);
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < Q_R; ++k) {
          if (!pass[k]) continue;
          atomicAdd(s.gcnt + static_cast<long long>(gid[k]) * s.gstride, 1ULL);
          atomicOr(s.touched + (gid[k] >> 5), 1u << (gid[k] & 31));
#pragma unroll
          for (int a = 0; a < Q_NA; ++a) {
            __int128 qv;
            if (q_is_int(a)) {
              qv = static_cast<__int128>(static_cast<long long>(v[k][a]));
            } else {
              const double dv = __longlong_as_double(static_cast<long long>(v[k][a]));
              fabsmax = fmax(fabsmax, fabs(dv));
              if (!f64_to_q64(dv, qv)) {
                set_fallback(s.err, FR_Q64_CONVERT);
                qv = 0;
              }
            }
            atomic_add_limbs(s.gacc + static_cast<long long>(gid[k]) * s.gstride + a * kLimbWords, qv);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    // int64 sums are exact only while |v| * rows < 2^63: otherwise the exact
    // path (hash groups: checked per group against the scan's max at output)
    if constexpr (Q_MODE == MODE_HASH) {
      if (s.absmax_out && absmax) atomicMax(s.absmax_out, absmax);
      else if (!s.absmax_out && static_cast<double>(absmax) * static_cast<double>(s.n) >= 9.0e18) set_fallback(s.err, FR_INT_RANGE);
      q64_range_check(fabsmax, s.n, s.err, s.qfrac);
      if (s.fmax_out && fabsmax > 0.0) atomicMax(s.fmax_out, __double_as_longlong(fabsmax));
    } else if (static_cast<double>(absmax) * static_cast<double>(s.n) >= 9.0e18) {
      set_fallback(s.err, FR_INT_RANGE);
    }
    if constexpr (Q_MODE == MODE_BUILDGRP) q64_range_check(fabsmax, s.n, s.err);
    if constexpr (Q_MODE == MODE_SMALL) {
#pragma unroll
      for (int gg = 0; gg < Q_SLOTS; ++gg) {
#pragma unroll
        for (int a = 0; a <= Q_NA; ++a) {
#if Q_REGACC
          unsigned long long x = racc[gg][a];
#else
          unsigned long long x = s_cell[(gg * (Q_NA + 1) + a) * Q_CT + ct];
#endif
          const bool is_int = a == Q_NA || q_is_int(a);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) x = add_acc(is_int, x, __shfl_xor_sync(0xffffffffu, x, o));
          if (lane == 0) s_wred[gg][a][cw] = x;
        }
      }
    }
    if constexpr (Q_MODE == MODE_SCALAR) {
#pragma unroll
      for (int a = 0; a < Q_NA; ++a) {
        unsigned long long x = acc[a];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x = add_acc(q_is_int(a), x, __shfl_xor_sync(0xffffffffu, x, o));
        if (lane == 0) s_wred[0][a][cw] = x;
      }
      unsigned long long c = cnt;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if (lane == 0) s_wred[0][Q_NA][cw] = c;
    }
  }
  __syncthreads();
  if constexpr (Q_MODE == MODE_SCALAR) {
    if (threadIdx.x == 0) {
      unsigned long long* out = s.part + static_cast<long long>(blockIdx.x) * (kMaxAcc + 1);
      for (int a = 0; a < Q_NA; ++a) {
        unsigned long long tot = s_wred[0][a][0];
        for (int w = 1; w < Q_CW; ++w) tot = add_acc(q_is_int(a), tot, s_wred[0][a][w]);
        out[a] = tot;
      }
      unsigned long long c = 0;
      for (int w = 0; w < Q_CW; ++w) c += s_wred[0][Q_NA][w];
      out[kMaxAcc] = c;
    }
  } else if constexpr (Q_MODE == MODE_SMALL) {
    // slot overflow: the 8-slot kernel reruns the scan (err[1]) or, with
    // every slot in use, the exact per-instruction path does (err[0])
    if (s_overflow && threadIdx.x == 0) atomicExch(reinterpret_cast<unsigned long long*>(s.err) + (Q_SLOTS < kGroups ? 1 : 0), 1ULL);
    SmallPart* out = reinterpret_cast<SmallPart*>(s.part) + blockIdx.x;
    for (int sl = threadIdx.x; sl < kGroups; sl += blockDim.x) {
      if (sl >= Q_SLOTS) {
        out->codes[sl] = 0xffffffffu;
        out->cnt[sl] = 0;
        continue;
      }
      out->codes[sl] = s_codes[sl];
      unsigned long long c = 0;
      for (int w = 0; w < Q_CW; ++w) c += s_wred[sl][Q_NA][w];
      out->cnt[sl] = c;
      for (int a = 0; a < Q_NA; ++a) {
        unsigned long long tot = s_wred[sl][a][0];
        for (int w = 1; w < Q_CW; ++w) tot = add_acc(q_is_int(a), tot, s_wred[sl][a][w]);
        out->acc[sl][a] = tot;
      }
    }
  }
}

}  // namespace fz
}  // namespace tqp
