// Skeleton of a TMA-staged build-side kernel (large build sides), compiled at
// run time by NVRTC (jit.cu) after the generated hook
//
//   QB_CW, QB_ROWS                           consumer warps, rows per tile
//   B_ASSIGN, B_ZREC                         as jit_build.cuh
//   void qb_rows(t, b, stage, ct, row0, pass, key, flags)
//        terms, string terms, LIKE flags and child probes of the thread's
//        QB_R rows of the staged tile, phase by phase (fused.cu's generator)
//
// The staging is the fact scan's (jit_tile.cuh): a persistent CTA per SM,
// warp 0 streams every build column the rows read (key, term, probe-key and
// string columns) into a shared-memory ring with cp.async.bulk + mbarrier
// transaction counts; QB_CW consumer warps evaluate the rows and insert as
// jit_build.cuh does (plain stores, presence bits OR-reduced per warp, the
// group record of a group-assigning build zeroed by the inserting row).
#pragma once

namespace tqp {
namespace fz {

constexpr int QB_CT = QB_CW * 32;
constexpr int QB_R = QB_ROWS / QB_CT;

extern "C" __global__ void __launch_bounds__(QB_CT + 32, 1) q_build_tile(const TileSpec t, const BuildSpec b) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem);
  unsigned long long* empty = full + kMaxStages;
  unsigned char* stages = smem + 256;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long ntiles = (b.n + QB_ROWS - 1) / QB_ROWS;
  const int nst = t.stages;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], QB_CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      int st = 0;
      unsigned ph = 0;
      long long it = 0;
      for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        if (it >= nst) mbar_wait(&empty[st], ph ^ 1u);
        issue_tile(t, stages + static_cast<size_t>(st) * t.stage_bytes, &full[st], tile);
        if (++st == nst) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
    return;
  }
  const int ct = threadIdx.x - 32;
  unsigned dup = 0;
  int st = 0;
  unsigned ph = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const unsigned char* stage = stages + static_cast<size_t>(st) * t.stage_bytes;
    mbar_wait(&full[st], ph);
    const long long row0 = tile * QB_ROWS;
    bool pass[QB_R];
    long long key[QB_R];
    unsigned flags[QB_R];
    qb_rows(t, b, stage, ct, row0, pass, key, flags);
    unsigned old[QB_R], set[QB_R];
#pragma unroll
    for (int k = 0; k < QB_R; ++k) {
      old[k] = set[k] = 0u;
      if (!__any_sync(0xffffffffu, pass[k])) continue;  // warp-uniform
      const long long r = row0 + k * QB_CT + ct;
      long long idx = -1;
      if (pass[k]) {
        idx = key[k] - b.kmin;
        if (idx < 0 || idx >= b.range) {
          set_fallback(b.err, FR_BUILD_RANGE);
          idx = -1;
        } else {
#if B_ASSIGN
          {
            ulonglong2* rec = reinterpret_cast<ulonglong2*>(b.zrec + idx * B_ZREC);
#pragma unroll
            for (int w = 0; w < B_ZREC / 2; ++w) rec[w] = make_ulonglong2(0ULL, 0ULL);
          }
#endif
#if B_ROWREC
          b.zrec[idx * B_ZREC] = static_cast<unsigned long long>(r + 1) << 32;
#else
          b.table[idx] = static_cast<unsigned long long>(r + 1) | (static_cast<unsigned long long>(flags[k]) << 57);
#endif
        }
      }
#if B_UNIQUE
      presence_insert_unique(b.bitmap, idx);
#else
      presence_insert(b.bitmap, idx, old[k], set[k], dup);
#endif
    }
#pragma unroll
    for (int k = 0; k < QB_R; ++k) dup |= old[k] & set[k];
    // release the stage only after every value read from it has been used
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (++st == nst) {
      st = 0;
      ph ^= 1u;
    }
  }
  build_dup_check(dup, b.err);
}

}  // namespace fz
}  // namespace tqp
