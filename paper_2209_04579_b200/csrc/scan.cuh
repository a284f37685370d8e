// Single-pass decoupled-lookback tile scan primitives (shared by the prefix
// sum, compaction and radix-sort kernels).
#pragma once

#include "device.cuh"

#ifndef TQP_LOOKBACK_SLEEP
#define TQP_LOOKBACK_SLEEP 0
#endif

namespace tqp {

// 16-byte tile descriptor {status, value}; published and read as one 128-bit
// word so a reader never sees a status without its value.
enum : long long { TILE_INVALID = 0, TILE_PARTIAL = 1, TILE_INCLUSIVE = 2 };

__device__ __forceinline__ void tile_publish(longlong2* desc, int tile, long long status, long long value) {
  asm volatile("st.relaxed.gpu.global.v2.s64 [%0], {%1, %2};" ::"l"(desc + tile), "l"(status), "l"(value)
               : "memory");
}

// Must be a volatile (re-issued) load: a plain __ldcg may be hoisted out of
// the spin loop below, which would then read unpublished tiles as zero.
__device__ __forceinline__ longlong2 tile_read(const longlong2* p) {
  longlong2 d;
  asm volatile("ld.relaxed.gpu.global.v2.s64 {%0, %1}, [%2];" : "=l"(d.x), "=l"(d.y) : "l"(p) : "memory");
  return d;
}

// Called by ALL lanes of one warp; returns the exclusive prefix of `tile`
// (sum of aggregates of tiles 0..tile-1) and publishes this tile's inclusive
// value. Wrapping uint64 arithmetic.
__device__ __forceinline__ long long tile_lookback(longlong2* desc, int tile, long long agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) tile_publish(desc, 0, TILE_INCLUSIVE, agg);
    return 0;
  }
  if (lane == 0) tile_publish(desc, tile, TILE_PARTIAL, agg);
  unsigned long long excl = 0;
  int base = tile - 1;
  while (true) {
    int idx = base - lane;
    longlong2 d = make_longlong2(TILE_INCLUSIVE, 0);
    if (idx >= 0) {
      d = tile_read(desc + idx);
#if TQP_LOOKBACK_SLEEP
      for (unsigned ns = TQP_LOOKBACK_SLEEP; d.x == TILE_INVALID; ns = ns < 1024 ? 2 * ns : ns) {
        __nanosleep(ns);
        d = tile_read(desc + idx);
      }
#else
      while (d.x == TILE_INVALID) d = tile_read(desc + idx);
#endif
    }
    unsigned incl = __ballot_sync(0xffffffffu, d.x == TILE_INCLUSIVE);
    int stop = incl ? __ffs(incl) - 1 : 31;
    unsigned long long v = lane <= stop ? static_cast<unsigned long long>(d.y) : 0ULL;
    excl += warp_sum(v);
    if (incl) break;
    base -= 32;
  }
  if (lane == 0) tile_publish(desc, tile, TILE_INCLUSIVE, static_cast<long long>(excl + static_cast<unsigned long long>(agg)));
  return static_cast<long long>(excl);
}

// Block-wide exclusive scan of one value per thread (uint64 wrapping).
// Returns the exclusive prefix; *total gets the block sum. Uses `warp_tot`
// (>= 32 entries of shared memory).
__device__ __forceinline__ unsigned long long block_exclusive_scan(unsigned long long v, unsigned long long* warp_tot,
                                                                   unsigned long long* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = (blockDim.x + 31) >> 5;
  unsigned long long incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = lane < nwarps ? warp_tot[lane] : 0ULL;
    unsigned long long wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < nwarps) warp_tot[lane] = wi - w;  // exclusive warp offsets
    if (lane == nwarps - 1) warp_tot[32] = wi;
  }
  __syncthreads();
  unsigned long long r = warp_tot[warp] + incl - v;
  *total = warp_tot[32];
  __syncthreads();
  return r;
}

}  // namespace tqp
