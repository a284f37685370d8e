// Micro-benchmark of the group walk behind the fused top-k (csrc/fused.cu):
// 15 M key slots, ~10 % present (presence bitmap), ~20 % of those with rows;
// per present slot read the row count and the three limb words, form the
// first sort key word and keep a per-warp minimum. Variants isolate the cost
// of the walk structure (compaction vs per-lane slots, unrolling, occupancy).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/topk_walk_probe tools/topk_walk_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long key_of(const unsigned long long* limbs, unsigned g) {
  const unsigned long long* w = limbs + 3ULL * g;
  const unsigned __int128 u = (unsigned __int128)w[0] + ((unsigned __int128)w[1] << 42) +
                              ((unsigned __int128)(__int128)(long long)w[2] << 84);
  const double d = (double)(__int128)u * 5.421010862427522e-20;
  const unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return ~((b >> 63) ? ~b : (b ^ 0x8000000000000000ULL));
}

// V2/V3: lane = slot, chunks of 32 slots, U chunks per iteration
template <int U>
__global__ void walk_lane(const unsigned* present, const unsigned long long* cnt, const unsigned long long* limbs,
                          long long n, unsigned long long* out) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  unsigned long long best = ~0ULL;
  for (long long c = warp * U; c * 32 < n; c += nw * U) {
    unsigned pw[U];
    unsigned long long gc[U], k0[U];
#pragma unroll
    for (int u = 0; u < U; ++u) pw[u] = (c + u) * 32 < n ? __ldg(present + c + u) : 0u;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned g = (unsigned)((c + u) * 32 + lane);
      gc[u] = ((pw[u] >> lane) & 1u) ? __ldg(cnt + g) : 0ULL;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned g = (unsigned)((c + u) * 32 + lane);
      k0[u] = gc[u] ? key_of(limbs, g) : ~0ULL;
      best = k0[u] < best ? k0[u] : best;
    }
  }
  for (int o = 16; o; o >>= 1) {
    unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o);
    best = x < best ? x : best;
  }
  if (lane == 0) atomicMin(out, best);
}

// V4: lane = slot, count and limbs loaded together (no dependency on count)
template <int U>
__global__ void walk_lane_spec(const unsigned* present, const unsigned long long* cnt, const unsigned long long* limbs,
                               long long n, unsigned long long* out) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  unsigned long long best = ~0ULL;
  for (long long c = warp * U; c * 32 < n; c += nw * U) {
    unsigned pw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) pw[u] = (c + u) * 32 < n ? __ldg(present + c + u) : 0u;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned g = (unsigned)((c + u) * 32 + lane);
      const bool p = (pw[u] >> lane) & 1u;
      const unsigned long long gc = p ? __ldg(cnt + g) : 0ULL;
      const unsigned long long k = p ? key_of(limbs, g) : ~0ULL;
      const unsigned long long k0 = gc ? k : ~0ULL;
      best = k0 < best ? k0 : best;
    }
  }
  for (int o = 16; o; o >>= 1) {
    unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o);
    best = x < best ? x : best;
  }
  if (lane == 0) atomicMin(out, best);
}

// V1: compaction of a 1024-slot super-chunk into shared memory, then batches
__global__ void walk_compact(const unsigned* present, const unsigned long long* cnt, const unsigned long long* limbs,
                             long long n, unsigned long long* out) {
  __shared__ unsigned s_slot[8][1024];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned* sidx = s_slot[warp];
  unsigned long long best = ~0ULL;
  for (long long sb = blockIdx.x * 8LL + warp; sb * 1024 < n; sb += gridDim.x * 8LL) {
    const long long base = sb * 1024, wbase = base + 32LL * lane;
    unsigned w = wbase < n ? __ldg(present + (wbase >> 5)) : 0u;
    const int c = __popc(w);
    int off = c;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, off, o);
      if (lane >= o) off += y;
    }
    const int total = __shfl_sync(0xffffffffu, off, 31);
    off -= c;
    while (w) {
      const int bit = __ffs(w) - 1;
      w &= w - 1;
      sidx[off++] = (unsigned)(wbase - base) + bit;
    }
    __syncwarp();
    for (int c0 = 0; c0 < total; c0 += 128) {
      unsigned long long gc[4];
      unsigned gq[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = c0 + u * 32 + lane;
        gq[u] = i < total ? (unsigned)base + sidx[i] : 0u;
        gc[u] = i < total ? __ldg(cnt + gq[u]) : 0ULL;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const unsigned long long k0 = gc[u] ? key_of(limbs, gq[u]) : ~0ULL;
        best = k0 < best ? k0 : best;
      }
    }
    __syncwarp();
  }
  for (int o = 16; o; o >>= 1) {
    unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o);
    best = x < best ? x : best;
  }
  if (lane == 0) atomicMin(out, best);
}

int main() {
  const long long n = 15000000;
  const long long words = (n + 31) / 32;
  std::vector<unsigned> hp(words, 0);
  std::vector<unsigned long long> hc(n, 0);
  std::mt19937_64 rng(7);
  for (long long i = 0; i < n; ++i) {
    if (rng() % 100 < 10) {
      hp[i >> 5] |= 1u << (i & 31);
      hc[i] = (rng() % 5 == 0) ? 1 + rng() % 7 : 0;
    } else {
      hc[i] = rng();  // garbage where absent
    }
  }
  unsigned* dp;
  unsigned long long *dc, *dl, *dout;
  cudaMalloc(&dp, words * 4);
  cudaMalloc(&dc, n * 8);
  cudaMalloc(&dl, n * 24);
  cudaMalloc(&dout, 8);
  cudaMemcpy(dp, hp.data(), words * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, hc.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemset(dl, 0x11, n * 24);
  void* flush;
  cudaMalloc(&flush, 512 << 20);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time = [&](const char* name, auto launch) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaMemset(flush, r, 512 << 20);  // evict L2
      cudaMemset(dout, 0xff, 8);
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    unsigned long long o;
    cudaMemcpy(&o, dout, 8, cudaMemcpyDeviceToHost);
    printf("%-34s %8.1f us  (%llx) %s\n", name, best * 1e3, o, cudaGetErrorString(cudaGetLastError()));
  };
  for (int bps : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, sizeof nm, "compact1024 256t x %d/SM", bps);
    time(nm, [&] { walk_compact<<<sms * bps, 256>>>(dp, dc, dl, n, dout); });
    snprintf(nm, sizeof nm, "lane U1 256t x %d/SM", bps);
    time(nm, [&] { walk_lane<1><<<sms * bps, 256>>>(dp, dc, dl, n, dout); });
    snprintf(nm, sizeof nm, "lane U4 256t x %d/SM", bps);
    time(nm, [&] { walk_lane<4><<<sms * bps, 256>>>(dp, dc, dl, n, dout); });
    snprintf(nm, sizeof nm, "lane-spec U4 256t x %d/SM", bps);
    time(nm, [&] { walk_lane_spec<4><<<sms * bps, 256>>>(dp, dc, dl, n, dout); });
  }
  return 0;
}
