// Micro-benchmark: cost of a warp-level k-way merge of 8 sorted lists in
// shared memory (the top-k block merge, csrc/fused.cu merge_lists), timed with
// clock64 inside the kernel, 1 block per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/merge_probe tools/merge_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int kW>
__device__ __forceinline__ unsigned long long merge(const unsigned long long (*lists)[32], const int* len, int k, int& cnt) {
  const int lane = threadIdx.x & 31;
  int hp = 0;
  unsigned long long out = ~0ULL;
  cnt = 0;
  for (int r = 0; r < k; ++r) {
    unsigned long long hv = lane < kW && hp < len[lane] ? lists[lane][hp] : ~0ULL;
    int hl = lane < kW && hp < len[lane] ? lane : 32;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ov = __shfl_xor_sync(0xffffffffu, hv, o);
      const int ol = __shfl_xor_sync(0xffffffffu, hl, o);
      if (ov < hv || (ov == hv && ol < hl)) { hv = ov; hl = ol; }
    }
    if (hl == 32) break;
    if (lane == hl) ++hp;
    if (lane == r) out = hv;
    ++cnt;
  }
  return out;
}

__global__ void k_probe(int k, long long* cyc, unsigned long long* sink, int mode) {
  __shared__ unsigned long long s_wv[8][32];
  __shared__ int s_wn[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  s_wv[warp][lane] = (unsigned long long)(blockIdx.x * 7919 + warp * 131 + lane * 17) * 2654435761ULL;
  if (lane == 0) s_wn[warp] = 10;
  __syncthreads();
  if (warp == 0) {
    long long t0 = clock64();
    int cnt;
    unsigned long long v = 0;
    if (mode == 0) v = merge<8>(s_wv, s_wn, k, cnt);
    else {
      unsigned long long x = s_wv[0][lane];
      for (int i = 0; i < 50; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1 + (i & 15)) + 1;
      v = x;
    }
    long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * 32 + lane] = v;
  }
}

int main() {
  long long* cyc; unsigned long long* sink;
  cudaMalloc(&cyc, 148 * 8); cudaMalloc(&sink, 148 * 32 * 8);
  for (int mode = 0; mode < 2; ++mode)
    for (int it = 0; it < 3; ++it) {
      k_probe<<<148, 256>>>(10, cyc, sink, mode);
      long long h[148];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0, mn = 1LL << 60;
      for (int i = 0; i < 148; ++i) { mx = h[i] > mx ? h[i] : mx; mn = h[i] < mn ? h[i] : mn; }
      printf("mode %d (%s): cycles min %lld max %lld\n", mode, mode ? "50 dependent shfl" : "merge k=10", mn, mx);
    }
  return 0;
}
