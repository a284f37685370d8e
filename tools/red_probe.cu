// Throughput of non-returning 64-bit global atomics (RED.E.ADD.64) on the
// B200: the bound of the hash-group scan (qg: 5 REDs per passing row into a
// 40-byte group record). Rows pick a group by a multiplicative hash (random
// slots, as l_partkey) or sequentially; each row adds to K consecutive words
// of its record (record stride S words).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/red_probe tools/red_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_red(unsigned long long* t, long long groups, long long rows, int k, int stride, int seq) {
  const long long n = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += n) {
    const unsigned long long h = seq ? static_cast<unsigned long long>(r) : static_cast<unsigned long long>(r) * 0x9E3779B97F4A7C15ULL;
    const long long g = seq ? static_cast<long long>(h % groups) : static_cast<long long>((h >> 20) % groups);
    unsigned long long* p = t + g * stride;
    for (int j = 0; j < k; ++j)
      asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p + j), "l"(static_cast<unsigned long long>(r)) : "memory");
  }
}

int main() {
  const long long rows = 35000000;
  unsigned long long* t;
  cudaMalloc(&t, 16ull << 30 >> 4 << 4);  // 1 GB
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Cfg { long long groups; int k, stride, seq; };
  const Cfg cfgs[] = {
      {2000000, 5, 5, 0}, {2000000, 1, 5, 0}, {2000000, 3, 3, 0}, {2000000, 4, 4, 0}, {2000000, 5, 8, 0},
      {2000000, 1, 1, 0}, {2000000, 1, 4, 0}, {2000000, 2, 2, 0}, {200000, 5, 5, 0}, {20000000, 5, 5, 0},
      {2000000, 5, 5, 1}, {2000000, 1, 1, 1}, {2000000, 1, 4, 1}};
  for (const Cfg& c : cfgs) {
    for (int blocks : {148 * 4, 148 * 8}) {
      cudaMemset(t, 0, c.groups * c.stride * 8);
      k_red<<<blocks, 256>>>(t, c.groups, rows, c.k, c.stride, c.seq);
      cudaEventRecord(a);
      for (int i = 0; i < 5; ++i) k_red<<<blocks, 256>>>(t, c.groups, rows, c.k, c.stride, c.seq);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ms /= 5;
      printf("groups %9lld k %d stride %d %s blocks %4d: %.3f ms  %.1f G red/s  %.1f G rows/s\n", c.groups, c.k,
             c.stride, c.seq ? "seq " : "hash", blocks, ms, rows * c.k / (ms * 1e6), rows / (ms * 1e6));
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
