// i128_to_f64_rn (fz_layout.cuh) against the compiler's __int128 -> double
// conversion on random and edge values (bit-identical expected):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//     -Iinclude -Ipaper_2209_04579_b200/csrc -o tools/i128_check tools/i128_check.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "fz_layout.cuh"
using namespace tqp::fz;

__global__ void k_check(unsigned long long seed, long long n, unsigned long long* bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long x = seed + i * 0x9E3779B97F4A7C15ULL;
    auto mix = [](unsigned long long z) {
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
      return z ^ (z >> 31);
    };
    const unsigned long long a = mix(x), b = mix(x + 1), c = mix(x + 2);
    unsigned __int128 u = (static_cast<unsigned __int128>(a) << 64) | b;
    const int sh = static_cast<int>(c % 128);  // every magnitude
    u >>= sh;
    if (c & (1ULL << 40)) u |= 1;                          // sticky-only patterns
    if (c & (1ULL << 41)) u &= ~static_cast<unsigned __int128>(0x3ff);  // exact ties
    if (c & (1ULL << 42)) u = (u >> 11) << 11 | (static_cast<unsigned __int128>(1) << 10);  // halfway cases
    __int128 v = static_cast<__int128>(u);
    if (c & (1ULL << 43)) v = -v;
    const double want = static_cast<double>(v), got = i128_to_f64_rn(v);
    if (__double_as_longlong(want) != __double_as_longlong(got)) atomicAdd(bad, 1ULL);
  }
}

int main() {
  unsigned long long* bad;
  cudaMallocManaged(&bad, 8);
  *bad = 0;
  const long long n = 1LL << 30;
  k_check<<<148 * 8, 256>>>(12345, n, bad);
  cudaDeviceSynchronize();
  printf("i128_to_f64_rn: %lld values, %llu mismatches (%s)\n", n, *bad, cudaGetErrorString(cudaGetLastError()));
  return *bad != 0;
}
