// Streaming-bandwidth probe for the fact-scan design space on B200:
//   mode 0: 1-D bulk TMA (cp.async.bulk) ring, 1 producer lane + consumer warps
//   mode 1: plain 128-bit vector loads, grid-stride, U-way unrolled
// Reads `ncols` columns of `rows` x 8 B, sums them (so nothing is dead).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe tools/bw_probe.cu
//   ./bw_probe rows ncols tile_rows stages consumers
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k_tma(const double* const* cols, int ncols, long long rows, int tile_rows, int stages, double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned long long* full = (unsigned long long*)smem;
  unsigned long long* empty = full + 16;
  unsigned char* st = smem + 256;
  const int stage_bytes = tile_rows * 8 * ncols;
  const int nconsumer_warps = blockDim.x / 32 - 1;
  const long long ntiles = (rows + tile_rows - 1) / tile_rows;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[i])), "r"(nconsumer_warps));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  double acc = 0;
  if (warp == 0) {
    if (lane == 0) {
      long long it = 0;
      for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        int s = it % stages;
        if (it >= stages) {
          unsigned ph = ((it / stages) - 1) & 1;
          asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(
                           smem_u32(&empty[s])),
                       "r"(ph));
        }
        long long r0 = t * tile_rows;
        long long nr = rows - r0 < tile_rows ? rows - r0 : tile_rows;
        unsigned bytes = (unsigned)(nr * 8);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                     "r"(bytes * ncols));
        for (int c = 0; c < ncols; ++c) {
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           smem_u32(st + s * stage_bytes + c * tile_rows * 8)),
                       "l"(cols[c] + r0), "r"(bytes), "r"(smem_u32(&full[s])));
        }
      }
    }
  } else {
    const int ct = threadIdx.x - 32, nct = blockDim.x - 32;
    long long it = 0;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      int s = it % stages;
      unsigned ph = (it / stages) & 1;
      asm volatile("{.reg .pred p; W2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W2;}" ::"r"(
                       smem_u32(&full[s])),
                   "r"(ph));
      const double* base = (const double*)(st + s * stage_bytes);
      for (int c = 0; c < ncols; ++c)
        for (int r = ct; r < tile_rows; r += nct) acc += base[c * tile_rows + r];
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])));
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

template <int U>
__global__ void k_ldg(const double* const* cols, int ncols, long long rows, double* out) {
  double acc = 0;
  const long long npairs = rows / 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < npairs; q += stride * U) {
    double2 v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (c < ncols && q + u * stride < npairs) v[u][c] = __ldg((const double2*)cols[c] + q + u * stride);
        else v[u][c] = make_double2(0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc += v[u][c].x + v[u][c].y;
  }
  if (acc == 12345.678) out[0] = acc;
}

int main(int argc, char** argv) {
  long long rows = argc > 1 ? atoll(argv[1]) : 60000000LL;
  int ncols = argc > 2 ? atoi(argv[2]) : 4;
  int tile_rows = argc > 3 ? atoi(argv[3]) : 1024;
  int stages = argc > 4 ? atoi(argv[4]) : 6;
  int consumers = argc > 5 ? atoi(argv[5]) : 8;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* cols[8];
  for (int c = 0; c < ncols; ++c) {
    cudaMalloc(&cols[c], rows * 8);
    cudaMemset(cols[c], 0, rows * 8);
  }
  double** dcols;
  cudaMalloc(&dcols, sizeof(cols));
  cudaMemcpy(dcols, cols, sizeof(cols), cudaMemcpyHostToDevice);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double bytes = (double)rows * 8 * ncols;
  size_t smem = 256 + (size_t)stages * tile_rows * 8 * ncols;
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k_tma<<<sms, 32 * (consumers + 1), smem>>>(dcols, ncols, rows, tile_rows, stages, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("tma  tile=%d stages=%d consumers=%d : %.3f ms  %.0f GB/s  (%s)\n", tile_rows, stages, consumers, ms,
           bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k_ldg<4><<<sms * 8, 256>>>(dcols, ncols, rows, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("ldg  U=4 grid=%d: %.3f ms  %.0f GB/s\n", sms * 8, ms, bytes / ms / 1e6);
  }
  return 0;
}
