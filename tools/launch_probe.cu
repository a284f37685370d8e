// Host cost of one kernel launch by kind (static kernel vs a library kernel
// loaded at run time, small vs 2 KB parameter struct) and of the other
// stream-ordered calls a fused unit makes (memset, pool alloc/free, 32 B
// D2H + stream sync).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/launch_probe tools/launch_probe.cu -lcuda
#include <chrono>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <vector>

struct Big { unsigned long long w[256]; };
__global__ void k_small(int x, int* o) { if (x < 0) *o = x; }
__global__ void k_big(Big b, int* o) { if (b.w[3] == 7) *o = 1; }

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  int* o;
  cudaMalloc(&o, 64);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  Big b{};
  const int N = 2000;
  auto bench = [&](const char* name, auto&& f) {
    for (int i = 0; i < 100; ++i) f();
    cudaStreamSynchronize(s);
    double t0 = now_us();
    for (int i = 0; i < N; ++i) f();
    double t1 = now_us();
    cudaStreamSynchronize(s);
    printf("%-40s %7.2f us/call\n", name, (t1 - t0) / N);
  };
  bench("static kernel, 4 B arg", [&] { k_small<<<148, 256, 0, s>>>(1, o); });
  bench("static kernel, 2 KB struct arg", [&] { k_big<<<148, 256, 0, s>>>(b, o); });
  // the same kernels through the runtime's library API (as NVRTC cubins are)
  cudaLibrary_t lib;
  // load this binary's own module via cudaGetFuncBySymbol instead: library API needs a cubin image,
  // so approximate with cudaLaunchKernel on the function pointer
  bench("cudaLaunchKernel, 2 KB struct", [&] {
    void* args[] = {&b, &o};
    cudaLaunchKernel((const void*)k_big, dim3(148), dim3(256), args, 0, s);
  });
  (void)lib;
  cudaMemPool_t pool;
  cudaDeviceGetDefaultMemPool(&pool, 0);
  unsigned long long thr = ~0ULL;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  void* p = nullptr;
  bench("cudaMallocFromPoolAsync+cudaFreeAsync 64MB", [&] {
    cudaMallocFromPoolAsync(&p, 64 << 20, pool, s);
    cudaFreeAsync(p, s);
  });
  void* m;
  cudaMalloc(&m, 16 << 20);
  bench("cudaMemsetAsync 4 KB", [&] { cudaMemsetAsync(m, 0, 4096, s); });
  bench("cudaMemsetAsync 15 MB", [&] { cudaMemsetAsync(m, 0, 15 << 20, s); });
  long long* h;
  cudaMallocHost(&h, 64);
  bench("D2H 32 B pinned + cudaStreamSynchronize", [&] {
    cudaMemcpyAsync(h, o, 32, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
  });
  bench("empty kernel + cudaStreamSynchronize", [&] {
    k_small<<<1, 32, 0, s>>>(1, o);
    cudaStreamSynchronize(s);
  });
  cudaEvent_t e;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  bench("cudaEventRecord", [&] { cudaEventRecord(e, s); });
  // graph of 4 kernels + memset
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  cudaMemsetAsync(m, 0, 4096, s);
  for (int i = 0; i < 4; ++i) k_big<<<148, 256, 0, s>>>(b, o);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  bench("graph launch (memset + 4 kernels)", [&] { cudaGraphLaunch(ge, s); });
  return 0;
}
