// Host cost of single stream-ordered calls on an idle GPU (each call timed
// alone, the stream synchronised before it): kernel launches by parameter
// size, memset, pool alloc/free, 32 B D2H + stream sync, graph launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/launch_probe tools/launch_probe.cu
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

template <int W> struct Blob { unsigned long long w[W]; };
__global__ void k_small(int x, int* o) { if (x < 0) *o = x; }
template <int W> __global__ void k_blob(Blob<W> b, int* o) { if (b.w[3] == 7) *o = 1; }

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  int* o;
  cudaMalloc(&o, 64);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  auto bench = [&](const char* name, auto&& f) {
    std::vector<double> v;
    for (int i = 0; i < 300; ++i) {
      cudaStreamSynchronize(s);
      const double t0 = now_us();
      f();
      v.push_back(now_us() - t0);
    }
    cudaStreamSynchronize(s);
    std::sort(v.begin(), v.end());
    printf("%-44s median %6.2f us  p10 %6.2f\n", name, v[v.size() / 2], v[v.size() / 10]);
  };
  Blob<128> b1{};
  Blob<256> b2{};
  Blob<420> b3{};
  Blob<1000> b4{};
  bench("launch, 4 B param", [&] { k_small<<<148, 256, 0, s>>>(1, o); });
  bench("launch, 1 KB param", [&] { k_blob<128><<<148, 256, 0, s>>>(b1, o); });
  bench("launch, 2 KB param", [&] { k_blob<256><<<148, 256, 0, s>>>(b2, o); });
  bench("launch, 3.4 KB param", [&] { k_blob<420><<<148, 256, 0, s>>>(b3, o); });
  bench("launch, 8 KB param", [&] { k_blob<1000><<<148, 256, 0, s>>>(b4, o); });
  bench("2 launches 3.4 KB back to back", [&] { k_blob<420><<<148, 256, 0, s>>>(b3, o); k_blob<420><<<148, 256, 0, s>>>(b3, o); });
  cudaMemPool_t pool;
  cudaDeviceGetDefaultMemPool(&pool, 0);
  unsigned long long thr = ~0ULL;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  void* p = nullptr;
  bench("cudaMallocFromPoolAsync 64 MB", [&] { cudaMallocFromPoolAsync(&p, 64 << 20, pool, s); });
  cudaFreeAsync(p, s);
  void* m;
  cudaMalloc(&m, 16 << 20);
  bench("cudaMemsetAsync 4 KB", [&] { cudaMemsetAsync(m, 0, 4096, s); });
  long long* h;
  cudaMallocHost(&h, 64);
  bench("D2H 32 B pinned + cudaStreamSynchronize", [&] {
    cudaMemcpyAsync(h, o, 32, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
  });
  bench("cudaStreamSynchronize (idle)", [&] { cudaStreamSynchronize(s); });
  bench("launch 4 B + cudaStreamSynchronize", [&] {
    k_small<<<1, 32, 0, s>>>(1, o);
    cudaStreamSynchronize(s);
  });
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  cudaMemsetAsync(m, 0, 4096, s);
  for (int i = 0; i < 4; ++i) k_blob<420><<<148, 256, 0, s>>>(b3, o);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  bench("graph launch (memset + 4 x 3.4 KB kernels)", [&] { cudaGraphLaunch(ge, s); });
  return 0;
}
