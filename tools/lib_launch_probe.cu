// Host cost of launching a run-time loaded (library) kernel, as the NVRTC
// pipeline kernels are: cudaLaunchKernel with the cudaKernel_t vs the
// driver's cuLaunchKernel with the CUfunction of the current context.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lib_launch_probe tools/lib_launch_probe.cu -lcuda
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <vector>
struct Blob { unsigned long long w[420]; };
static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
int main(int argc, char** argv) {
  int* o;
  cudaMalloc(&o, 64);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaLibrary_t lib;
  if (cudaLibraryLoadFromFile(&lib, argc > 1 ? argv[1] : "tools/_blob.cubin", nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess) { printf("load failed\n"); return 1; }
  cudaKernel_t k;
  cudaLibraryGetKernel(&k, lib, "k_lib");
  CUfunction f;
  cuKernelGetFunction(&f, reinterpret_cast<CUkernel>(k));
  Blob b{};
  void* args[] = {&b, &o};
  auto bench = [&](const char* name, auto&& fn) {
    std::vector<double> v;
    for (int i = 0; i < 300; ++i) {
      cudaStreamSynchronize(s);
      const double t0 = now_us();
      fn();
      v.push_back(now_us() - t0);
    }
    cudaStreamSynchronize(s);
    std::sort(v.begin(), v.end());
    printf("%-48s median %6.2f us  p10 %6.2f\n", name, v[v.size() / 2], v[v.size() / 10]);
  };
  bench("cudaLaunchKernel(cudaKernel_t), 3.4 KB", [&] { cudaLaunchKernel((const void*)k, dim3(148), dim3(256), args, 0, s); });
  bench("cuLaunchKernel(CUfunction), 3.4 KB", [&] { cuLaunchKernel(f, 148, 1, 1, 256, 1, 1, 0, (CUstream)s, args, nullptr); });
  bench("2x cudaLaunchKernel(cudaKernel_t)", [&] { cudaLaunchKernel((const void*)k, dim3(148), dim3(256), args, 0, s); cudaLaunchKernel((const void*)k, dim3(148), dim3(256), args, 0, s); });
  bench("2x cuLaunchKernel(CUfunction)", [&] { cuLaunchKernel(f, 148, 1, 1, 256, 1, 1, 0, (CUstream)s, args, nullptr); cuLaunchKernel(f, 148, 1, 1, 256, 1, 1, 0, (CUstream)s, args, nullptr); });
  return 0;
}
