// NVRTC front end for the specialised pipeline kernels (jit.hpp).
#include <nvrtc.h>

#include <map>
#include <mutex>
#include <vector>

#include "jit.hpp"
#include "tqp_internal.hpp"

namespace tqp {
namespace {

// build.py embeds the headers the generated kernels include (jit_embed.inc):
// kJitHeaderNames / kJitHeaderSrc / kJitHeaderCount
#include "jit_embed.inc"

struct Cache {
  std::mutex mu;
  std::map<std::string, const void*> kernels;  // key: entry + '\0' + source
};

Cache& cache() {
  static Cache c;
  return c;
}

void nvrtc_check(nvrtcResult r, const char* what) {
  if (r != NVRTC_SUCCESS) throw Error(TQP_ERR_CUDA, std::string("nvrtc: ") + nvrtcGetErrorString(r) + " in " + what);
}

}  // namespace

const void* jit_kernel(const std::string& src, const char* entry) {
  Cache& c = cache();
  std::lock_guard<std::mutex> lock(c.mu);
  const std::string key = std::string(entry) + '\0' + src;
  auto it = c.kernels.find(key);
  if (it != c.kernels.end()) return it->second;

  nvrtcProgram prog;
  nvrtc_check(nvrtcCreateProgram(&prog, src.c_str(), "tqp_pipeline.cu", kJitHeaderCount, kJitHeaderSrc, kJitHeaderNames),
              "nvrtcCreateProgram");
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--device-int128", "-lineinfo",
                        "-default-device", "--extra-device-vectorization"};
  nvrtcResult r = nvrtcCompileProgram(prog, static_cast<int>(sizeof(opts) / sizeof(opts[0])), opts);
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    if (n) nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    throw Error(TQP_ERR_CUDA, "nvrtc failed to compile a pipeline kernel:\n" + log.substr(0, 1500));
  }
  size_t n = 0;
  nvrtc_check(nvrtcGetCUBINSize(prog, &n), "nvrtcGetCUBINSize");
  std::vector<char> cubin(n);
  nvrtc_check(nvrtcGetCUBIN(prog, cubin.data()), "nvrtcGetCUBIN");
  nvrtcDestroyProgram(&prog);

  cudaLibrary_t lib;
  TQP_CUDA(cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
  cudaKernel_t k;
  TQP_CUDA(cudaLibraryGetKernel(&k, lib, entry));
  const void* fn = reinterpret_cast<const void*>(k);
  c.kernels[key] = fn;  // libraries live for the process
  return fn;
}

int jit_compiled_count() {
  Cache& c = cache();
  std::lock_guard<std::mutex> lock(c.mu);
  return static_cast<int>(c.kernels.size());
}

}  // namespace tqp
