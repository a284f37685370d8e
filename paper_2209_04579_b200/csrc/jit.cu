// NVRTC front end for the specialised pipeline kernels (jit.hpp).
//
// NVRTC is bound at run time from the toolkit this library was built with
// (dlopen by absolute path, RTLD_LOCAL), not through the dynamic linker: a
// process that imported torch first already holds torch's bundled
// libnvrtc.so.12 (12.8), and an ordinary -lnvrtc would bind to that one by
// SONAME. The generated kernels must not depend on import order - the Q1
// register-accumulator kernel measured 365 us with NVRTC 12.9 and 458 us
// with 12.8 on the same B200.
#include <dlfcn.h>
#include <nvrtc.h>

#include <atomic>
#include <cstdlib>
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

// Compiled kernels, least-recently-used bounded: a long-lived process that
// keeps meeting new predicates (every literal is part of a kernel's source)
// would otherwise keep every code object loaded. At the bound (TQP_JIT_CACHE
// libraries, default 512) the least recently requested library is unloaded
// after a device synchronisation (no launch of it can be in flight); the
// epoch counter tells kernel-pointer caches (the per-unit memo, Ctx's
// attribute caches) to drop what they hold.
struct Entry {
  const void* fn = nullptr;
  cudaLibrary_t lib = nullptr;
  unsigned long long tick = 0;
};
struct Cache {
  std::mutex mu;
  std::map<std::string, Entry> kernels;  // key: entry + '\0' + source
  unsigned long long tick = 0;
  size_t cap = 0;
};
std::atomic<long long> g_epoch{0};

Cache& cache() {
  static Cache c;
  return c;
}

#ifndef TQP_NVRTC_PATH
#define TQP_NVRTC_PATH "/usr/local/cuda/lib64/libnvrtc.so.12"
#endif

struct Nvrtc {
  const char* (*GetErrorString)(nvrtcResult);
  nvrtcResult (*Version)(int*, int*);
  nvrtcResult (*CreateProgram)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*);
  nvrtcResult (*CompileProgram)(nvrtcProgram, int, const char* const*);
  nvrtcResult (*GetProgramLogSize)(nvrtcProgram, size_t*);
  nvrtcResult (*GetProgramLog)(nvrtcProgram, char*);
  nvrtcResult (*GetCUBINSize)(nvrtcProgram, size_t*);
  nvrtcResult (*GetCUBIN)(nvrtcProgram, char*);
  nvrtcResult (*DestroyProgram)(nvrtcProgram*);
  int major = 0, minor = 0;
};

// TQP_NVRTC (environment) overrides the library path
const Nvrtc& nvrtc() {
  static const Nvrtc api = [] {
    const char* env = std::getenv("TQP_NVRTC");
    const char* path = env && *env ? env : TQP_NVRTC_PATH;
    void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) throw Error(TQP_ERR_CUDA, std::string("nvrtc: cannot load ") + path + ": " + dlerror());
    Nvrtc a{};
    auto sym = [&](const char* name) {
      void* f = dlsym(h, name);
      if (!f) throw Error(TQP_ERR_CUDA, std::string("nvrtc: missing symbol ") + name + " in " + path);
      return f;
    };
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("nvrtcGetErrorString"));
    a.Version = reinterpret_cast<decltype(a.Version)>(sym("nvrtcVersion"));
    a.CreateProgram = reinterpret_cast<decltype(a.CreateProgram)>(sym("nvrtcCreateProgram"));
    a.CompileProgram = reinterpret_cast<decltype(a.CompileProgram)>(sym("nvrtcCompileProgram"));
    a.GetProgramLogSize = reinterpret_cast<decltype(a.GetProgramLogSize)>(sym("nvrtcGetProgramLogSize"));
    a.GetProgramLog = reinterpret_cast<decltype(a.GetProgramLog)>(sym("nvrtcGetProgramLog"));
    a.GetCUBINSize = reinterpret_cast<decltype(a.GetCUBINSize)>(sym("nvrtcGetCUBINSize"));
    a.GetCUBIN = reinterpret_cast<decltype(a.GetCUBIN)>(sym("nvrtcGetCUBIN"));
    a.DestroyProgram = reinterpret_cast<decltype(a.DestroyProgram)>(sym("nvrtcDestroyProgram"));
    a.Version(&a.major, &a.minor);
    return a;
  }();
  return api;
}

void nvrtc_check(nvrtcResult r, const char* what) {
  if (r != NVRTC_SUCCESS)
    throw Error(TQP_ERR_CUDA, std::string("nvrtc: ") + nvrtc().GetErrorString(r) + " in " + what);
}

}  // namespace

int jit_nvrtc_version() {
  const Nvrtc& a = nvrtc();
  return a.major * 1000 + a.minor * 10;
}

const void* jit_kernel(const std::string& src, const char* entry) {
  Cache& c = cache();
  std::lock_guard<std::mutex> lock(c.mu);
  const std::string key = std::string(entry) + '\0' + src;
  auto it = c.kernels.find(key);
  if (it != c.kernels.end()) {
    it->second.tick = ++c.tick;
    return it->second.fn;
  }
  if (!c.cap) {
    const char* e = std::getenv("TQP_JIT_CACHE");
    c.cap = e && std::atoi(e) > 0 ? static_cast<size_t>(std::atoi(e)) : 512;
  }
  while (c.kernels.size() >= c.cap) {
    auto lru = c.kernels.begin();
    for (auto j = c.kernels.begin(); j != c.kernels.end(); ++j)
      if (j->second.tick < lru->second.tick) lru = j;
    TQP_CUDA(cudaDeviceSynchronize());
    TQP_CUDA(cudaLibraryUnload(lru->second.lib));
    c.kernels.erase(lru);
    ++g_epoch;
  }

  const Nvrtc& api = nvrtc();
  nvrtcProgram prog;
  nvrtc_check(api.CreateProgram(&prog, src.c_str(), "tqp_pipeline.cu", kJitHeaderCount, kJitHeaderSrc, kJitHeaderNames),
              "nvrtcCreateProgram");
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--device-int128", "-lineinfo",
                        "-default-device", "--extra-device-vectorization"};
  nvrtcResult r = api.CompileProgram(prog, static_cast<int>(sizeof(opts) / sizeof(opts[0])), opts);
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    api.GetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    if (n) api.GetProgramLog(prog, &log[0]);
    api.DestroyProgram(&prog);
    throw Error(TQP_ERR_CUDA, "nvrtc failed to compile a pipeline kernel:\n" + log.substr(0, 1500));
  }
  size_t n = 0;
  nvrtc_check(api.GetCUBINSize(prog, &n), "nvrtcGetCUBINSize");
  std::vector<char> cubin(n);
  nvrtc_check(api.GetCUBIN(prog, cubin.data()), "nvrtcGetCUBIN");
  api.DestroyProgram(&prog);

  cudaLibrary_t lib;
  TQP_CUDA(cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
  cudaKernel_t k;
  TQP_CUDA(cudaLibraryGetKernel(&k, lib, entry));
  const void* fn = reinterpret_cast<const void*>(k);
  c.kernels[key] = Entry{fn, lib, ++c.tick};
  return fn;
}

long long jit_epoch() { return g_epoch.load(); }

int jit_compiled_count() {
  Cache& c = cache();
  std::lock_guard<std::mutex> lock(c.mu);
  return static_cast<int>(c.kernels.size());
}

}  // namespace tqp
