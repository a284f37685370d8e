// Run-time specialised pipeline kernels: NVRTC compiles a generated kernel
// (fused.cu's generator + jit_tile.cuh) for sm_100a once per distinct source
// per process; the cubin is loaded with cudaLibraryLoadData and launched like
// any other kernel (the handle is a `const void*` for cudaLaunchKernel).
#pragma once

#include <string>

namespace tqp {

// Compiles (or returns the cached) kernel `entry` of `src`. Throws Error
// (TQP_ERR_CUDA) with the NVRTC log on failure.
const void* jit_kernel(const std::string& src, const char* entry);

// Number of kernels currently loaded (at most TQP_JIT_CACHE, default 512).
int jit_compiled_count();

// Incremented whenever a least-recently-used kernel library is unloaded:
// holders of kernel pointers re-fetch (jit_kernel) when it changed.
long long jit_epoch();

// Version of the NVRTC the kernels are compiled with (major * 1000 + minor * 10).
int jit_nvrtc_version();

}  // namespace tqp
