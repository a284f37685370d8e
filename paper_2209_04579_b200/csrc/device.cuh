// Device-side helpers shared by the kernel translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "tqp_internal.hpp"

namespace tqp {

constexpr long long kNoBad = 0x7fffffffffffffffLL;

// Error kinds written to Ctx::d_err[2] by kernels that can fail.
enum ErrKind : long long {
  EK_NONE = 0,
  EK_DIV0 = 1,
  EK_OVERFLOW = 2,
  EK_OOB = 3,
  EK_NAN = 4,
  EK_NOT_SORTED = 5,
  EK_NEG_COUNT = 6,
  EK_DECREASE = 7,
  EK_RANGE = 8,
  EK_EMPTY = 9,
};

__device__ __forceinline__ void note_bad(long long* err, long long i) {
  atomicMin(reinterpret_cast<long long*>(err), i);
}

__device__ __forceinline__ int64_t gtid() { return static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t gstride() { return static_cast<int64_t>(gridDim.x) * blockDim.x; }

// Signed-overflow-checked arithmetic (the __builtin_*_overflow contract of
// kernels.cpp:246-262): returns true on overflow, r gets the wrapped value.
__device__ __forceinline__ bool add_ovf(int64_t x, int64_t y, int64_t* r) {
  uint64_t u = static_cast<uint64_t>(x) + static_cast<uint64_t>(y);
  *r = static_cast<int64_t>(u);
  return ((x ^ *r) & (y ^ *r)) < 0;
}
__device__ __forceinline__ bool sub_ovf(int64_t x, int64_t y, int64_t* r) {
  uint64_t u = static_cast<uint64_t>(x) - static_cast<uint64_t>(y);
  *r = static_cast<int64_t>(u);
  return ((x ^ y) & (x ^ *r)) < 0;
}
__device__ __forceinline__ bool mul_ovf(int64_t x, int64_t y, int64_t* r) {
  int64_t lo = static_cast<int64_t>(static_cast<uint64_t>(x) * static_cast<uint64_t>(y));
  int64_t hi = __mul64hi(x, y);
  *r = lo;
  return hi != (lo >> 63);
}
__device__ __forceinline__ bool add_ovf(int32_t x, int32_t y, int32_t* r) {
  int64_t w = static_cast<int64_t>(x) + y;
  *r = static_cast<int32_t>(w);
  return w != *r;
}
__device__ __forceinline__ bool sub_ovf(int32_t x, int32_t y, int32_t* r) {
  int64_t w = static_cast<int64_t>(x) - y;
  *r = static_cast<int32_t>(w);
  return w != *r;
}
__device__ __forceinline__ bool mul_ovf(int32_t x, int32_t y, int32_t* r) {
  int64_t w = static_cast<int64_t>(x) * y;
  *r = static_cast<int32_t>(w);
  return w != *r;
}

// Order-preserving unsigned transform of sort keys (radix sort). Float64:
// -0.0 is canonicalised to +0.0 first because the reference's `<` treats
// them as equal (stable_sort keeps their input order, kernels.cpp:419-421).
__device__ __forceinline__ uint64_t radix_key(int64_t v) { return static_cast<uint64_t>(v) ^ 0x8000000000000000ULL; }
__device__ __forceinline__ uint64_t radix_key(int32_t v) { return static_cast<uint32_t>(v) ^ 0x80000000u; }
__device__ __forceinline__ uint64_t radix_key(uint8_t v) { return v; }
__device__ __forceinline__ uint64_t radix_key(double d) {
  if (d == 0.0) d = 0.0;
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(d));
  return (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace tqp

// dtype dispatch over the four reference dtypes (STR8 behaves as uint8 data)
#define TQP_DISPATCH(dtype, T, ...)                                    \
  switch (dtype) {                                                     \
    case TQP_BOOL:                                                     \
    case TQP_STR8: { using T = uint8_t; __VA_ARGS__; } break;          \
    case TQP_I32: { using T = int32_t; __VA_ARGS__; } break;           \
    case TQP_I64: { using T = int64_t; __VA_ARGS__; } break;           \
    case TQP_F64: { using T = double; __VA_ARGS__; } break;            \
    default: ::tqp::kernel_fail("bad dtype tag");                      \
  }
