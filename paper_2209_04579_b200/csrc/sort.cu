// Stable LSD radix sort (8-bit digits) replacing the reference's serial
// std::stable_sort (argsort_stable, kernels.cpp:411-424) and the per-byte
// refinement passes of SortPermRows (executor.cpp:44-68).
//
// Per pass: a per-tile digit histogram, one decoupled-lookback scan over the
// digit-major (digit, tile) counts, and a stable scatter where each warp
// ranks equal digits with __match_any_sync and tiles are processed in row
// order. Passes whose digit is constant over all keys are skipped (found by
// an OR-reduction of key ^ key[0]), so a 1-byte string column costs one
// pass and dense int64 keys only their varying low bytes.
#include <string>

#include "scan.cuh"

namespace tqp {
namespace k {
Tensor prefix_sum_raw(Ctx& c, const Tensor& x, int64_t* first_overflow);
}
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;

template <typename T>
__global__ void k_make_keys(const T* __restrict__ col, const int64_t* __restrict__ perm, int64_t n, int64_t m,
                            int64_t j, bool desc, uint64_t* __restrict__ out, long long* err) {
  for (int64_t i = gtid(); i < n; i += gstride()) {
    int64_t r = perm ? perm[i] : i;
    T v = col[r * m + j];
    if constexpr (std::is_same_v<T, double>) {
      if (isnan(v)) note_bad(err, i);
    }
    uint64_t u = radix_key(v);
    out[i] = desc ? ~u : u;
  }
}

__global__ void k_diff_or(const uint64_t* __restrict__ keys, int64_t n, unsigned long long* out) {
  uint64_t first = keys[0];
  uint64_t acc = 0;
  for (int64_t i = gtid(); i < n; i += gstride()) acc |= keys[i] ^ first;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc |= __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicOr(out, static_cast<unsigned long long>(acc));
}

__global__ void k_perm_bounds(const int64_t* __restrict__ p, int64_t n, int64_t rows, long long* err) {
  for (int64_t i = gtid(); i < n; i += gstride())
    if (p[i] < 0 || p[i] >= rows) note_bad(err, i);
}

__global__ void k_identity(int64_t* __restrict__ p, int64_t n) {
  for (int64_t i = gtid(); i < n; i += gstride()) p[i] = i;
}

__global__ void __launch_bounds__(kThreads) k_hist(const uint64_t* __restrict__ keys, int64_t n, int shift,
                                                   int64_t tiles, int64_t* __restrict__ counts) {
  __shared__ unsigned int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
#pragma unroll 4
  for (int j = 0; j < kItems; ++j) {
    int64_t i = base + j * kThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255], 1u);
  }
  __syncthreads();
  counts[static_cast<int64_t>(threadIdx.x) * tiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kThreads) k_scatter(const uint64_t* __restrict__ kin, const int64_t* __restrict__ pin,
                                                      uint64_t* __restrict__ kout, int64_t* __restrict__ pout, int64_t n,
                                                      int shift, int64_t tiles, const int64_t* __restrict__ offs) {
  __shared__ long long s_run[256];
  __shared__ long long s_w[kWarps][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  s_run[threadIdx.x] = offs[static_cast<int64_t>(threadIdx.x) * tiles + blockIdx.x];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
  const unsigned lt = (1u << lane) - 1u;
  for (int j = 0; j < kItems; ++j) {
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s_w[w][threadIdx.x] = 0;
    __syncthreads();
    int64_t i = base + j * kThreads + threadIdx.x;
    bool valid = i < n;
    uint64_t key = valid ? kin[i] : 0;
    int64_t pay = valid ? pin[i] : 0;
    int d = valid ? static_cast<int>((key >> shift) & 255) : 256;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    int rank = __popc(peers & lt);
    if (valid && rank == 0) s_w[warp][d] = __popc(peers);
    __syncthreads();
    {
      int dd = threadIdx.x;
      long long run = s_run[dd];
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        long long cnt = s_w[w][dd];
        s_w[w][dd] = run;
        run += cnt;
      }
      s_run[dd] = run;
    }
    __syncthreads();
    if (valid) {
      long long dst = s_w[warp][d] + rank;
      kout[dst] = key;
      pout[dst] = pay;
    }
    __syncthreads();
  }
}

}  // namespace

namespace k {

// Sorts `payload` (int64 vector, or identity when null) by radix keys built
// from column j of `col` (gathered through `perm` when non-null).
Tensor radix_sort_cols(Ctx& c, const Tensor& col, int64_t j, const Tensor* perm, bool desc, const char* kernel) {
  int64_t n = perm ? perm->rows : col.rows;
  Tensor payload;
  if (perm) {
    payload = *perm;
  } else {
    payload = c.alloc(TQP_I64, n, 1);
    if (n) {
      k_identity<<<c.grid_for(n, 256), 256, 0, c.stream>>>(payload.ptr<int64_t>(), n);
      c.count_launch();
    }
  }
  if (n == 0) return payload;
  Tensor keys = c.alloc(TQP_I64, n, 1);
  c.reset_err();
  TQP_DISPATCH(col.dtype, T,
               k_make_keys<T><<<c.grid_for(n, 256), 256, 0, c.stream>>>(col.ptr<T>(), perm ? perm->ptr<int64_t>() : nullptr,
                                                                        n, col.cols, j, desc,
                                                                        reinterpret_cast<uint64_t*>(keys.data()), c.d_err));
  c.count_launch();
  if (c.read_err() >= 0) kernel_fail(std::string(kernel) + ": NaN in keys");
  if (n == 1) return payload;
  auto orbuf = c.alloc_bytes(8);
  TQP_CUDA(cudaMemsetAsync(orbuf->ptr, 0, 8, c.stream));
  k_diff_or<<<c.grid_for(n, 256, 1, 4), 256, 0, c.stream>>>(reinterpret_cast<uint64_t*>(keys.data()), n,
                                                             static_cast<unsigned long long*>(orbuf->ptr));
  c.count_launch();
  unsigned long long diff = 0;
  TQP_CUDA(cudaMemcpyAsync(&diff, orbuf->ptr, 8, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  if (!diff) return payload;
  int64_t tiles = (n + kTile - 1) / kTile;
  Tensor counts = c.alloc(TQP_I64, tiles * 256, 1);
  Tensor k2 = c.alloc(TQP_I64, n, 1), p2 = c.alloc(TQP_I64, n, 1);
  // payload may be shared with the caller (immutable): write to fresh buffers
  Tensor kin = keys, pin = payload, kout = k2, pout = p2;
  bool first = true;
  for (int shift = 0; shift < 64; shift += 8) {
    if (!((diff >> shift) & 255ULL)) continue;
    k_hist<<<tiles, kThreads, 0, c.stream>>>(reinterpret_cast<uint64_t*>(kin.data()), n, shift, tiles,
                                               counts.ptr<int64_t>());
    int64_t ovf;
    Tensor offs = prefix_sum_raw(c, counts, &ovf);
    k_scatter<<<tiles, kThreads, 0, c.stream>>>(reinterpret_cast<uint64_t*>(kin.data()), pin.ptr<int64_t>(),
                                                 reinterpret_cast<uint64_t*>(kout.data()), pout.ptr<int64_t>(), n, shift,
                                                 tiles, offs.ptr<int64_t>());
    c.count_launch(2);
    if (first) {
      // never overwrite the caller's payload: allocate a second ping buffer
      kin = kout;
      pin = pout;
      kout = c.alloc(TQP_I64, n, 1);
      pout = c.alloc(TQP_I64, n, 1);
      first = false;
    } else {
      std::swap(kin, kout);
      std::swap(pin, pout);
    }
  }
  return pin;
}

Tensor radix_sort_payload(Ctx& c, const Tensor& keys, const Tensor* perm, bool descending) {
  return radix_sort_cols(c, keys, 0, perm, descending, "argsort_stable");
}

Tensor argsort_stable(Ctx& c, const Tensor& keys) {
  if (!keys.is_vector()) kernel_fail("argsort_stable: expected a vector (m=1)");
  return radix_sort_cols(c, keys, 0, nullptr, false, "argsort_stable");
}

// SortPermRows (executor.cpp:44-68): one stable pass per key column, last
// column first; a descending pass is a stable descending sort, which is what
// reverse -> argsort -> flip computes.
Tensor sort_perm_rows(Ctx& c, const Tensor& key, const Tensor& perm, bool asc) {
  if (perm.dtype != TQP_I64) kernel_fail(std::string("gather: expected int64, got ") + dtype_name(perm.dtype));
  if (!perm.is_vector()) kernel_fail("gather: expected a vector (m=1)");
  if (perm.rows) {
    // the reference gathers the key column through perm (executor.cpp:51):
    // same bounds contract and message as gather
    c.reset_err();
    k_perm_bounds<<<c.grid_for(perm.rows, 256), 256, 0, c.stream>>>(perm.ptr<int64_t>(), perm.rows, key.rows, c.d_err);
    c.count_launch();
    int64_t bad = c.read_err();
    if (bad >= 0) {
      int64_t v = read_scalar<int64_t>(c, perm, bad);
      kernel_fail("gather: index " + std::to_string(v) + " at position " + std::to_string(bad) +
                      " out of bounds [0," + std::to_string(key.rows) + ")",
                  bad);
    }
  }
  Tensor p = perm;
  for (int64_t j = key.cols - 1; j >= 0; --j) p = radix_sort_cols(c, key, j, &p, !asc, "argsort_stable");
  return p;
}

}  // namespace k
}  // namespace tqp
