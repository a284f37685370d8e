#include <cstdlib>
// Runtime: context, stream-ordered device memory, tensor upload/download.
// Replaces the reference's host-only storage (tensor.hpp:105-121) and the
// thread-pool backend (backend.cpp:27-178) with one CUDA stream per context
// and a stream-ordered memory pool; slots freed at their last use return
// memory to the pool without a device synchronisation.
#include <cstring>
#include <string>

#include "device.cuh"
#include "jit.hpp"

namespace tqp {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw Error(TQP_ERR_CUDA, std::string("cuda: ") + cudaGetErrorString(e) + " (" + what + ")");
  }
}

DevBuf::~DevBuf() {
  if (ready) {  // never used on the context stream: free after the producer
    if (ctx) cudaStreamWaitEvent(ctx->stream, ready, 0);
    cudaEventDestroy(ready);
    ready = nullptr;
  }
  if (!ptr || !ctx) return;
  if (bucket >= 0) {
    std::lock_guard<std::mutex> lk(ctx->small_mu);
    ctx->small_free[bucket].push_back(ptr);
    return;
  }
  cudaFreeAsync(ptr, ctx->stream);
}

size_t dtype_size(int dtype) {
  switch (dtype) {
    case TQP_BOOL: return 1;
    case TQP_I32: return 4;
    case TQP_I64: return 8;
    case TQP_F64: return 8;
    case TQP_STR8: return 1;
  }
  return 0;
}

size_t Tensor::elem_size() const { return dtype_size(dtype); }

const char* dtype_name(int dtype) {
  switch (dtype) {
    case TQP_BOOL: return "bool";
    case TQP_I32: return "int32";
    case TQP_I64: return "int64";
    case TQP_F64: return "float64";
    case TQP_STR8: return "int32";  // strings are Int32 tensors in the reference
  }
  return "?";
}

const char* logical_type_name(int lt) {
  switch (lt) {
    case TQP_LT_INT64: return "int64";
    case TQP_LT_FLOAT64: return "float64";
    case TQP_LT_DATE: return "date";
    case TQP_LT_UTF8: return "utf8";
    case TQP_LT_BOOL: return "bool";
  }
  return "?";
}

int physical_dtype(int lt) {
  switch (lt) {
    case TQP_LT_INT64: return TQP_I64;
    case TQP_LT_FLOAT64: return TQP_F64;
    case TQP_LT_DATE: return TQP_I64;
    case TQP_LT_UTF8: return TQP_STR8;
    case TQP_LT_BOOL: return TQP_BOOL;
  }
  return -1;
}

void Ctx::jit_epoch_check() {
  const long long e = jit_epoch();
  if (e == jit_epoch_seen_) return;
  jit_epoch_seen_ = e;
  static_smem_.clear();
  occupancy_.clear();
  smem_set.clear();
}

std::shared_ptr<DevBuf> Ctx::alloc_bytes(size_t bytes) {
  auto b = std::make_shared<DevBuf>();
  b->ctx = this;
  b->bytes = bytes;
  if (!bytes) return b;
  if (!pool_only && bytes <= (size_t(256) << (kSmallBuckets - 1))) {
    int i = 0;
    while ((size_t(256) << i) < bytes) ++i;
    b->bucket = i;
    {
      std::lock_guard<std::mutex> lk(small_mu);
      if (!small_free[i].empty()) {
        b->ptr = small_free[i].back();
        small_free[i].pop_back();
        return b;
      }
    }
    TQP_CUDA(cudaMallocFromPoolAsync(&b->ptr, size_t(256) << i, pool, stream));
    return b;
  }
  TQP_CUDA(cudaMallocFromPoolAsync(&b->ptr, bytes, pool, stream));
  return b;
}

std::shared_ptr<long long> Ctx::pinned_slot() {
  std::lock_guard<std::mutex> lk(small_mu);
  if (pinned_free.empty()) {
    long long* chunk = nullptr;
    TQP_CUDA(cudaMallocHost(&chunk, 4096));
    pinned_chunks.push_back(chunk);
    for (int i = 0; i < 128; ++i) pinned_free.push_back(chunk + 4 * i);
  }
  long long* p = pinned_free.back();
  pinned_free.pop_back();
  p[0] = p[1] = p[2] = p[3] = 0;
  return std::shared_ptr<long long>(p, [this](long long* q) {
    std::lock_guard<std::mutex> lk2(small_mu);
    pinned_free.push_back(q);
  });
}

void Ctx::release_pinned() {
  for (long long* ch : pinned_chunks) cudaFreeHost(ch);
  pinned_chunks.clear();
  pinned_free.clear();
}

void Ctx::release_stages() {
  for (auto& s : stages) {
    if (s.ptr) cudaFree(s.ptr);
    if (s.freed) cudaEventDestroy(s.freed);
    s = Stage{};
  }
}

void Ctx::release_small() {
  std::lock_guard<std::mutex> lk(small_mu);
  for (auto& v : small_free) {
    for (void* p : v) cudaFreeAsync(p, stream);
    v.clear();
  }
}

Tensor Ctx::alloc(int dtype, int64_t rows, int64_t cols) {
  Tensor t;
  t.dtype = dtype;
  t.rows = rows;
  t.cols = cols;
  // pad to 16 B so vectorised kernels may read whole 128-bit words
  size_t bytes = static_cast<size_t>(rows * cols) * dtype_size(dtype);
  t.buf = alloc_bytes((bytes + 15) & ~size_t(15));
  t.buf->bytes = bytes;
  return t;
}

void Ctx::sync() { TQP_CUDA(cudaStreamSynchronize(stream)); }

void Ctx::reset_err() {
  TQP_CUDA(cudaMemcpyAsync(d_err, h_err + kPinnedErrInit, 3 * sizeof(long long), cudaMemcpyHostToDevice, stream));
}

int64_t Ctx::read_err(long long* aux, long long* kind) {
  TQP_CUDA(cudaMemcpyAsync(h_err, d_err, 3 * sizeof(long long), cudaMemcpyDeviceToHost, stream));
  sync();
  if (aux) *aux = h_err[1];
  if (kind) *kind = h_err[2];
  return h_err[0] == kNoBad ? -1 : h_err[0];
}

long long* Ctx::check_slot(bool* is_deferred) {
  if (defer_checks && deferred.size() < static_cast<size_t>(kMaxDeferred)) {
    *is_deferred = true;
    return d_defer + 4 * deferred.size();
  }
  *is_deferred = false;
  reset_err();
  return d_err;
}

void Ctx::check_deferred() {
  if (deferred.empty()) return;
  const size_t n = deferred.size();
  std::vector<DeferredCheck> list;
  list.swap(deferred);
  TQP_CUDA(cudaMemcpyAsync(h_err + kPinnedRead, d_defer, 4 * n * sizeof(long long), cudaMemcpyDeviceToHost, stream));
  sync();
  // slots back to "no error" (ordered before any later use on the stream)
  TQP_CUDA(cudaMemcpyAsync(d_defer, h_err + kPinnedDeferInit, 4 * n * sizeof(long long), cudaMemcpyHostToDevice, stream));
  for (size_t i = 0; i < n; ++i) {
    const long long bad = h_err[kPinnedRead + 4 * i];
    if (bad != kNoBad) {
      const int64_t row = bad / list[i].cols;
      kernel_fail(list[i].msg + std::to_string(row), row);
    }
  }
}

int Ctx::grid_for(int64_t n, int block, int per_thread, int waves) const {
  int64_t need = (n + static_cast<int64_t>(block) * per_thread - 1) / (static_cast<int64_t>(block) * per_thread);
  int64_t cap = static_cast<int64_t>(num_sms) * waves;
  if (need < 1) need = 1;
  return static_cast<int>(need < cap ? need : cap);
}

Tensor upload(Ctx& c, int dtype, int64_t rows, int64_t cols, const void* host) {
  if (rows < 0 || cols < 1) kernel_fail("tensor: buffer length does not match shape");
  Tensor t = c.alloc(dtype, rows, cols);
  if (t.bytes()) TQP_CUDA(cudaMemcpyAsync(t.data(), host, t.bytes(), cudaMemcpyHostToDevice, c.stream));
  return t;
}

void download(Ctx& c, const Tensor& t, void* host) {
  if (t.bytes()) TQP_CUDA(cudaMemcpyAsync(host, t.data(), t.bytes(), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
}

namespace {
__global__ void k_i32_to_u8(const int32_t* __restrict__ in, uint8_t* __restrict__ out, int64_t n) {
  for (int64_t i = gtid(); i < n; i += gstride()) out[i] = static_cast<uint8_t>(in[i]);
}
__global__ void k_u8_to_i32(const uint8_t* __restrict__ in, int32_t* __restrict__ out, int64_t n) {
  for (int64_t i = gtid(); i < n; i += gstride()) out[i] = in[i];
}
}  // namespace

namespace k {
Tensor utf8_i32_to_str8(Ctx& c, const Tensor& t) {
  Tensor o = c.alloc(TQP_STR8, t.rows, t.cols);
  int64_t n = t.size();
  if (n) {
    k_i32_to_u8<<<c.grid_for(n, 256), 256, 0, c.stream>>>(t.ptr<int32_t>(), o.ptr<uint8_t>(), n);
    c.count_launch();
  }
  return o;
}
Tensor str8_to_i32(Ctx& c, const Tensor& t) {
  Tensor o = c.alloc(TQP_I32, t.rows, t.cols);
  int64_t n = t.size();
  if (n) {
    k_u8_to_i32<<<c.grid_for(n, 256), 256, 0, c.stream>>>(t.ptr<uint8_t>(), o.ptr<int32_t>(), n);
    c.count_launch();
  }
  return o;
}
}  // namespace k

}  // namespace tqp
