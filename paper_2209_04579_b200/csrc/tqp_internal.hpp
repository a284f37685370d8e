// Internal C++ interfaces of libtqp_b200.so (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <mutex>
#include <vector>
#include <cstdlib>
#include <cstdio>
#include <chrono>

#include "tqp_b200.h"

namespace tqp {

// Error carrying the reference's exception class (tqp_error_code) and
// message; the C boundary converts it into a tqp_status.
struct Error : std::runtime_error {
  int code;
  int64_t bad_row;
  Error(int c, const std::string& m, int64_t row = -1) : std::runtime_error(m), code(c), bad_row(row) {}
};
[[noreturn]] inline void kernel_fail(const std::string& m, int64_t row = -1) { throw Error(TQP_ERR_KERNEL, m, row); }
[[noreturn]] inline void exec_fail(const std::string& m) { throw Error(TQP_ERR_EXEC, m); }
[[noreturn]] inline void plan_fail(const std::string& m) { throw Error(TQP_ERR_PLAN, m); }

void cuda_check(cudaError_t e, const char* what);
#define TQP_CUDA(x) ::tqp::cuda_check((x), #x)

struct Ctx;

// Stream-ordered device allocation (freed on the owning context's stream).
struct DevBuf {
  Ctx* ctx = nullptr;
  void* ptr = nullptr;
  size_t bytes = 0;
  int bucket = -1;  // >= 0: a small block of the context's host-side cache
  // derived state of an immutable tensor living in this buffer, computed once
  // (reduce.cu: the validated segment plan of a segment-id vector)
  std::shared_ptr<void> seg_plan;
  // written on another stream (a column decoded on the context's decode
  // stream): `ctx->stream` waits for this event before the first use
  // (Ctx::wait_ready), then it is dropped
  cudaEvent_t ready = nullptr;
  ~DevBuf();
};

// Immutable device tensor: the device analogue of tensql::Tensor
// (tensor.hpp:49-122), shared by reference.
struct Tensor {
  int dtype = TQP_I64;
  int64_t rows = 0, cols = 1;
  std::shared_ptr<DevBuf> buf;

  int64_t size() const { return rows * cols; }
  bool is_vector() const { return cols == 1; }
  bool is_scalar() const { return rows == 1 && cols == 1; }
  bool same_shape(const Tensor& o) const { return rows == o.rows && cols == o.cols; }
  size_t elem_size() const;
  size_t bytes() const { return static_cast<size_t>(size()) * elem_size(); }
  template <typename T>
  T* ptr() const { return buf ? static_cast<T*>(buf->ptr) : nullptr; }
  void* data() const { return buf ? buf->ptr : nullptr; }
};

const char* dtype_name(int dtype);  // reference names (tensor.cpp:5-13); STR8 -> "int32"
size_t dtype_size(int dtype);
const char* logical_type_name(int lt);
int physical_dtype(int lt);  // device physical dtype of a logical type

// TQP_HOST_PROF=1: wall-clock marks of a host-side section (a fused unit,
// an execution), one stderr line per section (where host time goes)
struct HostProf {
  bool on;
  const char* tag;
  std::vector<std::pair<const char*, std::chrono::steady_clock::time_point>> m;
  explicit HostProf(const char* t = "unit") : on(std::getenv("TQP_HOST_PROF") != nullptr), tag(t) { mark("start"); }
  void mark(const char* what) {
    if (on) m.emplace_back(what, std::chrono::steady_clock::now());
  }
  ~HostProf() {
    if (!on || m.size() < 2) return;
    std::string o = std::string("[tqp host ") + tag + "]";
    for (size_t i = 1; i < m.size(); ++i)
      o += std::string(" ") + m[i].first + "=" +
           std::to_string(std::chrono::duration_cast<std::chrono::microseconds>(m[i].second - m[i - 1].second).count());
    std::fprintf(stderr, "%s us\n", o.c_str());
  }
};

struct Ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaMemPool_t pool = nullptr;
  // device scratch for kernel error reporting: [0] first bad index
  // (atomicMin, INT64_MAX = none), [1] aux value, [2] error kind
  long long* d_err = nullptr;
  long long* h_err = nullptr;  // pinned: [0, 3) error mirror, then the regions below
  // pinned host words for small copies (pageable copies stage through the
  // driver): constant upload sources and a readback area
  static constexpr int kPinnedWords = 512;
  static constexpr int kPinnedErrInit = 8;     // {INT64_MAX, 0, 0}
  static constexpr int kPinnedMinMax = 64;     // kPinnedMinMaxPairs x {INT64_MAX, INT64_MIN}
  static constexpr int kPinnedMinMaxPairs = 64;
  static constexpr int kPinnedDeferInit = 192;  // kMaxDeferred x {INT64_MAX, 0, 0, 0}
  static constexpr int kPinnedRead = 256;      // 256 words of readback
  static constexpr int kPinnedUnitErr = 480;   // a deferred fused unit's error words (4)
  // Deferred checks (executor steps only): an instruction whose one host
  // interaction is its error check (arith's division by zero / overflow)
  // gets its own device error slot instead of a round trip; the executor
  // reads every slot of a step in one readback (check_deferred) before the
  // step's next synchronous error or its end, and the first failing
  // instruction in program order is reported, as if checked in place.
  static constexpr int kMaxDeferred = 16;
  long long* d_defer = nullptr;  // kMaxDeferred x 4 words
  bool defer_checks = false;
  struct DeferredCheck {
    std::string msg;  // message up to the row number
    int64_t cols;     // reported row = flat index / cols
  };
  std::vector<DeferredCheck> deferred;
  // error slot of the next check: a fresh deferred slot while deferring
  // (and one is free), else d_err after reset_err()
  long long* check_slot(bool* is_deferred);
  void check_deferred();
  std::atomic<int64_t> launches{0};
  // Small blocks (error words, scalars, partials, output columns of a few
  // rows) are recycled through a host-side free list per power-of-two size
  // instead of a cudaMallocAsync/cudaFreeAsync pair each: a query makes a
  // dozen of them and each driver call is host time between its kernels.
  // Reuse follows the stream order exactly as cudaFreeAsync on `stream`
  // does (a block freed after its last enqueued use is only handed to work
  // enqueued later on the same stream).
  static constexpr int kSmallBuckets = 9;  // 256 B << i, up to 64 KB
  // set while work is enqueued on another stream (codec.cu's decode stream):
  // the free list is ordered by `stream` only, so allocations bypass it
  bool pool_only = false;
  std::mutex small_mu;
  std::vector<void*> small_free[kSmallBuckets];
  void release_small();
  // Larger blocks go straight back to the stream-ordered pool, which reuses
  // them for any size (an exact-size host cache of them was tried: it kept
  // memory from the pool, which then grew for every new size - the
  // per-instruction path's temporaries, 11.8 -> 59 ms for Q1).

  Tensor alloc(int dtype, int64_t rows, int64_t cols);
  std::shared_ptr<DevBuf> alloc_bytes(size_t bytes);
  void sync();
  void reset_err();
  // copies d_err to host (syncs); returns first bad index or -1
  int64_t read_err(long long* aux = nullptr, long long* kind = nullptr);
  int grid_for(int64_t n, int block, int per_thread = 1, int waves = 8) const;
  void count_launch(int n = 1) { launches += n; }

  // optional per-kernel device timing (CUDA events on `stream`), drained by
  // the executor's timings
  int time_kernels = 0;  // 0 off, 1 every kernel, 2 fused fact-scan kernels only
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> kernel_events;
  // CSV file loader: pinned ring of upload buffers (csv.cu), kept for reuse
  unsigned char* csv_ring = nullptr;
  cudaEvent_t csv_ring_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // timing events are recycled (creating one per launch costs host time
  // between dependent launches)
  std::vector<cudaEvent_t> event_pool;
  // a second stream for host->device copies that may overlap the work of
  // `stream` (compressed column uploads); created on first use
  cudaStream_t copy_stream = nullptr;
  // Staging slots for encoded column uploads (codec.cu decode_column): a
  // column's host->device copy waits only for the decode that last read its
  // slot, not for everything queued on `stream`, so consecutive columns'
  // copies run back to back on the copy engine while earlier columns decode.
  struct Stage {
    void* ptr = nullptr;
    size_t cap = 0;
    cudaEvent_t freed = nullptr;  // recorded on `stream` after the slot's decode
  };
  static constexpr int kStages = 3;
  Stage stages[kStages];
  int stage_next = 0;
  void release_stages();
  // 4-word pinned host slots for asynchronous executions' deferred checks
  // (Executor::execute_async), carved from 4 KB pinned chunks
  std::vector<long long*> pinned_free, pinned_chunks;
  std::shared_ptr<long long> pinned_slot();
  void release_pinned();
  // decodes of encoded uploads run here, so the context stream's queued
  // work (a query over the previous tables) does not hold them up; the
  // decoded tensor carries a ready event (DevBuf::ready)
  cudaStream_t decode_stream = nullptr;
  cudaStream_t decodes() {
    if (!decode_stream) TQP_CUDA(cudaStreamCreateWithFlags(&decode_stream, cudaStreamNonBlocking));
    return decode_stream;
  }
  // orders `stream` after the producer of b (if one is still pending)
  void wait_ready(DevBuf& b) {
    if (!b.ready) return;
    TQP_CUDA(cudaStreamWaitEvent(stream, b.ready, 0));
    cudaEventDestroy(b.ready);  // released once the wait has consumed it
    b.ready = nullptr;
  }
  cudaStream_t copies() {
    if (!copy_stream) TQP_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    return copy_stream;
  }
  cudaEvent_t take_event() {
    cudaEvent_t e;
    if (!event_pool.empty()) {
      e = event_pool.back();
      event_pool.pop_back();
    } else {
      cudaEventCreate(&e);
    }
    return e;
  }
  void give_event(cudaEvent_t e) {
    if (e) event_pool.push_back(e);
  }
  cudaEvent_t kernel_begin(bool fact_scan = false) {
    if (!time_kernels || (time_kernels == 2 && !fact_scan)) return nullptr;
    cudaEvent_t e = take_event();
    cudaEventRecord(e, stream);
    return e;
  }
  void kernel_end(const std::string& name, cudaEvent_t start) {
    if (!start) return;
    cudaEvent_t e = take_event();
    cudaEventRecord(e, stream);
    kernel_events.push_back({name, {start, e}});
  }
  // per-device opt-in shared memory and per-kernel static shared memory,
  // queried once (driver calls between a unit's kernels are host time)
  int smem_optin_ = -1;
  std::map<const void*, size_t> static_smem_;
  int smem_optin() {
    if (smem_optin_ < 0) TQP_CUDA(cudaDeviceGetAttribute(&smem_optin_, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    return smem_optin_;
  }
  // the kernel-pointer caches below drop their entries when a JIT library
  // was unloaded (jit_epoch): a new kernel may reuse an old handle
  long long jit_epoch_seen_ = 0;
  void jit_epoch_check();
  size_t static_smem(const void* kernel) {
    jit_epoch_check();
    auto it = static_smem_.find(kernel);
    if (it != static_smem_.end()) return it->second;
    cudaFuncAttributes fa{};
    TQP_CUDA(cudaFuncGetAttributes(&fa, kernel));
    return static_smem_[kernel] = fa.sharedSizeBytes;
  }
  std::map<std::pair<const void*, int>, int> occupancy_;
  int blocks_per_sm(const void* kernel, int threads) {  // no dynamic shared memory
    jit_epoch_check();
    auto key = std::make_pair(kernel, threads);
    auto it = occupancy_.find(key);
    if (it != occupancy_.end()) return it->second;
    int n = 1;
    TQP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, 0));
    return occupancy_[key] = n;
  }
  // cudaFuncAttributeMaxDynamicSharedMemorySize, set once per (kernel, size)
  std::map<const void*, int> smem_set;
  cudaError_t ensure_smem(const void* kernel, int bytes) {
    jit_epoch_check();
    auto it = smem_set.find(kernel);
    if (it != smem_set.end() && it->second >= bytes) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) smem_set[kernel] = bytes;
    return e;
  }
};

Tensor upload(Ctx& c, int dtype, int64_t rows, int64_t cols, const void* host);
// compressed columnar host format (codec.cu)
int64_t codec_bound(int dtype, int64_t rows, int64_t cols);
int64_t codec_encode(int dtype, int64_t rows, int64_t cols, const void* host, void* out, int64_t cap, tqp_codec* c);
Tensor decode_column(Ctx& c, int dtype, int64_t rows, int64_t cols, const tqp_codec& k, const void* payload,
                     int64_t bytes);
void download(Ctx& c, const Tensor& t, void* host);
// Tensor::data<int64_t>() / item<int64_t>() of the reference (tensor.hpp:
// 84-100, tensor.cpp:35-39): a typed host access checks the dtype first
inline void check_i64_access(const Tensor& t) {
  if (t.dtype != TQP_I64) kernel_fail(std::string("tensor: dtype is ") + dtype_name(t.dtype) + ", accessed as int64");
}
template <typename T>
T read_scalar(Ctx& c, const Tensor& t, int64_t index = 0) {
  T v{};
  TQP_CUDA(cudaMemcpyAsync(&v, t.ptr<T>() + index, sizeof(T), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  return v;
}

// ---- kernel set (kernels.cu / scan.cu / sort.cu / reduce.cu) ---------------
namespace k {
Tensor compare(Ctx&, const Tensor& a, const Tensor& b, int op);
Tensor arith(Ctx&, const Tensor& a, const Tensor& b, int op);
Tensor logical(Ctx&, const Tensor& a, const Tensor& b, int op);
Tensor logical_not(Ctx&, const Tensor& v);
Tensor select_where(Ctx&, const Tensor& cond, const Tensor& a, const Tensor& b);
Tensor prefix_sum_exclusive(Ctx&, const Tensor& x);
Tensor compact(Ctx&, const Tensor& values, const Tensor& mask);
Tensor argsort_stable(Ctx&, const Tensor& keys);
Tensor gather(Ctx&, const Tensor& values, const Tensor& idx);
Tensor searchsorted(Ctx&, const Tensor& sorted, const Tensor& probes, int side);
Tensor expand_segments(Ctx&, const Tensor& starts, const Tensor& counts);
Tensor segment_starts(Ctx&, const Tensor& sorted_keys);
Tensor segmented_reduce(Ctx&, const Tensor& values, const Tensor& ids, int64_t num_segments, int op);
Tensor matmul(Ctx&, const Tensor& a, const Tensor& b);
Tensor substring_match(Ctx&, const Tensor& chars, const std::string& pattern, int anchor);
// plumbing
Tensor iota(Ctx&, int64_t n);
Tensor cast(Ctx&, const Tensor& t, int to);
Tensor exp_f64(Ctx&, const Tensor& t);
Tensor last_or_zero(Ctx&, const Tensor& t);
Tensor pack_cols(Ctx&, const std::vector<Tensor>& cols);
Tensor broadcast_rows(Ctx&, const Tensor& value, int64_t n);
Tensor pad_width_like(Ctx&, const Tensor& t, const Tensor& like);
Tensor sort_perm_rows(Ctx&, const Tensor& key, const Tensor& perm, bool asc);
Tensor string_compare(Ctx&, const Tensor& a, const Tensor& b, int op);
// helpers
Tensor utf8_i32_to_str8(Ctx&, const Tensor& t);
Tensor str8_to_i32(Ctx&, const Tensor& t);
// stable radix argsort of `keys` (vector) applied to payload `perm`
// (perm = nullptr means identity); descending via inverted digits
Tensor radix_sort_payload(Ctx&, const Tensor& keys, const Tensor* perm, bool descending);
// exclusive int64 scan; *first_overflow = first overflowing row or -1
Tensor prefix_sum_raw(Ctx&, const Tensor& x, int64_t* first_overflow);
Tensor prefix_sum_unchecked(Ctx&, const Tensor& x);
}  // namespace k

}  // namespace tqp

// C handles
struct tqp_tensor {
  tqp::Tensor t;
  std::atomic<int> refs{1};
};
struct tqp_ctx {
  tqp::Ctx c;
};
