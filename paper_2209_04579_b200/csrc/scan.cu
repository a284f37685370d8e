// Scan-shaped kernels: prefix_sum_exclusive (kernels.cpp:349-362), compact
// (kernels.cpp:364-409), expand_segments (kernels.cpp:486-516), searchsorted
// (kernels.cpp:457-484). The reference runs the scans serially; here they
// are single-pass decoupled-lookback scans over 2048-element tiles.
#include <string>

#include "scan.cuh"

namespace tqp {
namespace {

#ifndef TQP_SCAN_THREADS
#define TQP_SCAN_THREADS 256
#define TQP_SCAN_ITEMS 8
#endif
constexpr int kThreads = TQP_SCAN_THREADS;
constexpr int kItems = TQP_SCAN_ITEMS;  // rows per thread (warp-striped): 2048-row tiles
constexpr int kTile = kThreads * kItems;

struct ScanScratch {
  std::shared_ptr<DevBuf> buf;
  longlong2* desc;
  int* counter;
};

ScanScratch scan_scratch(Ctx& c, int64_t tiles) {
  ScanScratch s;
  size_t bytes = sizeof(longlong2) * (tiles + 1) + 16;
  s.buf = c.alloc_bytes(bytes);
  TQP_CUDA(cudaMemsetAsync(s.buf->ptr, 0, bytes, c.stream));
  s.desc = static_cast<longlong2*>(s.buf->ptr);
  s.counter = reinterpret_cast<int*>(s.desc + tiles + 1);
  return s;
}

// Exclusive int64 scan; reports the first row where the sequential
// accumulation overflows (the reference's check order, kernels.cpp:356-359).
// Warp-striped tiles: warp w of a tile owns rows [w * 32 * kItems, ...) of
// it, item j of lane l is row j * 32 + l, so every load and store of a warp
// is one contiguous 256-byte run (a blocked layout - kItems consecutive rows
// per thread - ran the scans at 0.3 of HBM bandwidth: each warp access
// touched 32 lines). Within a warp the rows are scanned item by item with
// shuffles, carrying the running total; warps combine through shared
// memory, tiles through the decoupled lookback.
__device__ __forceinline__ unsigned long long warp_incl_scan(unsigned long long v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// per-warp totals -> exclusive warp offsets (s_warp[w]) and the tile total
// (s_warp[kThreads / 32]); the tile's exclusive prefix from the lookback in
// *s_prefix. Called by every thread.
__device__ __forceinline__ void tile_offsets(unsigned long long wtotal, unsigned long long* s_warp, long long* s_prefix,
                                             longlong2* desc, int tile) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kW = kThreads / 32;
  if (lane == 0) s_warp[warp] = wtotal;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long w = lane < kW ? s_warp[lane] : 0ULL;
    const unsigned long long wi = warp_incl_scan(w);
    __syncwarp();
    if (lane < kW) s_warp[lane] = wi - w;
    const unsigned long long total = __shfl_sync(0xffffffffu, wi, kW - 1);
    const long long pfx = tile_lookback(desc, tile, static_cast<long long>(total));
    if (lane == 0) {
      s_warp[kW] = total;
      *s_prefix = pfx;
    }
  }
  __syncthreads();
}

// Occupancy sets this kernel's speed: a tile's loads are its only memory
// parallelism, so the warp scans are done twice (totals before the lookback,
// the exclusive prefixes after it) instead of keeping kItems prefixes in
// registers across it: 64 -> 32 registers (a few words spilled to L1), 4 -> 8 resident tiles per SM.
#ifndef TQP_SCAN_MINB
#define TQP_SCAN_MINB 8
#endif
__global__ void __launch_bounds__(kThreads, TQP_SCAN_MINB) k_prefix_sum(const int64_t* __restrict__ x, int64_t* __restrict__ out,
                                                         int64_t n, longlong2* desc, int* counter, long long* err) {
  __shared__ int s_tile;
  __shared__ unsigned long long s_warp[kThreads / 32 + 1];
  __shared__ long long s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1);
  __syncthreads();
  const int tile = s_tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wbase = static_cast<int64_t>(tile) * kTile + static_cast<int64_t>(warp) * 32 * kItems + lane;
  int64_t v[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) v[j] = wbase + j * 32 < n ? x[wbase + j * 32] : 0;
  unsigned long long lsum = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) lsum += static_cast<unsigned long long>(v[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
  tile_offsets(lsum, s_warp, &s_prefix, desc, tile);
  unsigned long long carry = static_cast<unsigned long long>(s_prefix) + s_warp[warp];
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const unsigned long long is = warp_incl_scan(static_cast<unsigned long long>(v[j]));
    const unsigned long long acc = carry + is - static_cast<unsigned long long>(v[j]);
    carry += __shfl_sync(0xffffffffu, is, 31);
    const int64_t i = wbase + j * 32;
    if (i < n) {
      out[i] = static_cast<int64_t>(acc);
      int64_t r;
      if (add_ovf(static_cast<int64_t>(acc), v[j], &r)) note_bad(err, i);
    }
  }
}

// Single-pass order-preserving compaction: a tile (dynamic id, so the
// lookback always waits on tiles already running) ranks its selected rows
// with one ballot + popcount per warp item, takes its output offset from the
// decoupled lookback, and each warp item's selected rows go to consecutive
// output rows (coalesced, warp-striped as the prefix sum). Rows of several
// columns (m > 1) are copied column by column per selected row.
template <typename T>
__global__ void __launch_bounds__(kThreads, 8) k_compact_onepass(const T* __restrict__ vals, const uint8_t* __restrict__ mask,
                                                              int64_t n, int64_t m, T* __restrict__ out, longlong2* desc,
                                                              int* counter) {
  __shared__ int s_tile;
  __shared__ unsigned long long s_warp[kThreads / 32 + 1];
  __shared__ long long s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1);
  __syncthreads();
  const int tile = s_tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t wbase = static_cast<int64_t>(tile) * kTile + static_cast<int64_t>(warp) * 32 * kItems + lane;
  unsigned ball[kItems];
  T v[kItems];
  unsigned carry = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int64_t i = wbase + j * 32;
    const bool sel = i < n && mask[i] != 0;
    if (m == 1) v[j] = i < n ? vals[i] : T{};
    ball[j] = __ballot_sync(0xffffffffu, sel);
    carry += __popc(ball[j]);
  }
  tile_offsets(carry, s_warp, &s_prefix, desc, tile);
  unsigned long long w = static_cast<unsigned long long>(s_prefix) + s_warp[warp];
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    if ((ball[j] >> lane) & 1u) {
      const unsigned long long pos = w + __popc(ball[j] & lt_mask);
      if (m == 1) {
        out[pos] = v[j];
      } else {
        const int64_t i = wbase + j * 32;
        for (int64_t q = 0; q < m; ++q) out[pos * m + q] = vals[i * m + q];
      }
    }
    w += __popc(ball[j]);
  }
}

__global__ void k_check_negative(const int64_t* __restrict__ c, int64_t n, long long* err) {
  for (int64_t i = gtid(); i < n; i += gstride())
    if (c[i] < 0) note_bad(err, i);
}

__global__ void k_expand(const int64_t* __restrict__ starts, const int64_t* __restrict__ offs, int64_t k,
                         int64_t total, int64_t* __restrict__ out) {
  for (int64_t j = gtid(); j < total; j += gstride()) {
    // last segment whose offset <= j (upper_bound - 1)
    int64_t lo = 0, hi = k;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (offs[mid] <= j) lo = mid + 1;
      else hi = mid;
    }
    int64_t s = lo - 1;
    out[j] = starts[s] + (j - offs[s]);
  }
}

template <typename T>
__global__ void k_nan_check(const T* __restrict__ v, int64_t n, long long* err) {
  if constexpr (std::is_same_v<T, double>) {
    for (int64_t i = gtid(); i < n; i += gstride())
      if (isnan(v[i])) note_bad(err, i);
  }
}

template <typename T>
__global__ void k_sorted_check(const T* __restrict__ v, int64_t n, long long* err) {
  for (int64_t i = gtid() + 1; i < n; i += gstride())
    if (v[i] < v[i - 1]) note_bad(err, i);
}

// Binary search with the top of the tree in shared memory: every block
// stages kSearchPivots evenly spaced keys, and a probe first finds its pivot
// interval there, then searches only that interval (n / kSearchPivots keys)
// in global memory. Each warp takes a contiguous run of probes (lane l: rows
// run + 32 t + l), so a lane's consecutive probes are 32 rows apart: when a
// probe is not below the lane's previous one (sorted probe columns, e.g.
// lineitem's l_orderkey), its answer is at or after the previous answer and
// an exponential search from there finds it in a step or two; otherwise (or
// after kGallop doublings) the pivot search runs. Result: the first index
// whose key does not go right (left: s[k] < x, right: s[k] <= x).
constexpr int kSearchPivots = 2048;
constexpr int kGallop = 8;
template <typename T>
__global__ void __launch_bounds__(256) k_searchsorted(const T* __restrict__ s, int64_t n, const T* __restrict__ p,
                                                      int64_t np, bool left, int64_t* __restrict__ out) {
  __shared__ T piv[kSearchPivots];
  const int64_t stride = n > kSearchPivots ? (n + kSearchPivots - 1) / kSearchPivots : 1;
  const int npiv = static_cast<int>((n + stride - 1) / stride);  // pivot j = s[j * stride]
  for (int j = threadIdx.x; j < npiv; j += blockDim.x) piv[j] = s[static_cast<int64_t>(j) * stride];
  __syncthreads();
  auto go_right = [&](T key, T x) { return left ? (key < x) : !(x < key); };
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t run = ((np + nwarps - 1) / nwarps + 31) & ~int64_t(31);
  const int64_t r0 = gw * run, r1 = r0 + run < np ? r0 + run : np;
  bool have = false;
  T px{};
  int64_t pans = 0;
  for (int64_t i = r0 + lane; i < r1; i += 32) {
    const T x = p[i];
    int64_t lo = 0, hi = n;
    bool found = false;
    if (have && !(x < px)) {
      // answer >= pans: gallop pans, pans + 1, pans + 3, pans + 7, ...
      lo = pans;
      int64_t step = 1;
      int d = 0;
      for (; d < kGallop; ++d) {
        const int64_t probe = lo + step - 1;
        if (probe >= n) {
          hi = n;
          found = true;
          break;
        }
        if (!go_right(s[probe], x)) {
          hi = probe;
          found = true;
          break;
        }
        lo = probe + 1;
        step <<= 1;
      }
    }
    if (!found) {
      // pivot interval, then the interval in global memory (within [lo, n))
      int plo = 0, phi = npiv;
      while (plo < phi) {
        const int mid = (plo + phi) >> 1;
        if (go_right(piv[mid], x)) plo = mid + 1;
        else phi = mid;
      }
      const int64_t a = plo == 0 ? 0 : static_cast<int64_t>(plo - 1) * stride + 1;
      hi = plo >= npiv ? n : static_cast<int64_t>(plo) * stride;
      lo = lo > a ? lo : a;
    }
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (go_right(s[mid], x)) lo = mid + 1;
      else hi = mid;
    }
    out[i] = lo;
    have = true;
    px = x;
    pans = lo;
  }
}

void require(bool ok, const std::string& msg) {
  if (!ok) kernel_fail(msg);
}

}  // namespace

namespace k {

// Exclusive scan of an int64 vector; fills `first_overflow` (or -1).
Tensor prefix_sum_raw(Ctx& c, const Tensor& x, int64_t* first_overflow) {
  int64_t n = x.rows;
  Tensor o = c.alloc(TQP_I64, n, 1);
  *first_overflow = -1;
  if (!n) return o;
  int64_t tiles = (n + kTile - 1) / kTile;
  auto s = scan_scratch(c, tiles);
  c.reset_err();
  k_prefix_sum<<<tiles, kThreads, 0, c.stream>>>(x.ptr<int64_t>(), o.ptr<int64_t>(), n, s.desc, s.counter, c.d_err);
  c.count_launch();
  *first_overflow = c.read_err();
  return o;
}

// Exclusive scan without the overflow readback (callers that know the sums fit).
Tensor prefix_sum_unchecked(Ctx& c, const Tensor& x) {
  int64_t n = x.rows;
  Tensor o = c.alloc(TQP_I64, n, 1);
  if (!n) return o;
  int64_t tiles = (n + kTile - 1) / kTile;
  auto s = scan_scratch(c, tiles);
  auto scratch_err = c.alloc_bytes(32);  // the kernel's overflow word, never read
  TQP_CUDA(cudaMemsetAsync(scratch_err->ptr, 0x7f, 8, c.stream));
  k_prefix_sum<<<tiles, kThreads, 0, c.stream>>>(x.ptr<int64_t>(), o.ptr<int64_t>(), n, s.desc, s.counter,
                                                 static_cast<long long*>(scratch_err->ptr));
  c.count_launch();
  return o;
}

Tensor prefix_sum_exclusive(Ctx& c, const Tensor& x) {
  require(x.is_vector(), "prefix_sum_exclusive: expected a vector (m=1)");
  if (x.dtype != TQP_I64) {
    kernel_fail(std::string("prefix_sum_exclusive: expected int64, got ") + dtype_name(x.dtype));
  }
  int64_t bad;
  Tensor o = prefix_sum_raw(c, x, &bad);
  if (bad >= 0) kernel_fail("prefix_sum_exclusive: overflow at row " + std::to_string(bad), bad);
  return o;
}

Tensor compact(Ctx& c, const Tensor& values, const Tensor& mask) {
  if (mask.dtype != TQP_BOOL) kernel_fail(std::string("compact: expected bool, got ") + dtype_name(mask.dtype));
  require(mask.is_vector(), "compact: expected a vector (m=1)");
  if (mask.rows != values.rows) {
    kernel_fail("compact: mask length " + std::to_string(mask.rows) + " does not match rows " +
                std::to_string(values.rows));
  }
  int64_t n = values.rows, m = values.cols;
  if (n == 0) return c.alloc(values.dtype, 0, m);
  // one pass (k_compact_onepass) into an output sized for every row; the
  // count comes back with the last tile's inclusive prefix (the one host
  // round trip: the result's shape), and a sparse result moves to a buffer
  // of its own size so the n-row buffer is not held
  const int64_t tiles = (n + kTile - 1) / kTile;
  ScanScratch sc = scan_scratch(c, tiles);
  Tensor o = c.alloc(values.dtype, n, m);
  TQP_DISPATCH(values.dtype, T,
               k_compact_onepass<T><<<tiles, kThreads, 0, c.stream>>>(values.ptr<T>(), mask.ptr<uint8_t>(), n, m,
                                                                      o.ptr<T>(), sc.desc, sc.counter));
  c.count_launch();
  long long* h = c.h_err + Ctx::kPinnedRead;
  TQP_CUDA(cudaMemcpyAsync(h, sc.desc + tiles - 1, sizeof(longlong2), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  const int64_t total = h[1];
  if (total * 2 < n) {
    Tensor t = c.alloc(values.dtype, total, m);
    if (total) TQP_CUDA(cudaMemcpyAsync(t.data(), o.data(), t.bytes(), cudaMemcpyDeviceToDevice, c.stream));
    return t;
  }
  o.rows = total;
  return o;
}

Tensor expand_segments(Ctx& c, const Tensor& starts, const Tensor& counts) {
  if (starts.dtype != TQP_I64) kernel_fail(std::string("expand_segments: expected int64, got ") + dtype_name(starts.dtype));
  if (counts.dtype != TQP_I64) kernel_fail(std::string("expand_segments: expected int64, got ") + dtype_name(counts.dtype));
  require(starts.is_vector(), "expand_segments: expected a vector (m=1)");
  require(counts.is_vector(), "expand_segments: expected a vector (m=1)");
  if (starts.rows != counts.rows) kernel_fail("expand_segments: starts/counts length mismatch");
  int64_t kk = starts.rows;
  if (kk == 0) return c.alloc(TQP_I64, 0, 1);
  c.reset_err();
  k_check_negative<<<c.grid_for(kk, 256), 256, 0, c.stream>>>(counts.ptr<int64_t>(), kk, c.d_err);
  c.count_launch();
  int64_t neg = c.read_err();
  if (neg >= 0) kernel_fail("expand_segments: negative count at row " + std::to_string(neg), neg);
  int64_t ovf;
  Tensor offs = prefix_sum_raw(c, counts, &ovf);
  if (ovf >= 0) kernel_fail("expand_segments: total length overflow");
  int64_t last_off = read_scalar<int64_t>(c, offs, kk - 1);
  int64_t last_cnt = read_scalar<int64_t>(c, counts, kk - 1);
  int64_t total;
  if (__builtin_add_overflow(last_off, last_cnt, &total)) kernel_fail("expand_segments: total length overflow");
  Tensor o = c.alloc(TQP_I64, total, 1);
  if (total) {
    k_expand<<<c.grid_for(total, 256), 256, 0, c.stream>>>(starts.ptr<int64_t>(), offs.ptr<int64_t>(), kk, total,
                                                           o.ptr<int64_t>());
    c.count_launch();
  }
  return o;
}

Tensor searchsorted(Ctx& c, const Tensor& sorted, const Tensor& probes, int side) {
  {
    int da = sorted.dtype, db = probes.dtype;
    if (da != db) {
      kernel_fail(std::string("searchsorted: dtype mismatch (") + dtype_name(da) + " vs " + dtype_name(db) + ")");
    }
  }
  require(sorted.is_vector(), "searchsorted: expected a vector (m=1)");
  require(probes.is_vector(), "searchsorted: expected a vector (m=1)");
  int64_t n = sorted.rows, np = probes.rows;
  Tensor o = c.alloc(TQP_I64, np, 1);
  TQP_DISPATCH(sorted.dtype, T, {
    if (std::is_same_v<T, double>) {
      c.reset_err();
      if (n) k_nan_check<T><<<c.grid_for(n, 256), 256, 0, c.stream>>>(sorted.ptr<T>(), n, c.d_err);
      if (np) k_nan_check<T><<<c.grid_for(np, 256), 256, 0, c.stream>>>(probes.ptr<T>(), np, c.d_err);
      c.count_launch(2);
      if (c.read_err() >= 0) kernel_fail("searchsorted: NaN in keys");
    }
    if (n > 1) {
      c.reset_err();
      k_sorted_check<T><<<c.grid_for(n, 256), 256, 0, c.stream>>>(sorted.ptr<T>(), n, c.d_err);
      c.count_launch();
      int64_t bad = c.read_err();
      if (bad >= 0) kernel_fail("searchsorted: input not non-decreasing at row " + std::to_string(bad), bad);
    }
    if (np) {
      k_searchsorted<T><<<c.grid_for(np, 256), 256, 0, c.stream>>>(sorted.ptr<T>(), n, probes.ptr<T>(), np,
                                                                   side == TQP_LEFT, o.ptr<int64_t>());
      c.count_launch();
    }
  });
  return o;
}

}  // namespace k
}  // namespace tqp
