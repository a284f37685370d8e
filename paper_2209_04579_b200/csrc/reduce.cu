// segmented_reduce (kernels.cpp:552-672) on device.
//
// Segment runs come from binary searches into the validated, non-decreasing
// ids (segment_runs' contract, kernels.cpp:552-580). Each segment is reduced
// in index order by contiguous per-lane chunks combined left to right, so:
//  - SUM over Int64/Int32 carries an exact 128-bit (sum, min prefix, max
//    prefix) monoid: an overflow is reported exactly when the reference's
//    sequential accumulation would overflow (kernels.cpp:660-664), for the
//    first such segment;
//  - MIN/MAX keep the earliest of equal values (the reference's `v < acc`
//    keeps the first: visible for -0.0 vs +0.0) and propagate NaN;
//  - Float64 SUM is a fixed-order tree (run-to-run deterministic; within
//    1e-9 relative of the reference's sequential / 4096-chunk orders).
// Segments longer than kLong rows are split over CTAs (64K-row chunks) whose
// partials are combined in chunk order.
#include <algorithm>
#include <string>
#include <vector>

#include <type_traits>

#include "device.cuh"

namespace tqp {
namespace {

constexpr int kLong = 4096;
constexpr int64_t kChunk = 65536;

template <typename T>
struct Part;

// ---- partial monoids ---------------------------------------------------------
struct SumF {
  double s = 0.0;
};
struct SumI {
  __int128 s = 0, mn = 0, mx = 0;
  bool empty = true;
  bool bounded = false;  // mn / mx are bounds of the prefixes, not their values (exact s)
};
template <typename T>
struct MinMax {
  T v{};
  int64_t idx = -1;  // -1: empty
  bool nan = false;
};

__device__ __forceinline__ SumF combine(SumF a, SumF b) { return {__dadd_rn(a.s, b.s)}; }
__device__ __forceinline__ SumI combine(const SumI& a, const SumI& b) {
  if (a.empty) return b;
  if (b.empty) return a;
  SumI r;
  r.empty = false;
  r.s = a.s + b.s;
  r.bounded = a.bounded || b.bounded;
  __int128 bmn = a.s + b.mn, bmx = a.s + b.mx;
  r.mn = a.mn < bmn ? a.mn : bmn;
  r.mx = a.mx > bmx ? a.mx : bmx;
  return r;
}
template <typename T>
__device__ __forceinline__ MinMax<T> combine_mm(const MinMax<T>& a, const MinMax<T>& b, bool is_min) {
  if (a.idx < 0) return b;
  if (b.idx < 0) return a;
  MinMax<T> r;
  r.nan = a.nan || b.nan;
  // a precedes b in index order: b wins only if strictly better
  bool take_b = is_min ? (b.v < a.v) : (b.v > a.v);
  r.v = take_b ? b.v : a.v;
  r.idx = take_b ? b.idx : a.idx;
  return r;
}

template <typename T>
__device__ __forceinline__ SumI sumi_one(T v) {
  SumI r;
  r.empty = false;
  r.s = r.mn = r.mx = static_cast<__int128>(v);
  return r;
}

// shuffle helpers for the partial structs
__device__ __forceinline__ SumF shfl(SumF p, int src) { return {__shfl_sync(0xffffffffu, p.s, src)}; }
__device__ __forceinline__ __int128 shfl128(__int128 v, int src) {
  unsigned long long lo = static_cast<unsigned long long>(v), hi = static_cast<unsigned long long>(v >> 64);
  lo = __shfl_sync(0xffffffffu, lo, src);
  hi = __shfl_sync(0xffffffffu, hi, src);
  return (static_cast<__int128>(static_cast<long long>(hi)) << 64) | lo;
}
__device__ __forceinline__ SumI shfl(const SumI& p, int src) {
  SumI r;
  r.s = shfl128(p.s, src);
  r.mn = shfl128(p.mn, src);
  r.mx = shfl128(p.mx, src);
  r.empty = __shfl_sync(0xffffffffu, static_cast<int>(p.empty), src);
  r.bounded = __shfl_sync(0xffffffffu, static_cast<int>(p.bounded), src);
  return r;
}
template <typename T>
__device__ __forceinline__ MinMax<T> shfl(const MinMax<T>& p, int src) {
  MinMax<T> r;
  if constexpr (sizeof(T) == 1) {
    r.v = static_cast<T>(__shfl_sync(0xffffffffu, static_cast<int>(p.v), src));
  } else {
    r.v = __shfl_sync(0xffffffffu, p.v, src);
  }
  r.idx = __shfl_sync(0xffffffffu, p.idx, src);
  r.nan = __shfl_sync(0xffffffffu, static_cast<int>(p.nan), src);
  return r;
}

// Ordered warp combine: lane l holds the partial of the l-th contiguous chunk;
// result (in lane 0) = p0 . p1 . ... . p31 in order.
template <typename P, typename F>
__device__ __forceinline__ P warp_ordered(P p, F comb) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    P q = shfl(p, (lane + o) & 31);
    if ((lane & (2 * o - 1)) == 0) p = comb(p, q);
  }
  return p;
}

// int64 sum monoid of v[a, b) in row order: an int64 running sum with its
// prefix min / max, four rows per step with every load issued first; a step
// whose adds overflow int64 is redone, and the rest of the run continued, in
// the exact 128-bit monoid. (Per row the 128-bit combine cost several times
// the row's load: the per-instruction int64 sums ran at 0.23 of HBM.)
__device__ __forceinline__ SumI sumi_run(const int64_t* __restrict__ v, int64_t a, int64_t b) {
  SumI p;
  if (a >= b) return p;
  int64_t r = 0, mn = 0, mx = 0;
  bool first = true;
  int64_t i = a;
  for (; i + 4 <= b; i += 4) {
    const int64_t x0 = v[i], x1 = v[i + 1], x2 = v[i + 2], x3 = v[i + 3];
    int64_t t0, t1, t2, t3;
    const bool o = add_ovf(r, x0, &t0) | add_ovf(t0, x1, &t1) | add_ovf(t1, x2, &t2) | add_ovf(t2, x3, &t3);
    if (o) break;
    const int64_t lo4 = min(min(t0, t1), min(t2, t3)), hi4 = max(max(t0, t1), max(t2, t3));
    mn = first ? lo4 : min(mn, lo4);
    mx = first ? hi4 : max(mx, hi4);
    first = false;
    r = t3;
  }
  for (; i < b; ++i) {
    int64_t t;
    if (add_ovf(r, v[i], &t)) break;
    mn = first ? t : min(mn, t);
    mx = first ? t : max(mx, t);
    first = false;
    r = t;
  }
  if (!first) {
    p.empty = false;
    p.s = r;
    p.mn = mn;
    p.mx = mx;
  }
  for (; i < b; ++i) p = combine(p, sumi_one(v[i]));  // past an int64 overflow: exact
  return p;
}

// ---- per-op accumulation over [lo, hi) by one warp (contiguous lane chunks)
template <typename T, int OP>
struct Acc;

template <>
struct Acc<double, TQP_SUM> {
  using P = SumF;
  __device__ static P one(double v, int64_t) { return {v}; }
  __device__ static P comb(P a, P b) { return combine(a, b); }
};
template <typename T>
struct AccSumI {
  using P = SumI;
  __device__ static P one(T v, int64_t) { return sumi_one(v); }
  __device__ static P comb(const P& a, const P& b) { return combine(a, b); }
};
template <>
struct Acc<int64_t, TQP_SUM> : AccSumI<int64_t> {};
template <>
struct Acc<int32_t, TQP_SUM> : AccSumI<int32_t> {};
template <typename T, bool IS_MIN>
struct AccMM {
  using P = MinMax<T>;
  __device__ static P one(T v, int64_t i) {
    P r;
    r.v = v;
    r.idx = i;
    if constexpr (std::is_same_v<T, double>) r.nan = isnan(v);
    return r;
  }
  __device__ static P comb(const P& a, const P& b) { return combine_mm(a, b, IS_MIN); }
};
template <typename T>
struct Acc<T, TQP_MIN> : AccMM<T, true> {};
template <typename T>
struct Acc<T, TQP_MAX> : AccMM<T, false> {};

template <typename T, int OP>
__device__ typename Acc<T, OP>::P warp_reduce_range(const T* __restrict__ v, int64_t lo, int64_t hi) {
  using A = Acc<T, OP>;
  using P = typename A::P;
  const int lane = threadIdx.x & 31;
  int64_t len = hi - lo;
  int64_t per = (len + 31) / 32;
  int64_t a = lo + lane * per, b = a + per < hi ? a + per : hi;
  P p{};
  if constexpr (std::is_same_v<T, int64_t> && OP == TQP_SUM) {
    p = sumi_run(v, a, b);
  } else {
    for (int64_t i = a; i < b; ++i) p = A::comb(p, A::one(v[i], i));
  }
  return warp_ordered(p, [](const P& x, const P& y) { return A::comb(x, y); });
}

template <typename T, int OP>
__device__ void write_result(T* out, int64_t s, const typename Acc<T, OP>::P& p, long long* err);

template <>
__device__ void write_result<double, TQP_SUM>(double* out, int64_t s, const SumF& p, long long*) {
  out[s] = p.s;
}
template <typename T>
__device__ void write_sumi(T* out, int64_t s, const SumI& p, long long* err) {
  const __int128 lo = static_cast<__int128>(std::numeric_limits<T>::min());
  const __int128 hi = static_cast<__int128>(std::numeric_limits<T>::max());
  if (!p.empty && (p.mn < lo || p.mx > hi)) note_bad(err, s);
  out[s] = static_cast<T>(p.s);
}
template <>
__device__ void write_result<int64_t, TQP_SUM>(int64_t* out, int64_t s, const SumI& p, long long* err) {
  write_sumi(out, s, p, err);
}
template <>
__device__ void write_result<int32_t, TQP_SUM>(int32_t* out, int64_t s, const SumI& p, long long* err) {
  write_sumi(out, s, p, err);
}
template <typename T>
__device__ void write_mm(T* out, int64_t s, const MinMax<T>& p) {
  if constexpr (std::is_same_v<T, double>) {
    out[s] = p.nan ? __longlong_as_double(0x7ff8000000000000LL) : p.v;
  } else {
    out[s] = p.v;
  }
}

// ---- kernels -------------------------------------------------------------------
__global__ void k_check_ids(const int64_t* __restrict__ ids, int64_t n, int64_t num, long long* err) {
  for (int64_t i = gtid(); i < n; i += gstride()) {
    int64_t s = ids[i], prev = i ? ids[i - 1] : -1;
    if (s < prev) note_bad(err, 2 * i);           // decrease (checked first)
    else if (s < 0 || s >= num) note_bad(err, 2 * i + 1);  // out of range
  }
}

__global__ void k_runs(const int64_t* __restrict__ ids, int64_t n, int64_t num, int64_t* __restrict__ lo,
                       int64_t* __restrict__ hi) {
  for (int64_t s = gtid(); s < num; s += gstride()) {
    int64_t a = 0, b = n;
    while (a < b) {
      int64_t m = (a + b) >> 1;
      if (ids[m] < s) a = m + 1;
      else b = m;
    }
    int64_t l = a;
    b = n;
    while (a < b) {
      int64_t m = (a + b) >> 1;
      if (ids[m] <= s) a = m + 1;
      else b = m;
    }
    lo[s] = l;
    hi[s] = a;
  }
}

__global__ void k_count(const int64_t* __restrict__ lo, const int64_t* __restrict__ hi, int64_t num,
                        int64_t* __restrict__ out) {
  for (int64_t s = gtid(); s < num; s += gstride()) out[s] = hi[s] - lo[s];
}

__global__ void k_first_empty(const int64_t* __restrict__ lo, const int64_t* __restrict__ hi, int64_t num,
                              long long* err) {
  for (int64_t s = gtid(); s < num; s += gstride())
    if (lo[s] == hi[s]) note_bad(err, s);
}

template <typename T, int OP>
__global__ void k_short(const T* __restrict__ v, const int64_t* __restrict__ lo, const int64_t* __restrict__ hi,
                        int64_t num, T* __restrict__ out, long long* err, int64_t* long_list,
                        unsigned long long* long_count) {
  const int64_t warp = gtid() >> 5, nw = gstride() >> 5;
  for (int64_t s = warp; s < num; s += nw) {
    int64_t a = lo[s], b = hi[s];
    if (b - a > kLong) {
      if ((threadIdx.x & 31) == 0) long_list[atomicAdd(long_count, 1ULL)] = s;
      continue;
    }
    auto p = warp_reduce_range<T, OP>(v, a, b);
    if ((threadIdx.x & 31) == 0) {
      if constexpr (OP == TQP_SUM) {
        write_result<T, OP>(out, s, p, err);
      } else {
        write_mm(out, s, p);
      }
    }
  }
}

// one CTA per (segment, chunk) work item; partials stored per item
template <typename T, int OP>
__global__ void k_long_chunks(const T* __restrict__ v, const int64_t* __restrict__ item_lo,
                              const int64_t* __restrict__ item_hi, typename Acc<T, OP>::P* __restrict__ parts) {
  using A = Acc<T, OP>;
  using P = typename A::P;
  __shared__ char smem_raw[32 * sizeof(P)];
  P* sp = reinterpret_cast<P*>(smem_raw);
  int64_t a = item_lo[blockIdx.x], b = item_hi[blockIdx.x];
  int nwarps = blockDim.x >> 5, warp = threadIdx.x >> 5;
  if constexpr (std::is_same_v<T, double> && OP == TQP_SUM) {
    // fp64 sums need no sequential order (the reference's own par backend
    // sums 4096-row chunks, backend.cpp:139-160): coalesced two-row loads,
    // per-thread sums, a fixed xor tree per warp and the warps in order -
    // deterministic run to run, within the fp64 tolerance of `ref`
    double sacc = 0.0;
    const int64_t a2 = (a + 1) & ~int64_t(1);
    if (threadIdx.x == 0 && a2 > a) sacc = v[a];
    const double2* v2 = reinterpret_cast<const double2*>(v + a2);
    const int64_t np = (b - a2) / 2;
    for (int64_t i = threadIdx.x; i < np; i += blockDim.x) {
      const double2 x = __ldg(v2 + i);
      sacc = __dadd_rn(sacc, __dadd_rn(x.x, x.y));
    }
    if (threadIdx.x == 0 && a2 + 2 * np < b) sacc = __dadd_rn(sacc, v[b - 1]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sacc = __dadd_rn(sacc, __shfl_xor_sync(0xffffffffu, sacc, o));
    if ((threadIdx.x & 31) == 0) sp[warp] = P{sacc};
    __syncthreads();
    if (threadIdx.x == 0) {
      P acc = sp[0];
      for (int w = 1; w < nwarps; ++w) acc = A::comb(acc, sp[w]);
      parts[blockIdx.x] = acc;
    }
    return;
  }
  if constexpr (std::is_same_v<T, int64_t> && OP == TQP_SUM) {
    // int64 sums: while max|v| x rows < 2^62 no prefix of the chunk can leave
    // int64, so a wrapping sum in any order is the exact chunk sum and
    // +-max|v| x rows bound every prefix (the partial is marked bounded:
    // k_long_finish decides overflow from the bounds or recomputes the
    // segment exactly). Coalesced two-row loads; else the ordered monoid.
    __shared__ unsigned long long s_sum[32], s_amax[32];
    unsigned long long sum = 0, amax = 0;
    const int64_t a2 = (a + 1) & ~int64_t(1);
    auto take = [&](int64_t x) {
      sum += static_cast<unsigned long long>(x);
      const unsigned long long ax = x < 0 ? 0ULL - static_cast<unsigned long long>(x) : static_cast<unsigned long long>(x);
      amax = ax > amax ? ax : amax;
    };
    if (threadIdx.x == 0 && a2 > a && a < b) take(v[a]);
    const longlong2* v2 = reinterpret_cast<const longlong2*>(v + a2);
    const int64_t np = b > a2 ? (b - a2) / 2 : 0;
    for (int64_t i = threadIdx.x; i < np; i += blockDim.x) {
      const longlong2 x = __ldg(v2 + i);
      take(x.x);
      take(x.y);
    }
    if (threadIdx.x == 0 && a2 + 2 * np < b && b - 1 >= a2) take(v[b - 1]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const unsigned long long y = __shfl_xor_sync(0xffffffffu, amax, o);
      amax = y > amax ? y : amax;
    }
    if ((threadIdx.x & 31) == 0) {
      s_sum[warp] = sum;
      s_amax[warp] = amax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < nwarps; ++w) {
        sum += s_sum[w];
        amax = s_amax[w] > amax ? s_amax[w] : amax;
      }
      s_sum[0] = static_cast<double>(amax) * static_cast<double>(b - a) < 4.0e18 ? 1ULL : 0ULL;  // < 2^62
      if (s_sum[0]) {
        P r;
        if (b > a) {
          r.empty = false;
          r.bounded = true;
          r.s = static_cast<__int128>(static_cast<long long>(sum));
          r.mx = static_cast<__int128>(amax) * static_cast<__int128>(b - a);
          r.mn = -r.mx;
        }
        parts[blockIdx.x] = r;
      }
    }
    __syncthreads();
    if (s_sum[0]) return;
  }
  int64_t len = b - a, per = (len + nwarps - 1) / nwarps;
  int64_t wa = a + warp * per, wb = wa + per < b ? wa + per : b;
  if (wa > wb) wa = wb;
  P p = warp_reduce_range<T, OP>(v, wa, wb);
  if ((threadIdx.x & 31) == 0) sp[warp] = p;
  __syncthreads();
  if (threadIdx.x == 0) {
    P acc = sp[0];
    for (int w = 1; w < nwarps; ++w) acc = A::comb(acc, sp[w]);
    parts[blockIdx.x] = acc;
  }
}

// One warp per long segment: lane l folds a contiguous run of the segment's
// chunk partials in order, then the lanes combine in lane order (the partial
// monoids are associative; the int64 sum's prefix bounds need the order)
template <typename T, int OP>
__global__ void k_long_finish(const typename Acc<T, OP>::P* __restrict__ parts, const int64_t* __restrict__ seg,
                              const int64_t* __restrict__ first_item, const int64_t* __restrict__ nitems, int64_t nlong,
                              T* __restrict__ out, long long* err, const T* __restrict__ v = nullptr,
                              const int64_t* __restrict__ seg_lo = nullptr, const int64_t* __restrict__ seg_hi = nullptr) {
  using A = Acc<T, OP>;
  using P = typename A::P;
  const int lane = threadIdx.x & 31;
  for (int64_t q = gtid() >> 5; q < nlong; q += gstride() >> 5) {
    const int64_t f = first_item[q], m = nitems[q];
    const int64_t per = (m + 31) / 32;
    const int64_t a = lane * per, b = a + per < m ? a + per : m;
    P p{};
    bool have = false;
    for (int64_t k = a; k < b; ++k) {
      p = have ? A::comb(p, parts[f + k]) : parts[f + k];
      have = true;
    }
    if (!have) p = parts[f];  // an idle lane repeats chunk 0 and is masked below
    // lanes without items must not contribute: fold only lanes [0, used)
    const int used = static_cast<int>((m + per - 1) / per);
    P acc = p;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      P other = shfl(acc, (lane + o) & 31);
      if ((lane & (2 * o - 1)) == 0 && lane + o < used) acc = A::comb(acc, other);
    }
    if constexpr (std::is_same_v<T, int64_t> && OP == TQP_SUM) {
      // bounded chunk partials whose bounds leave int64: whether a prefix
      // really overflows (and where) needs the ordered monoid over the rows
      const SumI a0 = shfl(acc, 0);
      const __int128 lo64 = static_cast<__int128>(std::numeric_limits<int64_t>::min());
      const __int128 hi64 = static_cast<__int128>(std::numeric_limits<int64_t>::max());
      if (a0.bounded && (a0.mn < lo64 || a0.mx > hi64)) acc = warp_reduce_range<T, OP>(v, seg_lo[seg[q]], seg_hi[seg[q]]);
    }
    if (lane == 0) {
      if constexpr (OP == TQP_SUM) {
        write_result<T, OP>(out, seg[q], acc, err);
      } else {
        write_mm(out, seg[q], acc);
      }
    }
  }
}

// The validated segment plan of a segment-id vector: run bounds, the first
// empty segment, and the chunking of the long segments. Tensors are
// immutable, so the plan is computed on the first segmented_reduce over the
// ids and kept with their buffer: the reference's lowering reduces every
// aggregate over the same ids (operator_plan.cpp:355-386; Q1: 8 reductions),
// and only the first pays the validation, the run bounds and the host round
// trips that size the long-segment work.
struct SegPlan {
  int64_t rows = -1, num = -1;
  Tensor lo, hi;
  int64_t first_empty = -1;
  int64_t nlong = 0, items = 0;
  Tensor d_ilo, d_ihi, d_seg, d_first, d_cnt;
  std::shared_ptr<DevBuf> long_scratch;  // k_short's list of long segments
};

std::shared_ptr<SegPlan> seg_plan(Ctx& c, const Tensor& ids, int64_t num) {
  if (ids.buf) {
    auto p = std::static_pointer_cast<SegPlan>(ids.buf->seg_plan);
    if (p && p->rows == ids.rows && p->num == num) return p;
  }
  auto p = std::make_shared<SegPlan>();
  p->rows = ids.rows;
  p->num = num;
  const int64_t n = ids.rows;
  if (n) {
    c.reset_err();
    k_check_ids<<<c.grid_for(n, 256), 256, 0, c.stream>>>(ids.ptr<int64_t>(), n, num, c.d_err);
    c.count_launch();
    int64_t bad = c.read_err();
    if (bad >= 0) {
      int64_t row = bad / 2;
      if (bad % 2 == 0) kernel_fail("segmented_reduce: segment_ids decrease at row " + std::to_string(row), row);
      int64_t s = read_scalar<int64_t>(c, ids, row);
      kernel_fail("segmented_reduce: segment id " + std::to_string(s) + " out of range [0," + std::to_string(num) +
                      ") at row " + std::to_string(row),
                  row);
    }
  }
  p->lo = c.alloc(TQP_I64, num, 1);
  p->hi = c.alloc(TQP_I64, num, 1);
  if (num) {
    k_runs<<<c.grid_for(num, 256), 256, 0, c.stream>>>(ids.ptr<int64_t>(), n, num, p->lo.ptr<int64_t>(), p->hi.ptr<int64_t>());
    c.count_launch();
    c.reset_err();
    k_first_empty<<<c.grid_for(num, 256), 256, 0, c.stream>>>(p->lo.ptr<int64_t>(), p->hi.ptr<int64_t>(), num, c.d_err);
    c.count_launch();
    p->first_empty = c.read_err();
    // long segments (> kLong rows) and their kChunk-row chunks
    std::vector<int64_t> lo(num), hi(num);
    TQP_CUDA(cudaMemcpyAsync(lo.data(), p->lo.data(), 8 * num, cudaMemcpyDeviceToHost, c.stream));
    TQP_CUDA(cudaMemcpyAsync(hi.data(), p->hi.data(), 8 * num, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    std::vector<int64_t> segs, ilo, ihi, first, cnt;
    for (int64_t q = 0; q < num; ++q) {
      if (hi[q] - lo[q] <= kLong) continue;
      segs.push_back(q);
      first.push_back(static_cast<int64_t>(ilo.size()));
      for (int64_t a = lo[q]; a < hi[q]; a += kChunk) {
        ilo.push_back(a);
        ihi.push_back(std::min(a + kChunk, hi[q]));
      }
      cnt.push_back(static_cast<int64_t>(ilo.size()) - first.back());
    }
    p->nlong = static_cast<int64_t>(segs.size());
    p->items = static_cast<int64_t>(ilo.size());
    if (p->nlong) {
      p->d_ilo = upload(c, TQP_I64, p->items, 1, ilo.data());
      p->d_ihi = upload(c, TQP_I64, p->items, 1, ihi.data());
      p->d_seg = upload(c, TQP_I64, p->nlong, 1, segs.data());
      p->d_first = upload(c, TQP_I64, p->nlong, 1, first.data());
      p->d_cnt = upload(c, TQP_I64, p->nlong, 1, cnt.data());
      c.sync();  // the host vectors outlive the uploads
    }
    p->long_scratch = c.alloc_bytes(sizeof(int64_t) * (p->nlong + 1) + 16);
  }
  if (ids.buf) ids.buf->seg_plan = p;
  return p;
}

template <typename T, int OP>
void run_reduce(Ctx& c, const Tensor& values, const SegPlan& pl, Tensor& out) {
  using P = typename Acc<T, OP>::P;
  const int64_t num = pl.num;
  // short segments: one warp each (k_short lists the long ones it skips into
  // scratch; the plan already holds them, so nothing is read back)
  auto* long_count = static_cast<unsigned long long*>(pl.long_scratch->ptr);
  auto* long_list = reinterpret_cast<int64_t*>(static_cast<char*>(pl.long_scratch->ptr) + 16);
  TQP_CUDA(cudaMemsetAsync(long_count, 0, 8, c.stream));
  k_short<T, OP><<<c.grid_for(num * 32, 256), 256, 0, c.stream>>>(values.ptr<T>(), pl.lo.ptr<int64_t>(),
                                                                  pl.hi.ptr<int64_t>(), num, out.ptr<T>(), c.d_err,
                                                                  long_list, long_count);
  c.count_launch();
  if (!pl.nlong) return;
  auto parts = c.alloc_bytes(sizeof(P) * pl.items);
  k_long_chunks<T, OP><<<pl.items, 256, 0, c.stream>>>(values.ptr<T>(), pl.d_ilo.ptr<int64_t>(), pl.d_ihi.ptr<int64_t>(),
                                                       static_cast<P*>(parts->ptr));
  k_long_finish<T, OP><<<c.grid_for(pl.nlong * 32, 128), 128, 0, c.stream>>>(
      static_cast<P*>(parts->ptr), pl.d_seg.ptr<int64_t>(), pl.d_first.ptr<int64_t>(), pl.d_cnt.ptr<int64_t>(), pl.nlong,
      out.ptr<T>(), c.d_err, values.ptr<T>(), pl.lo.ptr<int64_t>(), pl.hi.ptr<int64_t>());
  c.count_launch(2);
}

}  // namespace

namespace k {

Tensor segmented_reduce(Ctx& c, const Tensor& values, const Tensor& ids, int64_t num, int op) {
  if (!values.is_vector()) kernel_fail("segmented_reduce: expected a vector (m=1)");
  if (ids.dtype != TQP_I64) kernel_fail(std::string("segmented_reduce: expected int64, got ") + dtype_name(ids.dtype));
  if (!ids.is_vector()) kernel_fail("segmented_reduce: expected a vector (m=1)");
  if (values.rows != ids.rows) kernel_fail("segmented_reduce: values/segment_ids length mismatch");
  if (num < 0) kernel_fail("segmented_reduce: negative segment count");
  auto plan = seg_plan(c, ids, num);
  const Tensor& lo = plan->lo;
  const Tensor& hi = plan->hi;
  if (op == TQP_COUNT) {
    Tensor o = c.alloc(TQP_I64, num, 1);
    if (num) {
      k_count<<<c.grid_for(num, 256), 256, 0, c.stream>>>(lo.ptr<int64_t>(), hi.ptr<int64_t>(), num, o.ptr<int64_t>());
      c.count_launch();
    }
    return o;
  }
  if (values.dtype == TQP_BOOL || values.dtype == TQP_STR8) kernel_fail("segmented_reduce: bool values not supported");
  if (op == TQP_MIN || op == TQP_MAX) {
    if (plan->first_empty >= 0)
      kernel_fail("segmented_reduce: empty segment " + std::to_string(plan->first_empty) + " for " +
                  (op == TQP_MIN ? "min" : "max"));
  } else if (op != TQP_SUM) {
    kernel_fail("segmented_reduce: bad op");
  }
  Tensor out = c.alloc(values.dtype, num, 1);
  if (!num) return out;
  if (op == TQP_SUM) TQP_CUDA(cudaMemsetAsync(out.data(), 0, out.bytes(), c.stream));
  c.reset_err();
  switch (values.dtype) {
    case TQP_F64:
      if (op == TQP_SUM) run_reduce<double, TQP_SUM>(c, values, *plan, out);
      else if (op == TQP_MIN) run_reduce<double, TQP_MIN>(c, values, *plan, out);
      else run_reduce<double, TQP_MAX>(c, values, *plan, out);
      break;
    case TQP_I64:
      if (op == TQP_SUM) run_reduce<int64_t, TQP_SUM>(c, values, *plan, out);
      else if (op == TQP_MIN) run_reduce<int64_t, TQP_MIN>(c, values, *plan, out);
      else run_reduce<int64_t, TQP_MAX>(c, values, *plan, out);
      break;
    case TQP_I32:
      if (op == TQP_SUM) run_reduce<int32_t, TQP_SUM>(c, values, *plan, out);
      else if (op == TQP_MIN) run_reduce<int32_t, TQP_MIN>(c, values, *plan, out);
      else run_reduce<int32_t, TQP_MAX>(c, values, *plan, out);
      break;
    default: kernel_fail("segmented_reduce: unsupported dtype");
  }
  if (op == TQP_SUM && values.dtype != TQP_F64) {
    int64_t s = c.read_err();
    if (s >= 0) kernel_fail("segmented_reduce: sum overflow in segment " + std::to_string(s));
  }
  return out;
}

}  // namespace k
}  // namespace tqp
