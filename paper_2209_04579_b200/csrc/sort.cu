// Stable LSD radix sort (8-bit digits) replacing the reference's serial
// std::stable_sort (argsort_stable, kernels.cpp:411-424) and the per-byte
// refinement passes of SortPermRows (executor.cpp:44-68).
//
// Onesweep: one histogram kernel reads the keys once and counts the digits
// of every pass; then each pass is ONE kernel. A tile (dynamic id) ranks its
// keys stably (warp match_any ranks, per-warp running digit counts, warps
// combined in order), takes each digit's offset from the tiles before it by
// a decoupled lookback over per-(tile, digit) descriptors, reorders the tile
// by digit in shared memory and writes each digit's run contiguously. The
// last pass writes only the payload. Passes whose digit is constant over all
// keys are skipped (an OR-reduction of key ^ key[0]), so a 1-byte string
// column costs one pass and dense int64 keys only their varying low bytes.
#include <string>
#include <vector>

#include "scan.cuh"

namespace tqp {
namespace k {
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

// ---- onesweep ---------------------------------------------------------------
constexpr int kOsItems = 8;                    // keys per thread (warp-striped)
constexpr int kOsTile = kThreads * kOsItems;  // 2048 keys per tile
constexpr int kMaxPasses = 8;

// digit counts of every pass at once: hist[q][d] for the q-th active pass
__global__ void __launch_bounds__(kThreads) k_os_hist(const uint64_t* __restrict__ keys, int64_t n,
                                                      const int* __restrict__ shifts, int npass,
                                                      unsigned long long* __restrict__ hist) {
  __shared__ unsigned int h[kMaxPasses][256];
  for (int i = threadIdx.x; i < kMaxPasses * 256; i += kThreads) (&h[0][0])[i] = 0u;
  __syncthreads();
  int sh[kMaxPasses];
#pragma unroll
  for (int q = 0; q < kMaxPasses; ++q) sh[q] = q < npass ? shifts[q] : 0;
  for (int64_t i = gtid(); i < n; i += gstride()) {
    const uint64_t k = keys[i];
#pragma unroll
    for (int q = 0; q < kMaxPasses; ++q)
      if (q < npass) atomicAdd(&h[q][(k >> sh[q]) & 255], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npass * 256; i += kThreads) {
    const unsigned v = (&h[0][0])[i];
    if (v) atomicAdd(hist + i, static_cast<unsigned long long>(v));
  }
}

// (tile, digit) descriptor: status in bits 62-63, count below
constexpr unsigned long long kOsPartial = 1ULL << 62, kOsInclusive = 2ULL << 62, kOsCount = (1ULL << 62) - 1;

__global__ void __launch_bounds__(kThreads, 4) k_onesweep(const uint64_t* __restrict__ kin, const int64_t* __restrict__ pin,
                                                       uint64_t* __restrict__ kout, int64_t* __restrict__ pout, int64_t n,
                                                       int shift, const unsigned long long* __restrict__ hist,
                                                       unsigned long long* desc, int* counter, int write_keys) {
  __shared__ uint64_t sk[kOsTile];
  __shared__ int64_t sp[kOsTile];
  __shared__ unsigned short wcnt[kWarps][256];
  __shared__ long long s_gbase[256];  // digit's first output row for this tile
  __shared__ int s_tstart[256];       // digit's first row in the reordered tile
  __shared__ int s_wsum[kWarps];
  __shared__ unsigned long long s_hsum[kWarps];
  __shared__ unsigned long long s_excl[256];  // rows of the digit in earlier tiles
  __shared__ int s_tcnt[256];
  __shared__ unsigned char s_active[256];     // digits some key has
  __shared__ int s_nact[kWarps];
  __shared__ int s_tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1);
  for (int d = lane; d < 256; d += 32) wcnt[warp][d] = 0;
  __syncthreads();
  const int tile = s_tile;
  const int64_t wbase = static_cast<int64_t>(tile) * kOsTile + static_cast<int64_t>(warp) * 32 * kOsItems + lane;
  uint64_t key[kOsItems];
  int64_t pay[kOsItems];
  int rank[kOsItems];
#pragma unroll
  for (int j = 0; j < kOsItems; ++j) {
    const int64_t i = wbase + j * 32;
    key[j] = i < n ? kin[i] : 0;
    pay[j] = i < n ? pin[i] : 0;
  }
  // stable ranks within the warp: items in order, lanes in order
#pragma unroll
  for (int j = 0; j < kOsItems; ++j) {
    const bool valid = wbase + j * 32 < n;
    const int d = valid ? static_cast<int>((key[j] >> shift) & 255) : 256;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int leader = __ffs(peers) - 1;
    int b = 0;
    if (lane == leader && valid) {
      b = wcnt[warp][d];
      wcnt[warp][d] = static_cast<unsigned short>(b + __popc(peers));
    }
    b = __shfl_sync(0xffffffffu, b, leader);
    rank[j] = b + __popc(peers & lt);
    __syncwarp();
  }
  __syncthreads();
  // per digit (thread d): warps' counts -> exclusive offsets, the tile count
  const int d = threadIdx.x;
  int run = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const int c = wcnt[w][d];
    wcnt[w][d] = static_cast<unsigned short>(run);
    run += c;
  }
  const int tcnt = run;
  // digit starts within the tile: exclusive scan of the tile counts
  int incl = tcnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_wsum[warp] = incl;
  // lookback for digit d over the tiles before this one (digits no key has
  // skip it: no tile publishes or reads them). Each tile publishes its
  // counts first; with few active digits (low-cardinality keys: Q1's flags)
  // a whole warp walks one digit, 32 predecessors per step, otherwise a
  // thread walks its digit 4 predecessors per step. The walk length is the
  // distance to the newest inclusive tile, i.e. the tiles in flight / step
  // width: one predecessor per step held Q1's 1-byte sort to 0.28 of HBM.
  const unsigned long long hv = hist[d];
  unsigned long long* my = desc + static_cast<int64_t>(tile) * 256 + d;
  if (hv) atomicExch(my, (tile == 0 ? kOsInclusive : kOsPartial) | static_cast<unsigned long long>(tcnt));
  const unsigned act = __ballot_sync(0xffffffffu, hv != 0);
  if (lane == 0) s_nact[warp] = __popc(act);
  s_tcnt[d] = tcnt;
  s_excl[d] = 0;
  __syncthreads();
  int nact = 0, apre = 0;
  for (int w = 0; w < kWarps; ++w) {
    apre += w < warp ? s_nact[w] : 0;
    nact += s_nact[w];
  }
  if (hv) s_active[apre + __popc(act & lt)] = static_cast<unsigned char>(d);
  __syncthreads();
  if (tile > 0) {
    if (nact <= 4 * kWarps) {
      for (int a = warp; a < nact; a += kWarps) {
        const int dd = s_active[a];
        unsigned long long excl = 0;
        for (int base = tile - 1;; base -= 32) {
          const int t = base - lane;
          unsigned long long v = kOsInclusive;
          if (t >= 0) {
            const volatile unsigned long long* q =
                reinterpret_cast<const volatile unsigned long long*>(desc + static_cast<int64_t>(t) * 256 + dd);
            do {
              v = *q;
            } while (!(v >> 62));
          }
          const unsigned incl_m = __ballot_sync(0xffffffffu, (v & kOsInclusive) != 0);
          const int stop = incl_m ? __ffs(incl_m) - 1 : 31;  // newest inclusive tile, else the whole window
          unsigned long long c = lane <= stop ? (v & kOsCount) : 0ULL;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
          excl += c;
          if (incl_m) break;
        }
        if (lane == 0) {
          s_excl[dd] = excl;
          atomicExch(desc + static_cast<int64_t>(tile) * 256 + dd,
                     kOsInclusive | (excl + static_cast<unsigned long long>(s_tcnt[dd])));
        }
      }
    } else if (hv) {
      unsigned long long excl = 0;
      bool done = false;
      for (int t0 = tile - 1; !done; t0 -= 4) {
        unsigned long long v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = t0 - u;
          v[u] = t >= 0 ? *reinterpret_cast<const volatile unsigned long long*>(desc + static_cast<int64_t>(t) * 256 + d)
                        : kOsInclusive;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = t0 - u;
          while (!(v[u] >> 62)) v[u] = *reinterpret_cast<const volatile unsigned long long*>(desc + static_cast<int64_t>(t) * 256 + d);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (done) break;
          excl += v[u] & kOsCount;
          if (v[u] & kOsInclusive) done = true;
        }
      }
      s_excl[d] = excl;
      atomicExch(my, kOsInclusive | (excl + static_cast<unsigned long long>(tcnt)));
    }
  }
  // the digit's global start: rows of smaller digits (all tiles, an
  // exclusive scan of the pass histogram) + rows of this digit in earlier tiles
  unsigned long long hinc = hv;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, hinc, o);
    if (lane >= o) hinc += y;
  }
  if (lane == 31) s_hsum[warp] = hinc;
  __syncthreads();
  int wpre = 0;
  unsigned long long hpre = 0;
  for (int w = 0; w < warp; ++w) {
    wpre += s_wsum[w];
    hpre += s_hsum[w];
  }
  s_tstart[d] = wpre + incl - tcnt;
  s_gbase[d] = static_cast<long long>(hpre + hinc - hv + s_excl[d]);
  __syncthreads();
  // reorder the tile by digit (stable) in shared memory
#pragma unroll
  for (int j = 0; j < kOsItems; ++j) {
    if (wbase + j * 32 < n) {
      const int dj = static_cast<int>((key[j] >> shift) & 255);
      const int loc = s_tstart[dj] + wcnt[warp][dj] + rank[j];
      sk[loc] = key[j];
      sp[loc] = pay[j];
    }
  }
  __syncthreads();
  // each digit's run to consecutive output rows
  const int64_t tile_rows = n - static_cast<int64_t>(tile) * kOsTile < kOsTile ? n - static_cast<int64_t>(tile) * kOsTile : kOsTile;
  for (int i = threadIdx.x; i < tile_rows; i += kThreads) {
    const uint64_t k = sk[i];
    const int di = static_cast<int>((k >> shift) & 255);
    const int64_t dst = s_gbase[di] + (i - s_tstart[di]);
    if (write_keys) kout[dst] = k;
    pout[dst] = sp[i];
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
  std::vector<int> shifts;
  for (int shift = 0; shift < 64; shift += 8)
    if ((diff >> shift) & 255ULL) shifts.push_back(shift);
  const int npass = static_cast<int>(shifts.size());
  const int64_t tiles = (n + kOsTile - 1) / kOsTile;
  // one zeroed scratch: pass shifts, the digit histograms of every pass, and
  // per pass a tile counter and the (tile, digit) lookback descriptors
  const size_t hist_off = 64, ctr_off = hist_off + sizeof(unsigned long long) * 256 * kMaxPasses;
  const size_t desc_off = (ctr_off + sizeof(int) * kMaxPasses + 255) & ~size_t(255);
  const size_t desc_bytes = sizeof(unsigned long long) * 256 * static_cast<size_t>(tiles);
  // one descriptor array, cleared before each pass (all passes' at once
  // would be npass x 2 KB per 2048 keys: 4.8 GB for 600 M int64 keys)
  auto scratch = c.alloc_bytes(desc_off + desc_bytes);
  unsigned char* sb = static_cast<unsigned char*>(scratch->ptr);
  TQP_CUDA(cudaMemsetAsync(sb, 0, desc_off, c.stream));
  TQP_CUDA(cudaMemcpyAsync(sb, shifts.data(), sizeof(int) * npass, cudaMemcpyHostToDevice, c.stream));
  auto* hist = reinterpret_cast<unsigned long long*>(sb + hist_off);
  k_os_hist<<<c.grid_for(n, kThreads, 4, 4), kThreads, 0, c.stream>>>(reinterpret_cast<uint64_t*>(keys.data()), n,
                                                                      reinterpret_cast<const int*>(sb), npass, hist);
  c.count_launch();
  Tensor k2 = c.alloc(TQP_I64, n, 1), p2 = c.alloc(TQP_I64, n, 1);
  // payload may be shared with the caller (immutable): write to fresh buffers
  Tensor kin = keys, pin = payload, kout = k2, pout = p2;
  for (int q = 0; q < npass; ++q) {
    const bool last = q + 1 == npass;
    TQP_CUDA(cudaMemsetAsync(sb + desc_off, 0, desc_bytes, c.stream));
    k_onesweep<<<tiles, kThreads, 0, c.stream>>>(
        reinterpret_cast<uint64_t*>(kin.data()), pin.ptr<int64_t>(), reinterpret_cast<uint64_t*>(kout.data()),
        pout.ptr<int64_t>(), n, shifts[q], hist + 256 * q, reinterpret_cast<unsigned long long*>(sb + desc_off),
        reinterpret_cast<int*>(sb + ctr_off) + q, last ? 0 : 1);
    c.count_launch();
    if (q == 0) {
      // never overwrite the caller's payload: a second ping buffer
      kin = kout;
      pin = pout;
      if (!last) {
        kout = c.alloc(TQP_I64, n, 1);
        pout = c.alloc(TQP_I64, n, 1);
      }
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
