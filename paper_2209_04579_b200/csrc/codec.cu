// Compressed columnar host format (tqp_b200.h, "compressed columnar host
// format"): a lossless per-column codec chosen on the host and decoded on
// the device. The reference's loader only parses CSV text
// (proj/src/columnar.cpp:453-527); SURVEY.md 8(f)1 names a binary columnar
// format with pinned-staging DMA as the next step of the loader, so that an
// end-to-end run (host columns -> device -> query) is not bound by moving the
// reference's 8-byte values over PCIe.
//
// Encoding runs once per column (when the host copy is made), on the host's
// cores; every value is verified, so a column that does not fit a codec
// exactly stays RAW. Decoding is one grid-stride kernel per column.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "device.cuh"
#include "tqp_internal.hpp"

namespace tqp {
namespace {

// ---- host: parallel helpers --------------------------------------------------
int host_threads(int64_t n) {
  const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(hw, n / (1 << 20) + 1)));
}

template <typename F>
void parallel_chunks(int64_t n, F&& f) {  // f(thread, lo, hi)
  const int nt = host_threads(n);
  if (nt == 1) {
    f(0, 0, n);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t) {
    const int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
    th.emplace_back([&f, t, lo, hi] { f(t, lo, hi); });
  }
  for (auto& x : th) x.join();
}

// codes are bit-packed little-endian into 32-bit words: code i occupies
// bits [i * w, (i + 1) * w) of the stream (w = 1..32); one spare word at the
// end lets a decoder always read two words
int bits_for(uint64_t max_code) {
  int b = 1;
  while (b < 32 && (max_code >> b) != 0) ++b;
  return (max_code >> b) != 0 ? 0 : b;  // 0: does not fit 32 bits
}
int64_t packed_bytes(int64_t n, int w) { return 4 * ((n * w + 31) / 32 + 1); }

// packs code(i) for i in [0, n) in parallel; chunks start on 32-code
// boundaries so no two threads share a word
template <typename Code>
void pack_codes(int64_t n, int w, uint32_t* words, Code&& code) {
  std::memset(words, 0, static_cast<size_t>(packed_bytes(n, w)));
  const int64_t groups = (n + 31) / 32;
  parallel_chunks(groups, [&](int, int64_t g0, int64_t g1) {
    for (int64_t i = g0 * 32; i < std::min(n, g1 * 32); ++i) {
      const uint64_t u = code(i);
      const int64_t bit = i * w;
      const int64_t wi = bit >> 5;
      const int sh = static_cast<int>(bit & 31);
      words[wi] |= static_cast<uint32_t>(u << sh);
      if (sh + w > 32) words[wi + 1] |= static_cast<uint32_t>(u >> (32 - sh));
    }
  });
}

// ---- host: codecs --------------------------------------------------------------
// FOR over integers (int64 or byte values): base = min, scale = gcd of
// (v - min) (unsigned), codes of the fewest bits that hold (max - min) /
// scale.
struct ForPlan {
  int64_t base = 0;
  uint64_t scale = 1;
  int bits = 0;  // 0: does not fit
};

template <typename T>
ForPlan plan_for(const T* v, int64_t n) {
  ForPlan p;
  if (n == 0) return p;
  const int nt = host_threads(n);
  std::vector<int64_t> mn(nt, INT64_MAX), mx(nt, INT64_MIN);
  parallel_chunks(n, [&](int t, int64_t lo, int64_t hi) {
    int64_t a = INT64_MAX, b = INT64_MIN;
    for (int64_t i = lo; i < hi; ++i) {
      a = std::min<int64_t>(a, v[i]);
      b = std::max<int64_t>(b, v[i]);
    }
    mn[t] = a;
    mx[t] = b;
  });
  const int64_t lo = *std::min_element(mn.begin(), mn.end()), hi = *std::max_element(mx.begin(), mx.end());
  const uint64_t range = static_cast<uint64_t>(hi) - static_cast<uint64_t>(lo);
  std::vector<uint64_t> g(nt, 0);
  parallel_chunks(n, [&](int t, int64_t a, int64_t b) {
    uint64_t x = 0;
    for (int64_t i = a; i < b && x != 1; ++i) {
      const uint64_t d = static_cast<uint64_t>(static_cast<int64_t>(v[i])) - static_cast<uint64_t>(lo);
      if (x == 0 ? d != 0 : d % x != 0) x = std::gcd(x, d);
    }
    g[t] = x;
  });
  uint64_t scale = 0;
  for (uint64_t x : g) scale = std::gcd(scale, x);
  if (scale == 0) scale = 1;  // every value equal
  p.base = lo;
  p.scale = scale;
  p.bits = bits_for(range / scale);
  return p;
}

template <typename T>
int64_t pack_for(const T* v, int64_t n, const ForPlan& p, void* out, tqp_codec* c) {
  pack_codes(n, p.bits, static_cast<uint32_t*>(out), [&](int64_t i) {
    return (static_cast<uint64_t>(static_cast<int64_t>(v[i])) - static_cast<uint64_t>(p.base)) / p.scale;
  });
  c->codec = TQP_CODEC_FOR;
  c->width = p.bits;
  c->base = p.base;
  c->scale = static_cast<int64_t>(p.scale);
  return packed_bytes(n, p.bits);
}

template <typename T>
int64_t try_for(const T* v, int64_t n, void* out, int64_t cap, tqp_codec* c) {
  const ForPlan p = plan_for(v, n);
  if (!p.bits || packed_bytes(n, p.bits) > cap) return -1;
  return pack_for(v, n, p, out, c);
}

// DELTA over a non-decreasing int64 vector (sorted keys): e_0 = 0,
// e_i = v_i - v_(i-1) >= 0, codes e_i / scale (scale = gcd of the e_i);
// v_i = v_0 + scale * (sum of codes up to i). Returns the plan (bits 0: not
// sorted or does not fit).
ForPlan plan_delta(const int64_t* v, int64_t n) {
  ForPlan p;
  if (n < 2) return p;
  const int nt = host_threads(n);
  std::vector<uint64_t> g(nt, 0), mx(nt, 0);
  std::vector<char> unsorted(nt, 0);
  parallel_chunks(n, [&](int t, int64_t a, int64_t b) {
    uint64_t x = 0, m = 0;
    for (int64_t i = std::max<int64_t>(a, 1); i < b; ++i) {
      if (v[i] < v[i - 1]) {
        unsorted[t] = 1;
        return;
      }
      const uint64_t d = static_cast<uint64_t>(v[i]) - static_cast<uint64_t>(v[i - 1]);
      m = std::max(m, d);
      if (x != 1 && (x == 0 ? d != 0 : d % x != 0)) x = std::gcd(x, d);
    }
    g[t] = x;
    mx[t] = m;
  });
  for (char u : unsorted)
    if (u) return p;
  uint64_t scale = 0, m = 0;
  for (int t = 0; t < nt; ++t) {
    scale = std::gcd(scale, g[t]);
    m = std::max(m, mx[t]);
  }
  if (scale == 0) scale = 1;
  p.base = v[0];
  p.scale = scale;
  p.bits = bits_for(m / scale);
  return p;
}

int64_t pack_delta(const int64_t* v, int64_t n, const ForPlan& p, void* out, tqp_codec* c) {
  pack_codes(n, p.bits, static_cast<uint32_t*>(out), [&](int64_t i) {
    return i == 0 ? 0ull : (static_cast<uint64_t>(v[i]) - static_cast<uint64_t>(v[i - 1])) / p.scale;
  });
  c->codec = TQP_CODEC_DELTA;
  c->width = p.bits;
  c->base = p.base;
  c->scale = static_cast<int64_t>(p.scale);
  return packed_bytes(n, p.bits);
}

// DICT over float64 bit patterns (<= 256 distinct).
int64_t try_dict(const uint64_t* v, int64_t n, void* out, int64_t cap, tqp_codec* c) {
  if (n == 0) return -1;
  const int nt = host_threads(n);
  std::vector<std::vector<uint64_t>> sets(nt);
  std::vector<char> over(nt, 0);
  parallel_chunks(n, [&](int t, int64_t a, int64_t b) {
    std::vector<uint64_t>& s = sets[t];
    uint64_t last = 0;
    bool have = false;
    for (int64_t i = a; i < b; ++i) {
      if (have && v[i] == last) continue;
      if (std::find(s.begin(), s.end(), v[i]) == s.end()) {
        if (s.size() >= 256) {
          over[t] = 1;
          return;
        }
        s.push_back(v[i]);
      }
      last = v[i];
      have = true;
    }
  });
  for (char o : over)
    if (o) return -1;
  std::vector<uint64_t> dict;
  for (auto& s : sets) dict.insert(dict.end(), s.begin(), s.end());
  std::sort(dict.begin(), dict.end());
  dict.erase(std::unique(dict.begin(), dict.end()), dict.end());
  if (dict.size() > 256) return -1;
  const int w = bits_for(dict.size() - 1);
  const int64_t bytes = 8 * static_cast<int64_t>(dict.size()) + packed_bytes(n, w);
  if (bytes > cap) return -1;
  std::memcpy(out, dict.data(), 8 * dict.size());
  pack_codes(n, w, reinterpret_cast<uint32_t*>(static_cast<unsigned char*>(out) + 8 * dict.size()), [&](int64_t i) {
    return static_cast<uint64_t>(std::lower_bound(dict.begin(), dict.end(), v[i]) - dict.begin());
  });
  c->codec = TQP_CODEC_DICT;
  c->width = w;
  c->dict_n = static_cast<int32_t>(dict.size());
  return bytes;
}

// DEC over float64: v == (double)k / 10^d exactly for an integer k, every row.
int64_t try_dec(const double* v, int64_t n, void* out, int64_t cap, tqp_codec* c) {
  if (n == 0) return -1;
  const int nt = host_threads(n);
  for (int d : {0, 1, 2, 3, 4}) {  // the first exact one has the smallest code range
    const double scale = std::pow(10.0, d);
    std::vector<int64_t> mn(nt, INT64_MAX), mx(nt, INT64_MIN);
    std::vector<char> bad(nt, 0);
    parallel_chunks(n, [&](int t, int64_t a, int64_t b) {
      int64_t lo = INT64_MAX, hi = INT64_MIN;
      for (int64_t i = a; i < b; ++i) {
        const double x = v[i];
        if (!std::isfinite(x) || std::fabs(x) * scale >= 9.0e15) {
          bad[t] = 1;
          return;
        }
        const int64_t k = std::llrint(x * scale);
        const double back = static_cast<double>(k) / scale;
        uint64_t bx, bb;
        std::memcpy(&bx, &x, 8);
        std::memcpy(&bb, &back, 8);
        if (bx != bb) {
          bad[t] = 1;
          return;
        }
        lo = std::min(lo, k);
        hi = std::max(hi, k);
      }
      mn[t] = lo;
      mx[t] = hi;
    });
    if (std::find(bad.begin(), bad.end(), 1) != bad.end()) continue;
    const int64_t lo = *std::min_element(mn.begin(), mn.end()), hi = *std::max_element(mx.begin(), mx.end());
    const int w = bits_for(static_cast<uint64_t>(hi - lo));
    if (!w || packed_bytes(n, w) > cap) return -1;
    pack_codes(n, w, static_cast<uint32_t*>(out),
               [&](int64_t i) { return static_cast<uint64_t>(std::llrint(v[i] * scale) - lo); });
    c->codec = TQP_CODEC_DEC;
    c->width = w;
    c->base = lo;
    c->scale = static_cast<int64_t>(scale);
    return packed_bytes(n, w);
  }
  return -1;
}

// ROWDICT over byte rows (STR8 / BOOL, any width): <= 256 distinct rows of
// `cols` bytes, the dictionary rows (ascending bytes) then the codes.
int64_t try_rowdict(const uint8_t* v, int64_t n, int64_t cols, void* out, int64_t cap, tqp_codec* c) {
  if (n == 0) return -1;
  const int nt = host_threads(n);
  std::vector<std::vector<std::string>> sets(nt);
  std::vector<char> over(nt, 0);
  parallel_chunks(n, [&](int t, int64_t a, int64_t b) {
    std::vector<std::string>& s = sets[t];
    std::string row(static_cast<size_t>(cols), '\0');
    for (int64_t i = a; i < b; ++i) {
      row.assign(reinterpret_cast<const char*>(v + i * cols), static_cast<size_t>(cols));
      if (std::find(s.begin(), s.end(), row) == s.end()) {
        if (s.size() >= 256) {
          over[t] = 1;
          return;
        }
        s.push_back(row);
      }
    }
  });
  for (char o : over)
    if (o) return -1;
  std::vector<std::string> dict;
  for (auto& s : sets) dict.insert(dict.end(), s.begin(), s.end());
  std::sort(dict.begin(), dict.end());
  dict.erase(std::unique(dict.begin(), dict.end()), dict.end());
  if (dict.size() > 256) return -1;
  const int w = bits_for(dict.size() - 1);
  const int64_t dict_bytes = (static_cast<int64_t>(dict.size()) * cols + 7) & ~int64_t(7);
  const int64_t bytes = dict_bytes + packed_bytes(n, w);
  if (bytes > cap) return -1;
  unsigned char* o = static_cast<unsigned char*>(out);
  std::memset(o, 0, static_cast<size_t>(dict_bytes));
  for (size_t d = 0; d < dict.size(); ++d) std::memcpy(o + d * cols, dict[d].data(), static_cast<size_t>(cols));
  pack_codes(n, w, reinterpret_cast<uint32_t*>(o + dict_bytes), [&](int64_t i) {
    const std::string_view row(reinterpret_cast<const char*>(v + i * cols), static_cast<size_t>(cols));
    return static_cast<uint64_t>(
        std::lower_bound(dict.begin(), dict.end(), row, [](const std::string& a, std::string_view b) { return a < b; }) -
        dict.begin());
  });
  c->codec = TQP_CODEC_ROWDICT;
  c->width = w;
  c->dict_n = static_cast<int32_t>(dict.size());
  return bytes;
}

// ---- device: decoders ------------------------------------------------------------
__device__ __forceinline__ uint32_t unpack(const uint32_t* __restrict__ words, int64_t i, int w) {
  const int64_t bit = i * w;
  const int64_t wi = bit >> 5;
  const uint64_t two = static_cast<uint64_t>(__ldg(words + wi)) | (static_cast<uint64_t>(__ldg(words + wi + 1)) << 32);
  return static_cast<uint32_t>((two >> (bit & 31)) & ((w == 32 ? 0x100000000ull : (1ull << w)) - 1));
}

template <typename T>
__global__ void k_decode_for(const uint32_t* __restrict__ words, int w, int64_t n, int64_t base, int64_t scale,
                             T* __restrict__ out) {
  for (int64_t i = gtid(); i < n; i += gstride())
    out[i] = static_cast<T>(static_cast<uint64_t>(base) + static_cast<uint64_t>(scale) * unpack(words, i, w));
}

__global__ void k_delta_finish(const int64_t* __restrict__ excl, const int64_t* __restrict__ step, int64_t n,
                               int64_t base, int64_t* __restrict__ out) {
  for (int64_t i = gtid(); i < n; i += gstride())
    out[i] = static_cast<int64_t>(static_cast<uint64_t>(base) + static_cast<uint64_t>(excl[i]) + static_cast<uint64_t>(step[i]));
}

__global__ void k_decode_rowdict(const uint8_t* __restrict__ dict, const uint32_t* __restrict__ words, int w,
                                 int64_t n, int64_t cols, uint8_t* __restrict__ out) {
  for (int64_t e = gtid(); e < n * cols; e += gstride()) {
    const int64_t r = e / cols;
    out[e] = dict[static_cast<int64_t>(unpack(words, r, w)) * cols + (e - r * cols)];
  }
}

__global__ void k_decode_dec(const uint32_t* __restrict__ words, int w, int64_t n, int64_t base, double scale,
                             double* __restrict__ out) {
  for (int64_t i = gtid(); i < n; i += gstride())
    out[i] = __ddiv_rn(static_cast<double>(base + static_cast<int64_t>(unpack(words, i, w))), scale);
}

__global__ void k_decode_dict(const unsigned long long* __restrict__ dict, int nd, const uint32_t* __restrict__ words,
                              int w, int64_t n, unsigned long long* __restrict__ out) {
  __shared__ unsigned long long s_dict[256];
  for (int i = threadIdx.x; i < nd; i += blockDim.x) s_dict[i] = dict[i];
  __syncthreads();
  for (int64_t i = gtid(); i < n; i += gstride()) out[i] = s_dict[unpack(words, i, w)];
}

}  // namespace

int64_t codec_bound(int dtype, int64_t rows, int64_t cols) {
  return rows * cols * static_cast<int64_t>(dtype_size(dtype)) + 8 * 256 + 64;
}

int64_t codec_encode(int dtype, int64_t rows, int64_t cols, const void* host, void* out, int64_t cap, tqp_codec* c) {
  if (rows < 0 || cols < 1 || dtype < TQP_BOOL || dtype > TQP_STR8) throw Error(TQP_ERR_ARG, "codec: bad column shape");
  *c = tqp_codec{};
  c->codec = TQP_CODEC_RAW;
  const int64_t raw = rows * cols * static_cast<int64_t>(dtype_size(dtype));
  // each attempt writes straight into `out`; a failed one leaves it to the
  // next, and RAW (below) overwrites whatever a failed attempt wrote
  if (cols == 1 && rows > 0 && dtype == TQP_I64) {
    const auto* v = static_cast<const int64_t*>(host);
    const ForPlan f = plan_for(v, rows), d = plan_delta(v, rows);
    const int64_t lim = std::min(cap, raw - 1);
    if (d.bits && (!f.bits || d.bits < f.bits) && packed_bytes(rows, d.bits) <= lim) return pack_delta(v, rows, d, out, c);
    if (f.bits && packed_bytes(rows, f.bits) <= lim) return pack_for(v, rows, f, out, c);
  }
  if (rows > 0 && (dtype == TQP_STR8 || dtype == TQP_BOOL)) {
    // byte rows: a row dictionary (<= 256 distinct rows), else one-byte
    // values by FOR
    const auto* v = static_cast<const uint8_t*>(host);
    int64_t b = try_rowdict(v, rows, cols, out, std::min(cap, raw - 1), c);
    if (b >= 0) return b;
    if (cols == 1) {
      b = try_for(v, rows, out, std::min(cap, raw - 1), c);
      if (b >= 0) return b;
    }
  }
  if (cols == 1 && rows > 0 && dtype == TQP_F64) {
    // DICT first (8 B x entries + 1 B per row); DEC can only beat it at one
    // byte per row too, so it is tried when DICT does not apply
    int64_t b = try_dict(static_cast<const uint64_t*>(host), rows, out, std::min(cap, raw - 1), c);
    if (b >= 0) return b;
    b = try_dec(static_cast<const double*>(host), rows, out, std::min(cap, raw - 1), c);
    if (b >= 0) return b;
  }
  *c = tqp_codec{};
  c->codec = TQP_CODEC_RAW;
  if (raw > cap) throw Error(TQP_ERR_ARG, "codec: output buffer too small");
  if (raw) std::memcpy(out, host, static_cast<size_t>(raw));
  return raw;
}

Tensor decode_column(Ctx& c, int dtype, int64_t rows, int64_t cols, const tqp_codec& k, const void* payload,
                     int64_t bytes) {
  if (rows < 0 || cols < 1) throw Error(TQP_ERR_ARG, "codec: bad column shape");
  if (k.codec == TQP_CODEC_RAW) {
    if (bytes != rows * cols * static_cast<int64_t>(dtype_size(dtype))) throw Error(TQP_ERR_ARG, "codec: payload size");
    return upload(c, dtype, rows, cols, payload);
  }
  const bool vec = cols == 1;
  const bool w_ok = k.width >= 1 && k.width <= 32;
  const bool byte_col = dtype == TQP_STR8 || dtype == TQP_BOOL;
  if (k.codec == TQP_CODEC_FOR && !(vec && (dtype == TQP_I64 || byte_col) && w_ok && bytes == packed_bytes(rows, k.width)))
    throw Error(TQP_ERR_ARG, "codec: bad FOR column");
  if (k.codec == TQP_CODEC_DEC && !(vec && dtype == TQP_F64 && w_ok && bytes == packed_bytes(rows, k.width) && k.scale > 0))
    throw Error(TQP_ERR_ARG, "codec: bad DEC column");
  if (k.codec == TQP_CODEC_DICT && !(vec && dtype == TQP_F64 && w_ok && k.dict_n >= 1 && k.dict_n <= 256 &&
                                     bytes == 8LL * k.dict_n + packed_bytes(rows, k.width)))
    throw Error(TQP_ERR_ARG, "codec: bad DICT column");
  if (k.codec == TQP_CODEC_DELTA && !(vec && dtype == TQP_I64 && w_ok && bytes == packed_bytes(rows, k.width)))
    throw Error(TQP_ERR_ARG, "codec: bad DELTA column");
  const int64_t rd_bytes = (static_cast<int64_t>(k.dict_n) * cols + 7) & ~int64_t(7);
  if (k.codec == TQP_CODEC_ROWDICT && !(byte_col && w_ok && k.dict_n >= 1 && k.dict_n <= 256 &&
                                        bytes == rd_bytes + packed_bytes(rows, k.width)))
    throw Error(TQP_ERR_ARG, "codec: bad ROWDICT column");
  if (k.codec < TQP_CODEC_RAW || k.codec > TQP_CODEC_ROWDICT) throw Error(TQP_ERR_ARG, "codec: unknown codec");
  // The copy runs on the context's copy stream into a staging slot (Ctx::
  // Stage): it waits only for the decode that last read the slot, so the
  // copies of consecutive columns run back to back. The decode runs on the
  // decode stream (allocations included: `stream` is swapped for this
  // function), which waits for the copy only; the tensor carries a ready
  // event that the context stream waits for at its first use (Ctx::
  // wait_ready), so work already queued there - a query over the previous
  // tables - overlaps this upload.
  struct StreamSwap {
    Ctx& c;
    cudaStream_t old;
    bool old_pool_only;
    StreamSwap(Ctx& c_, cudaStream_t s) : c(c_), old(c_.stream), old_pool_only(c_.pool_only) {
      c.stream = s;
      c.pool_only = true;  // the small-block free list is ordered by the context stream only
    }
    ~StreamSwap() {
      c.stream = old;
      c.pool_only = old_pool_only;
    }
  } swap(c, c.decodes());
  Tensor out = c.alloc(dtype, rows, cols);
  Ctx::Stage* slot = nullptr;
  if (bytes) {
    cudaStream_t cs = c.copies();
    slot = &c.stages[c.stage_next];
    c.stage_next = (c.stage_next + 1) % Ctx::kStages;
    if (slot->freed) TQP_CUDA(cudaStreamWaitEvent(cs, slot->freed, 0));
    if (slot->cap < static_cast<size_t>(bytes)) {
      if (slot->ptr) {
        TQP_CUDA(cudaStreamSynchronize(cs));  // the slot's last reader is done
        TQP_CUDA(cudaFree(slot->ptr));
      }
      const size_t cap = (std::max(static_cast<size_t>(bytes), 2 * slot->cap) + (size_t(1) << 20) - 1) & ~((size_t(1) << 20) - 1);
      TQP_CUDA(cudaMalloc(&slot->ptr, cap));
      slot->cap = cap;
    }
    TQP_CUDA(cudaMemcpyAsync(slot->ptr, payload, static_cast<size_t>(bytes), cudaMemcpyHostToDevice, cs));
    cudaEvent_t landed = c.take_event();
    TQP_CUDA(cudaEventRecord(landed, cs));
    TQP_CUDA(cudaStreamWaitEvent(c.stream, landed, 0));
    c.give_event(landed);
    if (!slot->freed) TQP_CUDA(cudaEventCreateWithFlags(&slot->freed, cudaEventDisableTiming));
  }
  struct SlotRelease {  // the slot is free again once the decode stream has run this column's decode
    Ctx& c;
    Ctx::Stage* s;
    ~SlotRelease() {
      if (s) cudaEventRecord(s->freed, c.stream);
    }
  } release{c, slot};
  // the decoded tensor's ready event, recorded after its last decode kernel
  auto ready = [&]() -> Tensor {
    if (out.buf && !out.buf->ready) {
      TQP_CUDA(cudaEventCreateWithFlags(&out.buf->ready, cudaEventDisableTiming));
      TQP_CUDA(cudaEventRecord(out.buf->ready, c.stream));
    }
    return out;
  };
  if (!rows) return ready();
  const int grid = c.grid_for(rows, 256, 4);
  const void* staged_ptr = slot ? slot->ptr : nullptr;
  const auto* words = static_cast<const uint32_t*>(staged_ptr);
  if (k.codec == TQP_CODEC_FOR) {
    if (byte_col)
      k_decode_for<uint8_t><<<grid, 256, 0, c.stream>>>(words, k.width, rows, k.base, k.scale, out.ptr<uint8_t>());
    else
      k_decode_for<int64_t><<<grid, 256, 0, c.stream>>>(words, k.width, rows, k.base, k.scale, out.ptr<int64_t>());
  } else if (k.codec == TQP_CODEC_DELTA) {
    // the steps, then their inclusive scan (exclusive scan + the step)
    Tensor steps = c.alloc(TQP_I64, rows, 1);
    k_decode_for<int64_t><<<grid, 256, 0, c.stream>>>(words, k.width, rows, 0, k.scale, steps.ptr<int64_t>());
    c.count_launch();
    // no overflow readback (and so no host round trip): the encoder has
    // verified that every prefix is a value of the column
    Tensor excl = k::prefix_sum_unchecked(c, steps);
    k_delta_finish<<<grid, 256, 0, c.stream>>>(excl.ptr<int64_t>(), steps.ptr<int64_t>(), rows, k.base, out.ptr<int64_t>());
  } else if (k.codec == TQP_CODEC_ROWDICT) {
    const auto* dict = static_cast<const uint8_t*>(staged_ptr);
    k_decode_rowdict<<<c.grid_for(rows * cols, 256, 4), 256, 0, c.stream>>>(
        dict, reinterpret_cast<const uint32_t*>(dict + rd_bytes), k.width, rows, cols, out.ptr<uint8_t>());
  } else if (k.codec == TQP_CODEC_DEC) {
    k_decode_dec<<<grid, 256, 0, c.stream>>>(words, k.width, rows, k.base, static_cast<double>(k.scale), out.ptr<double>());
  } else {
    const auto* dict = static_cast<const unsigned long long*>(staged_ptr);
    k_decode_dict<<<grid, 256, 0, c.stream>>>(dict, k.dict_n, reinterpret_cast<const uint32_t*>(dict + k.dict_n), k.width,
                                              rows, out.ptr<unsigned long long>());
  }
  c.count_launch();
  return ready();
}

}  // namespace tqp
