// CSV -> device columns: tensql::parse_csv_text /
// load_csv (columnar.cpp:453-527) with the parsing on the GPU.
//
//   host    header line: split + case-insensitive name check (the reference's
//           messages); the data bytes go to HBM in one copy
//   k_nl_count / k_nl_write   newline positions: per-chunk counts, one
//           exclusive scan, per-thread ballot offsets (128-bit loads)
//   k_csv_rows  one thread per line: split on the delimiter, parse every
//           field straight into its column (fparse.cuh: the same parsers the
//           CPU check holds to std::from_chars / encode_date), record string
//           extents, and the first error (line, field) by atomicMin on a key
//           that orders errors as the reference's row-major loop meets them
//   k_csv_slow  the rare float64 fields with > 19 significant digits whose
//           candidates differ: exact bignum comparison, one thread each
//   k_csv_str   Utf8 columns as zero-padded rows of width max(1, longest)
// An error is re-derived on the host from that one field's bytes, so the
// message is the reference's ("<origin>:<line>: column '<c>' (field k): ...").
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "device.cuh"
#include "executor.hpp"
#include "fparse.cuh"
#include "tqp_internal.hpp"

namespace tqp {
namespace {

constexpr int kNlThreads = 256;
constexpr int64_t kNlChunk = kNlThreads * 16 * 8;  // bytes per block: 8 x 16 B per thread

__global__ void __launch_bounds__(kNlThreads) k_nl_count(const unsigned char* __restrict__ d, int64_t n,
                                                         long long* __restrict__ counts) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kNlChunk;
  unsigned c = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int64_t off = base + (static_cast<int64_t>(k) * kNlThreads + threadIdx.x) * 16;
    if (off >= n) break;
    const uint4 v = *reinterpret_cast<const uint4*>(d + off);  // buffer padded to 16 B
    const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int64_t p = off + q * 4 + b;
        c += (p < n && ((w[q] >> (8 * b)) & 0xff) == '\n') ? 1u : 0u;
      }
  }
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ unsigned s[kNlThreads / 32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int i = 0; i < kNlThreads / 32; ++i) t += s[i];
    counts[blockIdx.x] = t;
  }
}

// same traversal order as k_nl_count; offsets[] is the exclusive scan
__global__ void __launch_bounds__(kNlThreads) k_nl_write(const unsigned char* __restrict__ d, int64_t n,
                                                         const long long* __restrict__ offsets,
                                                         long long* __restrict__ pos) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kNlChunk;
  __shared__ unsigned s_w[kNlThreads / 32];
  long long out = offsets[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = 0; k < 8; ++k) {
    const int64_t off = base + (static_cast<int64_t>(k) * kNlThreads + threadIdx.x) * 16;
    unsigned mask = 0;  // newline bytes of this thread's 16-byte word
    if (off < n) {
      const uint4 v = *reinterpret_cast<const uint4*>(d + off);
      const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (off + q * 4 + b < n && ((w[q] >> (8 * b)) & 0xff) == '\n') mask |= 1u << (q * 4 + b);
    }
    // block-wide exclusive scan of the per-thread counts (thread order = byte order)
    const unsigned c = __popc(mask);
    unsigned x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    unsigned before = 0, total = 0;
    for (int i = 0; i < kNlThreads / 32; ++i) {
      if (i < warp) before += s_w[i];
      total += s_w[i];
    }
    long long p = out + before + x - c;
    while (mask) {
      const int b = __ffs(mask) - 1;
      mask &= mask - 1;
      pos[p++] = off + b;
    }
    out += total;
    __syncthreads();
  }
}

struct CsvSpec {
  const unsigned char* d;  // the whole text (header line first), padded to 16 B
  int64_t n;
  const long long* nl;     // newline positions
  int64_t n_nl;
  int64_t rows;            // data lines parsed
  int ncols;
  unsigned char delim;
  int types[64];
  void* out[64];                  // I64/F64/date: 8 B; bool: 1 B
  long long* str_off[64];         // utf8: start offset per row
  int* str_len[64];               // utf8: length per row
  unsigned* maxlen;               // [ncols]
  unsigned long long* err;        // [0] first error key (min)
  unsigned long long* slow;       // [0] count, then (row << 8 | col) entries
  long long slow_cap;
};

// data line r: after newline r (newline 0 ends the header), up to the next
// newline or the end of the text; one trailing '\r' stripped
__device__ __forceinline__ void line_span(const CsvSpec& s, int64_t r, int64_t& a, int64_t& b) {
  a = s.nl[r] + 1;
  b = r + 1 < s.n_nl ? s.nl[r + 1] : s.n;
  if (b > a && s.d[b - 1] == '\r') --b;  // "\r\n" line ends
}

__device__ __forceinline__ void report(const CsvSpec& s, int64_t row, int field /* -1: field count */) {
  const unsigned long long key = static_cast<unsigned long long>(row) * (s.ncols + 1) + (field + 1);
  atomicMin(s.err, key);
}

__global__ void k_csv_rows(CsvSpec s) {
  for (int64_t r = gtid(); r < s.rows; r += gstride()) {
    int64_t a, b;
    line_span(s, r, a, b);
    // field count first (the reference checks it before parsing any field)
    int nf = 1;
    for (int64_t i = a; i < b; ++i) nf += s.d[i] == s.delim;
    if (nf != s.ncols) {
      report(s, r, -1);
      continue;
    }
    int64_t f0 = a;
    for (int j = 0; j < s.ncols; ++j) {
      int64_t f1 = f0;
      while (f1 < b && s.d[f1] != s.delim) ++f1;
      const unsigned char* p = s.d + f0;
      const int len = static_cast<int>(f1 - f0);
      bool bad = false;
      switch (s.types[j]) {
        case TQP_LT_INT64: {
          int64_t v = 0;
          bad = len == 0 || fp::parse_i64(p, len, v) != 0;
          static_cast<int64_t*>(s.out[j])[r] = v;
          break;
        }
        case TQP_LT_FLOAT64: {
          uint64_t bits = 0;
          fp::Decimal dec;
          const int rc = len == 0 ? 1 : fp::parse_f64_fast(p, len, bits, dec);
          if (rc == 5) {
            const unsigned long long k = atomicAdd(s.slow, 1ULL);
            if (static_cast<long long>(k) < s.slow_cap) s.slow[1 + k] = (static_cast<unsigned long long>(r) << 8) | j;
            else bad = true;  // cannot happen with the capacity sized to rows x float columns
          } else {
            bad = rc != 0;
          }
          static_cast<uint64_t*>(s.out[j])[r] = bits;
          break;
        }
        case TQP_LT_DATE: {
          int64_t ns = 0;
          int y, m, d;
          bad = len == 0 || fp::parse_date(p, len, ns, y, m, d) != 0;
          static_cast<int64_t*>(s.out[j])[r] = ns;
          break;
        }
        case TQP_LT_BOOL: {
          uint8_t v = 0;
          bad = len == 0 || fp::parse_bool(p, len, v) != 0;
          static_cast<uint8_t*>(s.out[j])[r] = v;
          break;
        }
        default: {  // utf8
          bad = len == 0 || !fp::valid_utf8(p, len);
          s.str_off[j][r] = f0;
          s.str_len[j][r] = len;
          if (!bad) atomicMax(s.maxlen + j, static_cast<unsigned>(len));
          break;
        }
      }
      if (bad) {
        report(s, r, j);
        break;  // the reference stops at the first bad field of the row
      }
      f0 = f1 + 1;
    }
  }
}

__global__ void k_csv_slow(CsvSpec s) {
  const long long cnt = static_cast<long long>(*s.slow);
  for (long long i = gtid(); i < cnt && i < s.slow_cap; i += gstride()) {
    const unsigned long long e = s.slow[1 + i];
    const int64_t r = static_cast<int64_t>(e >> 8);
    const int j = static_cast<int>(e & 0xff);
    int64_t a, b;
    line_span(s, r, a, b);
    int64_t f0 = a;
    for (int q = 0; q < j; ++q) {
      while (f0 < b && s.d[f0] != s.delim) ++f0;
      ++f0;
    }
    int64_t f1 = f0;
    while (f1 < b && s.d[f1] != s.delim) ++f1;
    uint64_t bits = 0;
    const int rc = fp::parse_f64(s.d + f0, static_cast<int>(f1 - f0), bits);
    static_cast<uint64_t*>(s.out[j])[r] = bits;
    if (rc != 0) report(s, r, j);
  }
}

__global__ void k_csv_str(const unsigned char* __restrict__ d, const long long* __restrict__ off,
                          const int* __restrict__ len, int64_t rows, int m, uint8_t* __restrict__ out) {
  for (int64_t i = gtid(); i < rows * m; i += gstride()) {
    const int64_t r = i / m;
    const int c = static_cast<int>(i % m);
    out[i] = c < len[r] ? d[off[r] + c] : 0;
  }
}

[[noreturn]] void enc_fail(const std::string& m) { throw Error(TQP_ERR_ENCODING, m); }

// the reference's message for a bad field (CsvColumnBuilder::parse)
std::string field_error(int type, const std::string& f) {
  const unsigned char* p = reinterpret_cast<const unsigned char*>(f.data());
  const int n = static_cast<int>(f.size());
  if (f.empty()) return "empty field (NULLs are not supported)";
  switch (type) {
    case TQP_LT_INT64: return "cannot parse int64 from '" + f + "'";
    case TQP_LT_FLOAT64: return "cannot parse float64 from '" + f + "'";
    case TQP_LT_BOOL: return "cannot parse bool from '" + f + "'";
    case TQP_LT_DATE: {
      int64_t ns;
      int y = 0, m = 0, d = 0;
      const int rc = fp::parse_date(p, n, ns, y, m, d);
      if (rc == 2)
        return "date: invalid calendar date " + std::to_string(y) + "-" + std::to_string(static_cast<unsigned>(m)) + "-" +
               std::to_string(static_cast<unsigned>(d));
      if (rc == 3) return "date: '" + f + "' outside the Int64 nanosecond range";
      return "date: malformed date '" + f + "' (expected YYYY-MM-DD)";
    }
    default: return "invalid UTF-8";
  }
}

}  // namespace

namespace {

std::vector<std::string> split_line(const std::string& line, char delimiter) {
  std::vector<std::string> f;
  for (size_t st = 0;;) {
    const size_t d = line.find(delimiter, st);
    if (d == std::string::npos) {
      f.push_back(line.substr(st));
      break;
    }
    f.push_back(line.substr(st, d - st));
    st = d + 1;
  }
  return f;
}

std::string device_bytes(Ctx& c, const unsigned char* d, int64_t a, int64_t b) {
  std::string out(static_cast<size_t>(std::max<int64_t>(0, b - a)), '\0');
  if (b > a) {
    TQP_CUDA(cudaMemcpyAsync(&out[0], d + a, static_cast<size_t>(b - a), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
  }
  return out;
}

long long device_word(Ctx& c, const long long* p) {
  long long v = 0;
  TQP_CUDA(cudaMemcpyAsync(&v, p, 8, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  return v;
}

}  // namespace

// `d`: the whole CSV text in HBM (16-byte aligned, 32 zero bytes of padding
// after `len`); `head`: the first `head_len` bytes of it on the host (at
// least the header line, or all of a text without a newline).
Table csv_parse_device(Ctx& c, const unsigned char* d, int64_t len, const unsigned char* head, int64_t head_len,
                       const std::vector<std::pair<std::string, int>>& schema, char delimiter, const std::string& origin) {
  if (schema.empty()) enc_fail(origin + ": schema has no columns");
  if (schema.size() > 64) throw Error(TQP_ERR_ARG, "csv: more than 64 columns");
  // ---- header (host: one line)
  if (len <= 0) enc_fail(origin + ": missing header line");
  const void* nlp = std::memchr(head, '\n', static_cast<size_t>(head_len));
  const int64_t hend = nlp ? static_cast<const unsigned char*>(nlp) - head : head_len;
  std::string header(reinterpret_cast<const char*>(head), static_cast<size_t>(hend));
  if (!header.empty() && header.back() == '\r') header.pop_back();
  const std::vector<std::string> hf = split_line(header, delimiter);
  const int ncols = static_cast<int>(schema.size());
  if (static_cast<int>(hf.size()) != ncols)
    enc_fail(origin + ":1: header has " + std::to_string(hf.size()) + " columns, schema has " + std::to_string(ncols));
  for (int i = 0; i < ncols; ++i)
    if (!iequals(hf[i], schema[i].first))
      enc_fail(origin + ":1: header column " + std::to_string(i + 1) + " is '" + hf[i] + "', schema expects '" +
               schema[i].first + "'");

  // ---- newline positions over the whole text (newline 0 ends the header)
  const int64_t dn = len;
  const int64_t nchunks = (dn + kNlChunk - 1) / kNlChunk;
  Tensor counts = c.alloc(TQP_I64, std::max<int64_t>(1, nchunks), 1);
  int64_t n_nl = 0;
  Tensor pos = c.alloc(TQP_I64, 1, 1);
  if (nlp) {
    k_nl_count<<<static_cast<unsigned>(nchunks), kNlThreads, 0, c.stream>>>(d, dn, counts.ptr<long long>());
    c.count_launch();
    Tensor cc = counts;
    cc.rows = nchunks;
    Tensor offs = k::prefix_sum_exclusive(c, cc);
    long long last[2] = {0, 0};
    TQP_CUDA(cudaMemcpyAsync(&last[0], offs.ptr<long long>() + nchunks - 1, 8, cudaMemcpyDeviceToHost, c.stream));
    TQP_CUDA(cudaMemcpyAsync(&last[1], counts.ptr<long long>() + nchunks - 1, 8, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    n_nl = last[0] + last[1];
    pos = c.alloc(TQP_I64, std::max<int64_t>(1, n_nl), 1);
    k_nl_write<<<static_cast<unsigned>(nchunks), kNlThreads, 0, c.stream>>>(d, dn, offs.ptr<long long>(),
                                                                            pos.ptr<long long>());
    c.count_launch();
  }
  // data lines: one after each newline, except after a final newline at the
  // end of the text; the last one is dropped when it is empty ("trailing
  // newline", columnar.cpp:504)
  int64_t rows = 0;
  if (n_nl) {
    const long long lastnl = device_word(c, pos.ptr<long long>() + n_nl - 1);
    rows = n_nl - 1 + (dn > lastnl + 1 ? 1 : 0);
    if (rows) {
      const long long a = device_word(c, pos.ptr<long long>() + rows - 1) + 1;
      const long long b = rows < n_nl ? device_word(c, pos.ptr<long long>() + rows) : dn;
      const std::string tail = device_bytes(c, d, std::max<long long>(a, b - 1), b);
      int64_t sl = b - a;
      if (sl > 0 && tail.back() == '\r') --sl;
      if (sl == 0) --rows;
    }
  }

  // ---- parse
  CsvSpec s{};
  s.d = d;
  s.n = dn;
  s.nl = pos.ptr<long long>();
  s.n_nl = n_nl;
  s.rows = rows;
  s.ncols = ncols;
  s.delim = static_cast<unsigned char>(delimiter);
  std::vector<Tensor> outs(ncols);
  std::vector<Tensor> soff(ncols), slen(ncols);
  int nfloat = 0;
  for (int j = 0; j < ncols; ++j) {
    const int lt = schema[j].second;
    s.types[j] = lt;
    if (lt == TQP_LT_UTF8) {
      soff[j] = c.alloc(TQP_I64, std::max<int64_t>(1, rows), 1);
      slen[j] = c.alloc(TQP_I32, std::max<int64_t>(1, rows), 1);
      s.str_off[j] = soff[j].ptr<long long>();
      s.str_len[j] = slen[j].ptr<int>();
    } else {
      outs[j] = c.alloc(physical_dtype(lt), rows, 1);
      s.out[j] = outs[j].data();
      nfloat += lt == TQP_LT_FLOAT64;
    }
  }
  auto aux = c.alloc_bytes(sizeof(unsigned long long) * 2 + sizeof(unsigned) * 64);
  s.err = static_cast<unsigned long long*>(aux->ptr);
  s.maxlen = reinterpret_cast<unsigned*>(s.err + 2);
  TQP_CUDA(cudaMemsetAsync(s.err, 0xff, 8, c.stream));
  TQP_CUDA(cudaMemsetAsync(s.maxlen, 0, sizeof(unsigned) * 64, c.stream));
  s.slow_cap = std::max<long long>(1, rows * nfloat);
  auto slow = c.alloc_bytes(sizeof(unsigned long long) * (s.slow_cap + 1));
  s.slow = static_cast<unsigned long long*>(slow->ptr);
  TQP_CUDA(cudaMemsetAsync(s.slow, 0, 8, c.stream));
  if (rows) {
    k_csv_rows<<<c.grid_for(rows, 256, 1, 32), 256, 0, c.stream>>>(s);
    k_csv_slow<<<c.num_sms, 128, 0, c.stream>>>(s);
    c.count_launch(2);
  }
  unsigned long long hdr[2 + 32];
  TQP_CUDA(cudaMemcpyAsync(hdr, s.err, sizeof(hdr), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  if (hdr[0] != ~0ULL) {
    const int64_t r = static_cast<int64_t>(hdr[0] / (ncols + 1));
    const int field = static_cast<int>(hdr[0] % (ncols + 1)) - 1;
    const long long a = device_word(c, pos.ptr<long long>() + r) + 1;
    const long long b = r + 1 < n_nl ? device_word(c, pos.ptr<long long>() + r + 1) : dn;
    std::string line = device_bytes(c, d, a, b);
    if (!line.empty() && line.back() == '\r') line.pop_back();
    const std::string where = origin + ":" + std::to_string(r + 2) + ": ";
    const std::vector<std::string> f = split_line(line, delimiter);
    if (field < 0) enc_fail(where + "expected " + std::to_string(ncols) + " fields, got " + std::to_string(f.size()));
    enc_fail(where + "column '" + schema[field].first + "' (field " + std::to_string(field + 1) +
             "): " + field_error(schema[field].second, f[field]));
  }
  // ---- strings
  Table t;
  t.rows = rows;
  for (int j = 0; j < ncols; ++j) {
    if (schema[j].second == TQP_LT_UTF8) {
      const int mm = std::max(1, static_cast<int>(reinterpret_cast<const unsigned*>(hdr + 2)[j]));
      outs[j] = c.alloc(TQP_STR8, rows, mm);
      if (rows) {
        k_csv_str<<<c.grid_for(rows * mm, 256, 4, 16), 256, 0, c.stream>>>(d, soff[j].ptr<long long>(), slen[j].ptr<int>(),
                                                                          rows, mm, outs[j].ptr<uint8_t>());
        c.count_launch();
      }
    }
    t.cols.push_back({schema[j].first, schema[j].second, outs[j]});
  }
  c.sync();  // the host text may be released by the caller
  return t;
}

Table csv_parse(Ctx& c, const unsigned char* text, int64_t len, const std::vector<std::pair<std::string, int>>& schema,
                char delimiter, const std::string& origin) {
  auto dbuf = c.alloc_bytes(static_cast<size_t>(std::max<int64_t>(0, len)) + 32);
  unsigned char* d = static_cast<unsigned char*>(dbuf->ptr);
  if (len > 0) TQP_CUDA(cudaMemcpyAsync(d, text, static_cast<size_t>(len), cudaMemcpyHostToDevice, c.stream));
  TQP_CUDA(cudaMemsetAsync(d + std::max<int64_t>(0, len), 0, 32, c.stream));
  return csv_parse_device(c, d, len, text, len, schema, delimiter, origin);
}

// load_csv: the file streams through a small ring of pinned buffers straight
// into one device buffer (reads overlap the copies; no pinned allocation of
// the file's size), then the device parse
Table csv_load(Ctx& c, const std::string& path, const std::vector<std::pair<std::string, int>>& schema, char delimiter) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) enc_fail("csv: cannot open '" + path + "'");
  const int64_t n = static_cast<int64_t>(in.tellg());
  in.seekg(0);
  constexpr int kRing = 4;
  constexpr int64_t kChunk = 16 << 20;
  if (!c.csv_ring) {
    TQP_CUDA(cudaMallocHost(&c.csv_ring, static_cast<size_t>(kRing * kChunk)));
    for (int i = 0; i < kRing; ++i) TQP_CUDA(cudaEventCreateWithFlags(&c.csv_ring_ev[i], cudaEventDisableTiming));
  }
  auto dbuf = c.alloc_bytes(static_cast<size_t>(n) + 32);
  unsigned char* d = static_cast<unsigned char*>(dbuf->ptr);
  std::string head;
  bool have_nl = false;
  for (int64_t off = 0, k = 0; off < n; off += kChunk, ++k) {
    const int slot = static_cast<int>(k % kRing);
    unsigned char* buf = c.csv_ring + slot * kChunk;
    if (k >= kRing) TQP_CUDA(cudaEventSynchronize(c.csv_ring_ev[slot]));  // its previous copy is done
    const int64_t m = std::min<int64_t>(kChunk, n - off);
    if (!in.read(reinterpret_cast<char*>(buf), m)) enc_fail("csv: cannot read '" + path + "'");
    if (!have_nl) {  // the header line stays on the host
      const void* p = std::memchr(buf, '\n', static_cast<size_t>(m));
      const int64_t take = p ? static_cast<const unsigned char*>(p) - buf + 1 : m;
      head.append(reinterpret_cast<const char*>(buf), static_cast<size_t>(take));
      have_nl = p != nullptr;
    }
    TQP_CUDA(cudaMemcpyAsync(d + off, buf, static_cast<size_t>(m), cudaMemcpyHostToDevice, c.stream));
    TQP_CUDA(cudaEventRecord(c.csv_ring_ev[slot], c.stream));
  }
  TQP_CUDA(cudaMemsetAsync(d + n, 0, 32, c.stream));
  return csv_parse_device(c, d, n, reinterpret_cast<const unsigned char*>(head.data()),
                          static_cast<int64_t>(head.size()), schema, delimiter, path);
}

}  // namespace tqp
