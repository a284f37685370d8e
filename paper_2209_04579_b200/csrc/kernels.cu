// Elementwise / row-wise kernels of the kernel set (kernels.hpp:28-78) and
// the executor plumbing ops (executor.cpp:110-278), as sm_100a grid-stride
// kernels. Each host wrapper reproduces the reference's shape/dtype contract
// and error text; fallible kernels report the first offending element through
// an atomicMin flag (FirstBadIndex, kernels.cpp:31-45), so the reported row
// does not depend on scheduling.
#include <algorithm>
#include <cmath>
#include <string>

#include "device.cuh"

namespace tqp {
namespace {

constexpr int kBlock = 256;

// ---- broadcast shape (kernels.cpp:46-88) ------------------------------------
struct Bcast {
  int64_t rows, cols;
  bool a_scalar, a_row, b_scalar, b_row;
};

bool broadcastable_into(const Tensor& s, int64_t rows, int64_t cols) {
  if (s.rows == rows && s.cols == cols) return true;
  return s.rows == 1 && (s.cols == 1 || s.cols == cols);
}

std::string shape_str(const Tensor& t) { return std::to_string(t.rows) + "x" + std::to_string(t.cols); }

Bcast broadcast_shape(const char* kernel, const Tensor& a, const Tensor& b) {
  Bcast s{};
  if (a.same_shape(b) || broadcastable_into(b, a.rows, a.cols)) {
    s.rows = a.rows;
    s.cols = a.cols;
  } else if (broadcastable_into(a, b.rows, b.cols)) {
    s.rows = b.rows;
    s.cols = b.cols;
  } else {
    kernel_fail(std::string(kernel) + ": shape mismatch (" + shape_str(a) + " vs " + shape_str(b) + ")");
  }
  auto classify = [&](const Tensor& t, bool& scalar, bool& row) {
    scalar = t.is_scalar() && !(s.rows == 1 && s.cols == 1);
    row = !t.is_scalar() && t.rows == 1 && s.rows > 1 && t.cols == s.cols;
    if (!scalar && !row && (t.rows != s.rows || t.cols != s.cols)) {
      kernel_fail(std::string(kernel) + ": shape mismatch");
    }
  };
  classify(a, s.a_scalar, s.a_row);
  classify(b, s.b_scalar, s.b_row);
  return s;
}

void require_same_dtype(const char* kernel, const Tensor& a, const Tensor& b) {
  int da = a.dtype == TQP_STR8 ? TQP_I32 : a.dtype, db = b.dtype == TQP_STR8 ? TQP_I32 : b.dtype;
  if (da != db || (a.dtype == TQP_STR8) != (b.dtype == TQP_STR8)) {
    if (da == db) kernel_fail(std::string(kernel) + ": mixed string and int32 operands");
    kernel_fail(std::string(kernel) + ": dtype mismatch (" + dtype_name(a.dtype) + " vs " + dtype_name(b.dtype) + ")");
  }
}
void require_vector(const char* kernel, const Tensor& t) {
  if (!t.is_vector()) kernel_fail(std::string(kernel) + ": expected a vector (m=1)");
}
void require_dtype(const char* kernel, const Tensor& t, int want) {
  if (t.dtype != want) {
    kernel_fail(std::string(kernel) + ": expected " + dtype_name(want) + ", got " + dtype_name(t.dtype));
  }
}

__device__ __forceinline__ int64_t bidx(int64_t flat, int64_t cols, bool scalar, bool row) {
  return scalar ? 0 : (row ? flat % cols : flat);
}

template <typename T, typename Out, typename F>
__global__ void k_binary(const T* __restrict__ a, const T* __restrict__ b, Out* __restrict__ out, int64_t n,
                         int64_t cols, bool as, bool ar, bool bs, bool br, F f, long long* err) {
  for (int64_t i = gtid(); i < n; i += gstride()) {
    out[i] = f(a[bidx(i, cols, as, ar)], b[bidx(i, cols, bs, br)], i, err);
  }
}

// no row broadcast: four independent rows per thread per
// step, every load issued before the first use (the one-row grid-stride
// loop above kept two loads in flight per thread: 0.76 of HBM for fp64 ops)
// (a scalar operand, as / bs, is read once)
template <typename T, typename Out, typename F>
__global__ void k_binary4(const T* __restrict__ a, const T* __restrict__ b, Out* __restrict__ out, int64_t n, bool as,
                          bool bs, F f, long long* err) {
  const int64_t st = gstride();
  const T a0 = as ? a[0] : T{}, b0 = bs ? b[0] : T{};
  for (int64_t i0 = gtid(); i0 < n; i0 += 4 * st) {
    T x[4], y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * st;
      if (i < n) {
        x[u] = as ? a0 : a[i];
        y[u] = bs ? b0 : b[i];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * st;
      if (i < n) out[i] = f(x[u], y[u], i, err);
    }
  }
}

template <typename T, typename Out, typename F>
Tensor binary(Ctx& c, const char* kernel, const Tensor& a, const Tensor& b, int out_dtype, F f, Bcast* shape = nullptr,
              long long* err = nullptr) {
  Bcast s = broadcast_shape(kernel, a, b);
  if (shape) *shape = s;
  Tensor o = c.alloc(out_dtype, s.rows, s.cols);
  int64_t n = s.rows * s.cols;
  if (n && !s.a_row && !s.b_row) {
    k_binary4<T, Out><<<c.grid_for(n, kBlock, 4), kBlock, 0, c.stream>>>(a.ptr<T>(), b.ptr<T>(), o.ptr<Out>(), n,
                                                                        s.a_scalar, s.b_scalar, f, err ? err : c.d_err);
    c.count_launch();
  } else if (n) {
    k_binary<T, Out><<<c.grid_for(n, kBlock), kBlock, 0, c.stream>>>(
        a.ptr<T>(), b.ptr<T>(), o.ptr<Out>(), n, s.cols, s.a_scalar, s.a_row, s.b_scalar, s.b_row, f,
        err ? err : c.d_err);
    c.count_launch();
  }
  return o;
}

struct CmpF {
  int op;
  template <typename T>
  __device__ uint8_t operator()(T x, T y, int64_t, long long*) const {
    switch (op) {
      case TQP_EQ: return x == y;
      case TQP_NE: return x != y;
      case TQP_LT: return x < y;
      case TQP_LE: return x <= y;
      case TQP_GT: return x > y;
      default: return x >= y;
    }
  }
};

struct ArithF64 {
  int op;
  __device__ double operator()(double x, double y, int64_t i, long long* err) const {
    switch (op) {
      case TQP_ADD: return __dadd_rn(x, y);
      case TQP_SUB: return __dsub_rn(x, y);
      case TQP_MUL: return __dmul_rn(x, y);
      default:
        if (y == 0.0) {
          note_bad(err, i);
          return 0.0;
        }
        return __ddiv_rn(x, y);
    }
  }
};

template <typename T>
struct ArithInt {
  int op;
  __device__ T operator()(T x, T y, int64_t i, long long* err) const {
    T r;
    bool ovf = op == TQP_ADD ? add_ovf(x, y, &r) : op == TQP_SUB ? sub_ovf(x, y, &r) : mul_ovf(x, y, &r);
    if (ovf) note_bad(err, i);
    return r;
  }
};

struct LogicF {
  int op;
  __device__ uint8_t operator()(uint8_t x, uint8_t y, int64_t, long long*) const {
    return op == TQP_AND ? (x && y) : (x || y);
  }
};

__global__ void k_not(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int64_t n) {
  for (int64_t i = gtid(); i < n; i += gstride()) out[i] = in[i] ? 0 : 1;
}

template <typename T>
__global__ void k_select(const uint8_t* __restrict__ cond, const T* __restrict__ a, const T* __restrict__ b,
                         T* __restrict__ out, int64_t rows, int64_t cols, int64_t cr, int64_t cc, int64_t ar,
                         int64_t ac, int64_t br, int64_t bc) {
  int64_t n = rows * cols;
  for (int64_t i = gtid(); i < n; i += gstride()) {
    int64_t r = i / cols, c = i % cols;
    bool sel = cond[(cr == 1 ? 0 : r) * cc + (cc == 1 ? 0 : c)] != 0;
    out[i] = sel ? a[(ar == 1 ? 0 : r) * ac + (ac == 1 ? 0 : c)] : b[(br == 1 ? 0 : r) * bc + (bc == 1 ? 0 : c)];
  }
}

template <typename From, typename To>
__global__ void k_cast(const From* __restrict__ in, To* __restrict__ out, int64_t n) {
  for (int64_t i = gtid(); i < n; i += gstride()) {
    if constexpr (std::is_same_v<To, uint8_t>) {
      out[i] = in[i] != From{} ? 1 : 0;
    } else {
      out[i] = static_cast<To>(in[i]);
    }
  }
}

__global__ void k_exp(const double* __restrict__ in, double* __restrict__ out, int64_t n) {
  for (int64_t i = gtid(); i < n; i += gstride()) out[i] = exp(in[i]);
}

__global__ void k_iota(int64_t* __restrict__ out, int64_t n) {
  for (int64_t i = gtid(); i < n; i += gstride()) out[i] = i;
}

template <typename T>
__global__ void k_bcast_rows(const T* __restrict__ v, T* __restrict__ out, int64_t n, int64_t m) {
  for (int64_t i = gtid(); i < n * m; i += gstride()) out[i] = v[i % m];
}

template <typename T>
__global__ void k_pad(const T* __restrict__ in, T* __restrict__ out, int64_t n, int64_t m, int64_t target) {
  for (int64_t i = gtid(); i < n * target; i += gstride()) {
    int64_t r = i / target, c = i % target;
    out[i] = c < m ? in[r * m + c] : T{0};
  }
}

__global__ void k_pack(const double* const* __restrict__ cols, double* __restrict__ out, int64_t n, int k) {
  for (int64_t i = gtid(); i < n * k; i += gstride()) out[i] = cols[i % k][i / k];
}

template <typename T>
__global__ void k_gather(const T* __restrict__ v, const int64_t* __restrict__ idx, T* __restrict__ out, int64_t k,
                         int64_t m, int64_t n, long long* err) {
  for (int64_t i = gtid(); i < k * m; i += gstride()) {
    int64_t r = i / m, c = i - r * m;
    int64_t j = idx[r];
    if (j < 0 || j >= n) {
      note_bad(err, r);
      continue;
    }
    out[i] = v[j * m + c];
  }
}

// vector fast path: one element per row
template <typename T>
__global__ void k_gather_vec(const T* __restrict__ v, const int64_t* __restrict__ idx, T* __restrict__ out, int64_t k,
                             int64_t n, long long* err) {
  for (int64_t i = gtid(); i < k; i += gstride()) {
    int64_t j = idx[i];
    if (j < 0 || j >= n) {
      note_bad(err, i);
      continue;
    }
    out[i] = __ldg(v + j);
  }
}

template <typename T>
__global__ void k_segment_starts(const T* __restrict__ kv, uint8_t* __restrict__ out, int64_t n, int64_t m) {
  for (int64_t i = gtid(); i < n; i += gstride()) {
    if (i == 0) {
      out[0] = 1;
      continue;
    }
    bool differs = false;
    for (int64_t j = 0; j < m && !differs; ++j) differs = kv[i * m + j] != kv[(i - 1) * m + j];
    out[i] = differs;
  }
}

// One-column keys: 16 flags per thread per step (one 16-byte store, the keys
// read as whole vectors for 1-byte keys), the previous key from the row before
// the run. Byte-at-a-time flags ran at 0.09 of HBM bandwidth on Q1's
// per-instruction group keys.
template <typename T>
__global__ void k_segment_starts1(const T* __restrict__ kv, uint8_t* __restrict__ out, int64_t n) {
  const int64_t nv = n / 16;
  for (int64_t t = gtid(); t < nv; t += gstride()) {
    const int64_t i0 = t * 16;
    T cur[16];
    if constexpr (sizeof(T) == 1) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(kv) + t);
      const unsigned wd[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int j = 0; j < 16; ++j) cur[j] = static_cast<T>((wd[j >> 2] >> (8 * (j & 3))) & 0xffu);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) cur[j] = __ldg(kv + i0 + j);
    }
    const T prev = i0 ? __ldg(kv + i0 - 1) : cur[0];
    unsigned o[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const bool d = j ? cur[j] != cur[j - 1] : (i0 == 0 || cur[0] != prev);
      o[j >> 2] |= static_cast<unsigned>(d) << (8 * (j & 3));
    }
    reinterpret_cast<uint4*>(out)[t] = make_uint4(o[0], o[1], o[2], o[3]);
  }
  for (int64_t i = nv * 16 + gtid(); i < n; i += gstride()) out[i] = i == 0 || kv[i] != kv[i - 1];
}

// String rows: either STR8 (bytes) or Int32 per byte (reference layout).
template <typename T>
__global__ void k_substring(const T* __restrict__ cv, uint8_t* __restrict__ out, int64_t n, int64_t m,
                            const uint8_t* __restrict__ pat, int64_t plen, int anchor) {
  for (int64_t i = gtid(); i < n; i += gstride()) {
    const T* row = cv + i * m;
    int64_t len = 0;
    while (len < m && row[len] != 0) ++len;
    auto match_at = [&](int64_t off) {
      for (int64_t j = 0; j < plen; ++j)
        if (static_cast<int32_t>(row[off + j]) != static_cast<int32_t>(pat[j])) return false;
      return true;
    };
    bool ok = false;
    if (plen <= len) {
      switch (anchor) {
        case TQP_START: ok = match_at(0); break;
        case TQP_END: ok = match_at(len - plen); break;
        case TQP_ANY:
          for (int64_t o = 0; o + plen <= len && !ok; ++o) ok = match_at(o);
          break;
        default: ok = len == plen && match_at(0); break;
      }
    }
    out[i] = ok;
  }
}

template <typename TA, typename TB>
__global__ void k_strcmp(const TA* __restrict__ a, const TB* __restrict__ b, uint8_t* __restrict__ out, int64_t rows,
                         int64_t arows, int64_t acols, int64_t brows, int64_t bcols, int op) {
  int64_t m = acols > bcols ? acols : bcols;
  for (int64_t i = gtid(); i < rows; i += gstride()) {
    int64_t ra = arows == 1 ? 0 : i, rb = brows == 1 ? 0 : i;
    int cmp = 0;
    for (int64_t j = 0; j < m && cmp == 0; ++j) {
      int32_t x = j < acols ? static_cast<int32_t>(a[ra * acols + j]) : 0;
      int32_t y = j < bcols ? static_cast<int32_t>(b[rb * bcols + j]) : 0;
      if (x != y) cmp = x < y ? -1 : 1;
    }
    bool r;
    switch (op) {
      case TQP_EQ: r = cmp == 0; break;
      case TQP_NE: r = cmp != 0; break;
      case TQP_LT: r = cmp < 0; break;
      case TQP_LE: r = cmp <= 0; break;
      case TQP_GT: r = cmp > 0; break;
      default: r = cmp >= 0; break;
    }
    out[i] = r;
  }
}

// fp64 GEMM for PREDICT (kernels.cpp:674-690) on the FP64 tensor cores
// (DMMA: mma.sync m8n8k4 f64). A block computes a 64 x 64 tile of C with 4
// warps (2 x 2, 32 x 32 each = 4 x 4 fragments); K is staged 16 wide in
// shared memory. The Hummingbird tree GEMMs (X.A with a one-hot feature
// selector, S.C and hit.leaf_index with small-integer operands) are exact on
// it (every product and partial sum is representable); dense linear models
// differ from Eigen's summation order within the fp64 tolerance.
constexpr int kMmBM = 64, kMmBN = 64, kMmBK = 16;
__global__ void __launch_bounds__(128) k_matmul(const double* __restrict__ A, const double* __restrict__ B,
                                                double* __restrict__ C, int64_t n, int64_t kk, int64_t p) {
  __shared__ double As[kMmBM][kMmBK + 1];
  __shared__ double Bs[kMmBK][kMmBN + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const int64_t bm = static_cast<int64_t>(blockIdx.x) * kMmBM, bn = static_cast<int64_t>(blockIdx.y) * kMmBN;  // rows on x (2^31 blocks)
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int64_t k0 = 0; k0 < kk; k0 += kMmBK) {
    for (int e = threadIdx.x; e < kMmBM * kMmBK; e += 128) {
      const int r = e / kMmBK, q = e % kMmBK;
      As[r][q] = (bm + r < n && k0 + q < kk) ? A[(bm + r) * kk + k0 + q] : 0.0;
    }
    for (int e = threadIdx.x; e < kMmBK * kMmBN; e += 128) {
      const int q = e / kMmBN, col = e % kMmBN;
      Bs[q][col] = (k0 + q < kk && bn + col < p) ? B[(k0 + q) * p + bn + col] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < kMmBK; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[wm * 32 + i * 8 + (lane >> 2)][ks + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[ks + (lane & 3)][wn * 32 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
                       : "d"(af[i]), "d"(bf[j]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = bm + wm * 32 + i * 8 + (lane >> 2);
    if (row >= n) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t col = bn + wn * 32 + j * 8 + (lane & 3) * 2;
      if (col < p) C[row * p + col] = acc[i][j][0];
      if (col + 1 < p) C[row * p + col + 1] = acc[i][j][1];
    }
  }
}

int string_like(const Tensor& t) { return t.dtype == TQP_STR8 || t.dtype == TQP_I32; }

}  // namespace

namespace k {

Tensor compare(Ctx& c, const Tensor& a, const Tensor& b, int op) {
  require_same_dtype("compare", a, b);
  Tensor out;
  TQP_DISPATCH(a.dtype, T, out = binary<T, uint8_t>(c, "compare", a, b, TQP_BOOL, CmpF{op}));
  return out;
}

Tensor arith(Ctx& c, const Tensor& a, const Tensor& b, int op) {
  require_same_dtype("arith", a, b);
  if (a.dtype == TQP_BOOL || a.dtype == TQP_STR8) kernel_fail("arith: bool operands not supported");
  if (op == TQP_DIV && a.dtype != TQP_F64) kernel_fail("arith: div requires float64 operands");
  if (op < TQP_ADD || op > TQP_DIV) kernel_fail("arith: bad op");
  Bcast s;
  Tensor out;
  if (a.dtype == TQP_F64) {
    if (op != TQP_DIV) return binary<double, double>(c, "arith", a, b, TQP_F64, ArithF64{op}, &s);
    bool dfr = false;
    long long* err = c.check_slot(&dfr);
    out = binary<double, double>(c, "arith", a, b, TQP_F64, ArithF64{op}, &s, err);
    const char* msg = "arith: division by zero at row ";
    if (dfr) {
      c.deferred.push_back({msg, s.cols});
    } else {
      int64_t bad = c.read_err();
      if (bad >= 0) kernel_fail(msg + std::to_string(bad / s.cols), bad / s.cols);
    }
    return out;
  }
  bool dfr = false;
  long long* err = c.check_slot(&dfr);
  if (a.dtype == TQP_I64) {
    out = binary<int64_t, int64_t>(c, "arith", a, b, TQP_I64, ArithInt<int64_t>{op}, &s, err);
  } else {
    out = binary<int32_t, int32_t>(c, "arith", a, b, TQP_I32, ArithInt<int32_t>{op}, &s, err);
  }
  const char* msg = "arith: integer overflow at row ";
  if (dfr) {
    c.deferred.push_back({msg, s.cols});
  } else {
    int64_t bad = c.read_err();
    if (bad >= 0) kernel_fail(msg + std::to_string(bad / s.cols), bad / s.cols);
  }
  return out;
}

Tensor logical(Ctx& c, const Tensor& a, const Tensor& b, int op) {
  require_dtype("logical", a, TQP_BOOL);
  require_dtype("logical", b, TQP_BOOL);
  return binary<uint8_t, uint8_t>(c, "logical", a, b, TQP_BOOL, LogicF{op});
}

Tensor logical_not(Ctx& c, const Tensor& v) {
  require_dtype("not", v, TQP_BOOL);
  Tensor o = c.alloc(TQP_BOOL, v.rows, v.cols);
  if (v.size()) {
    k_not<<<c.grid_for(v.size(), kBlock), kBlock, 0, c.stream>>>(v.ptr<uint8_t>(), o.ptr<uint8_t>(), v.size());
    c.count_launch();
  }
  return o;
}

Tensor select_where(Ctx& c, const Tensor& cond, const Tensor& a, const Tensor& b) {
  require_dtype("select_where", cond, TQP_BOOL);
  require_same_dtype("select_where", a, b);
  int64_t rows = std::max({cond.rows, a.rows, b.rows});
  int64_t cols = std::max({cond.cols, a.cols, b.cols});
  auto check = [&](const Tensor& x) {
    if ((x.rows != 1 && x.rows != rows) || (x.cols != 1 && x.cols != cols)) {
      kernel_fail("select_where: shape " + shape_str(x) + " does not broadcast to " + std::to_string(rows) + "x" +
                  std::to_string(cols));
    }
  };
  check(cond);
  check(a);
  check(b);
  Tensor o = c.alloc(a.dtype, rows, cols);
  if (rows * cols) {
    TQP_DISPATCH(a.dtype, T,
                 k_select<T><<<c.grid_for(rows * cols, kBlock), kBlock, 0, c.stream>>>(
                     cond.ptr<uint8_t>(), a.ptr<T>(), b.ptr<T>(), o.ptr<T>(), rows, cols, cond.rows, cond.cols,
                     a.rows, a.cols, b.rows, b.cols));
    c.count_launch();
  }
  return o;
}

Tensor gather(Ctx& c, const Tensor& values, const Tensor& idx) {
  require_dtype("gather", idx, TQP_I64);
  require_vector("gather", idx);
  int64_t n = values.rows, m = values.cols, kk = idx.rows;
  Tensor o = c.alloc(values.dtype, kk, m);
  if (kk * m == 0) return o;
  c.reset_err();
  TQP_DISPATCH(values.dtype, T, {
    if (m == 1) {
      k_gather_vec<T><<<c.grid_for(kk, kBlock), kBlock, 0, c.stream>>>(values.ptr<T>(), idx.ptr<int64_t>(),
                                                                         o.ptr<T>(), kk, n, c.d_err);
    } else {
      k_gather<T><<<c.grid_for(kk * m, kBlock), kBlock, 0, c.stream>>>(values.ptr<T>(), idx.ptr<int64_t>(),
                                                                         o.ptr<T>(), kk, m, n, c.d_err);
    }
  });
  c.count_launch();
  int64_t bad = c.read_err();
  if (bad >= 0) {
    int64_t v = read_scalar<int64_t>(c, idx, bad);
    kernel_fail("gather: index " + std::to_string(v) + " at position " + std::to_string(bad) +
                    " out of bounds [0," + std::to_string(n) + ")",
                bad);
  }
  return o;
}

Tensor segment_starts(Ctx& c, const Tensor& kv) {
  Tensor o = c.alloc(TQP_BOOL, kv.rows, 1);
  if (kv.rows) {
    if (kv.cols == 1) {
      TQP_DISPATCH(kv.dtype, T,
                   k_segment_starts1<T><<<c.grid_for(kv.rows, kBlock, 16), kBlock, 0, c.stream>>>(
                       kv.ptr<T>(), o.ptr<uint8_t>(), kv.rows));
    } else {
      TQP_DISPATCH(kv.dtype, T,
                   k_segment_starts<T><<<c.grid_for(kv.rows, kBlock), kBlock, 0, c.stream>>>(kv.ptr<T>(), o.ptr<uint8_t>(),
                                                                                             kv.rows, kv.cols));
    }
    c.count_launch();
  }
  return o;
}

Tensor matmul(Ctx& c, const Tensor& a, const Tensor& b) {
  require_dtype("matmul", a, TQP_F64);
  require_dtype("matmul", b, TQP_F64);
  if (a.cols != b.rows) {
    kernel_fail("matmul: inner dimensions differ (" + std::to_string(a.cols) + " vs " + std::to_string(b.rows) + ")");
  }
  Tensor o = c.alloc(TQP_F64, a.rows, b.cols);
  if (a.rows && b.cols) {
    dim3 grid(static_cast<unsigned>((a.rows + kMmBM - 1) / kMmBM), static_cast<unsigned>((b.cols + kMmBN - 1) / kMmBN));
    k_matmul<<<grid, 128, 0, c.stream>>>(a.ptr<double>(), b.ptr<double>(), o.ptr<double>(), a.rows, a.cols, b.cols);
    c.count_launch();
  }
  return o;
}

Tensor substring_match(Ctx& c, const Tensor& chars, const std::string& pattern, int anchor) {
  if (!string_like(chars)) require_dtype("substring_match", chars, TQP_I32);
  Tensor o = c.alloc(TQP_BOOL, chars.rows, 1);
  if (!chars.rows) return o;
  auto pat = c.alloc_bytes(pattern.size() + 1);
  TQP_CUDA(cudaMemcpyAsync(pat->ptr, pattern.data(), pattern.size() + 1, cudaMemcpyHostToDevice, c.stream));
  int g = c.grid_for(chars.rows, kBlock);
  if (chars.dtype == TQP_STR8) {
    k_substring<uint8_t><<<g, kBlock, 0, c.stream>>>(chars.ptr<uint8_t>(), o.ptr<uint8_t>(), chars.rows, chars.cols,
                                                     static_cast<uint8_t*>(pat->ptr), (int64_t)pattern.size(), anchor);
  } else {
    k_substring<int32_t><<<g, kBlock, 0, c.stream>>>(chars.ptr<int32_t>(), o.ptr<uint8_t>(), chars.rows, chars.cols,
                                                     static_cast<uint8_t*>(pat->ptr), (int64_t)pattern.size(), anchor);
  }
  c.count_launch();
  return o;
}

Tensor iota(Ctx& c, int64_t n) {
  if (n < 0) exec_fail("iota: negative length");
  Tensor o = c.alloc(TQP_I64, n, 1);
  if (n) {
    k_iota<<<c.grid_for(n, kBlock), kBlock, 0, c.stream>>>(o.ptr<int64_t>(), n);
    c.count_launch();
  }
  return o;
}

Tensor cast(Ctx& c, const Tensor& t, int to) {
  int from = t.dtype == TQP_STR8 ? TQP_I32 : t.dtype;
  if (from == to && t.dtype != TQP_STR8) return t;
  Tensor o = c.alloc(to, t.rows, t.cols);
  int64_t n = t.size();
  if (!n) return o;
  int g = c.grid_for(n, kBlock);
  auto launch_to = [&](auto in_tag) {
    using From = decltype(in_tag);
    const From* in = static_cast<const From*>(t.data());
    switch (to) {
      case TQP_BOOL: k_cast<From, uint8_t><<<g, kBlock, 0, c.stream>>>(in, o.ptr<uint8_t>(), n); break;
      case TQP_I32: k_cast<From, int32_t><<<g, kBlock, 0, c.stream>>>(in, o.ptr<int32_t>(), n); break;
      case TQP_I64: k_cast<From, int64_t><<<g, kBlock, 0, c.stream>>>(in, o.ptr<int64_t>(), n); break;
      case TQP_F64: k_cast<From, double><<<g, kBlock, 0, c.stream>>>(in, o.ptr<double>(), n); break;
      default: exec_fail("cast: bad target");
    }
  };
  switch (t.dtype) {
    case TQP_BOOL:
    case TQP_STR8: launch_to(uint8_t{}); break;
    case TQP_I32: launch_to(int32_t{}); break;
    case TQP_I64: launch_to(int64_t{}); break;
    case TQP_F64: launch_to(double{}); break;
    default: exec_fail("cast: bad source");
  }
  c.count_launch();
  return o;
}

Tensor exp_f64(Ctx& c, const Tensor& t) {
  Tensor o = c.alloc(TQP_F64, t.rows, t.cols);
  if (t.size()) {
    k_exp<<<c.grid_for(t.size(), kBlock), kBlock, 0, c.stream>>>(t.ptr<double>(), o.ptr<double>(), t.size());
    c.count_launch();
  }
  return o;
}

Tensor last_or_zero(Ctx& c, const Tensor& t) {
  check_i64_access(t);  // executor.cpp:239-242 reads data<int64_t>()
  Tensor o = c.alloc(TQP_I64, 1, 1);
  if (t.size() == 0) {
    TQP_CUDA(cudaMemsetAsync(o.data(), 0, 8, c.stream));
  } else {
    TQP_CUDA(cudaMemcpyAsync(o.data(), t.ptr<int64_t>() + t.size() - 1, 8, cudaMemcpyDeviceToDevice, c.stream));
  }
  return o;
}

Tensor pack_cols(Ctx& c, const std::vector<Tensor>& cols) {
  if (cols.empty()) exec_fail("pack: no columns");
  int64_t n = cols[0].rows;
  int kk = static_cast<int>(cols.size());
  std::vector<const double*> ptrs;
  for (const auto& col : cols) {
    if (col.rows != n || !col.is_vector()) exec_fail("pack: column shape mismatch");
    ptrs.push_back(col.ptr<double>());
  }
  Tensor o = c.alloc(TQP_F64, n, kk);
  auto dp = c.alloc_bytes(sizeof(double*) * kk);
  TQP_CUDA(cudaMemcpyAsync(dp->ptr, ptrs.data(), sizeof(double*) * kk, cudaMemcpyHostToDevice, c.stream));
  if (n) {
    k_pack<<<c.grid_for(n * kk, kBlock), kBlock, 0, c.stream>>>(static_cast<const double* const*>(dp->ptr),
                                                                o.ptr<double>(), n, kk);
    c.count_launch();
  }
  c.sync();  // ptrs must outlive the copy
  return o;
}

Tensor broadcast_rows(Ctx& c, const Tensor& v, int64_t n) {
  if (v.rows != 1) exec_fail("broadcast: value must have one row");
  Tensor o = c.alloc(v.dtype, n, v.cols);
  if (n) {
    TQP_DISPATCH(v.dtype, T,
                 k_bcast_rows<T><<<c.grid_for(n * v.cols, kBlock), kBlock, 0, c.stream>>>(v.ptr<T>(), o.ptr<T>(), n,
                                                                                         v.cols));
    c.count_launch();
  }
  return o;
}

Tensor pad_width_like(Ctx& c, const Tensor& t, const Tensor& like) {
  int64_t target = std::max(t.cols, like.cols);
  if (t.cols == target) return t;
  if (!string_like(t)) exec_fail("pad: expected an int32 string tensor");
  Tensor o = c.alloc(t.dtype, t.rows, target);
  if (t.rows) {
    TQP_DISPATCH(t.dtype, T,
                 k_pad<T><<<c.grid_for(t.rows * target, kBlock), kBlock, 0, c.stream>>>(t.ptr<T>(), o.ptr<T>(), t.rows,
                                                                                       t.cols, target));
    c.count_launch();
  }
  return o;
}

Tensor string_compare(Ctx& c, const Tensor& a, const Tensor& b, int op) {
  if (!string_like(a) || !string_like(b)) exec_fail("string_compare: expected int32 string tensors");
  int64_t rows = std::max(a.rows, b.rows);
  if ((a.rows != rows && a.rows != 1) || (b.rows != rows && b.rows != 1)) exec_fail("string_compare: row mismatch");
  Tensor o = c.alloc(TQP_BOOL, rows, 1);
  if (!rows) return o;
  int g = c.grid_for(rows, kBlock);
  auto go = [&](auto ta, auto tb) {
    using TA = decltype(ta);
    using TB = decltype(tb);
    k_strcmp<TA, TB><<<g, kBlock, 0, c.stream>>>(static_cast<const TA*>(a.data()), static_cast<const TB*>(b.data()),
                                                o.ptr<uint8_t>(), rows, a.rows, a.cols, b.rows, b.cols, op);
  };
  bool a8 = a.dtype == TQP_STR8, b8 = b.dtype == TQP_STR8;
  if (a8 && b8) go(uint8_t{}, uint8_t{});
  else if (a8) go(uint8_t{}, int32_t{});
  else if (b8) go(int32_t{}, uint8_t{});
  else go(int32_t{}, int32_t{});
  c.count_launch();
  return o;
}

}  // namespace k
}  // namespace tqp
