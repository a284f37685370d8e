// extern "C" boundary (include/tqp_b200.h): converts C++ errors into
// tqp_status and owns the opaque handles.
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "comm.hpp"
#include "executor.hpp"
#include "jit.hpp"

using namespace tqp;

struct tqp_table {
  Ctx* ctx = nullptr;
  Table t;
};
struct tqp_plan {
  Plan p;
};
struct tqp_executor {
  Ctx* ctx = nullptr;
  std::unique_ptr<Executor> ex;
  std::string explain;
};
struct tqp_result {
  Result r;
  std::vector<tqp_tensor*> handles;
};
struct tqp_pending {
  tqp_executor* ex = nullptr;
  AsyncResult a;
};

namespace {

void set_status(tqp_status* st, int code, const char* msg, int64_t row) {
  if (!st) return;
  st->code = code;
  st->bad_row = row;
  std::snprintf(st->msg, sizeof(st->msg), "%s", msg);
}
void ok_status(tqp_status* st) {
  if (st) {
    st->code = TQP_OK;
    st->bad_row = -1;
    st->msg[0] = 0;
  }
}

template <typename F>
auto guard(tqp_status* st, F&& f) -> decltype(f()) {
  ok_status(st);
  try {
    return f();
  } catch (const Error& e) {
    set_status(st, e.code, e.what(), e.bad_row);
  } catch (const std::exception& e) {
    set_status(st, TQP_ERR_CUDA, e.what(), -1);
  }
  using R = decltype(f());
  if constexpr (std::is_pointer_v<R>) return nullptr;
  else return static_cast<R>(-1);
}

tqp_tensor* wrap(Tensor t) {
  auto* h = new tqp_tensor;
  h->t = std::move(t);
  return h;
}

// every entry point reaches a tensor through T_, so a tensor still being
// decoded on the decode stream is waited for here (on the context stream)
const Tensor& T_(const tqp_tensor* t) {
  if (!t) throw Error(TQP_ERR_ARG, "null tensor handle");
  if (t->t.buf && t->t.buf->ready && t->t.buf->ctx) t->t.buf->ctx->wait_ready(*t->t.buf);
  return t->t;
}
// the tensor without waiting (metadata only: a table column is added while
// its decode may still run)
const Tensor& TH_(const tqp_tensor* t) {
  if (!t) throw Error(TQP_ERR_ARG, "null tensor handle");
  return t->t;
}
// the same for every column of the tables an executor call binds
void wait_tables(const TableSet& ts) {
  for (const auto& nt : ts)
    if (nt.second)
      for (const auto& col : nt.second->cols)
        if (col.t.buf && col.t.buf->ready && col.t.buf->ctx) col.t.buf->ctx->wait_ready(*col.t.buf);
}
Ctx& C_(tqp_ctx* c) {
  if (!c) throw Error(TQP_ERR_ARG, "null context");
  return c->c;
}

}  // namespace

extern "C" {

int tqp_abi_version(void) { return TQP_ABI_VERSION; }

tqp_ctx* tqp_init(int device, tqp_status* st) {
  return guard(st, [&]() -> tqp_ctx* {
    auto* h = new tqp_ctx;
    Ctx& c = h->c;
    c.device = device;
    TQP_CUDA(cudaSetDevice(device));
    TQP_CUDA(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, device));
    TQP_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    TQP_CUDA(cudaDeviceGetDefaultMemPool(&c.pool, device));
    uint64_t threshold = UINT64_MAX;  // keep freed blocks cached in the pool
    TQP_CUDA(cudaMemPoolSetAttribute(c.pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    TQP_CUDA(cudaMalloc(&c.d_err, 64));
    TQP_CUDA(cudaMallocHost(&c.h_err, sizeof(long long) * Ctx::kPinnedWords));
    // constant sources of small async uploads (see Ctx::kPinned*)
    c.h_err[Ctx::kPinnedErrInit] = 0x7fffffffffffffffLL;
    c.h_err[Ctx::kPinnedErrInit + 1] = 0;
    c.h_err[Ctx::kPinnedErrInit + 2] = 0;
    for (int i = 0; i < Ctx::kPinnedMinMaxPairs; ++i) {
      c.h_err[Ctx::kPinnedMinMax + 2 * i] = 0x7fffffffffffffffLL;
      c.h_err[Ctx::kPinnedMinMax + 2 * i + 1] = static_cast<long long>(0x8000000000000000ULL);
    }
    for (int i = 0; i < Ctx::kMaxDeferred; ++i) {
      long long* w = c.h_err + Ctx::kPinnedDeferInit + 4 * i;
      w[0] = 0x7fffffffffffffffLL;
      w[1] = w[2] = w[3] = 0;
    }
    TQP_CUDA(cudaMalloc(&c.d_defer, 4 * sizeof(long long) * Ctx::kMaxDeferred));
    TQP_CUDA(cudaMemcpy(c.d_defer, c.h_err + Ctx::kPinnedDeferInit, 4 * sizeof(long long) * Ctx::kMaxDeferred,
                        cudaMemcpyHostToDevice));
    return h;
  });
}

void tqp_shutdown(tqp_ctx* ctx) {
  if (!ctx) return;
  ctx->c.release_small();
  cudaStreamSynchronize(ctx->c.stream);
  if (ctx->c.copy_stream) cudaStreamSynchronize(ctx->c.copy_stream);
  if (ctx->c.decode_stream) cudaStreamSynchronize(ctx->c.decode_stream);
  ctx->c.release_stages();
  ctx->c.release_pinned();
  cudaFree(ctx->c.d_err);
  cudaFree(ctx->c.d_defer);
  cudaFreeHost(ctx->c.h_err);
  if (ctx->c.csv_ring) cudaFreeHost(ctx->c.csv_ring);
  for (auto& e : ctx->c.csv_ring_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->c.copy_stream) {
    cudaStreamSynchronize(ctx->c.copy_stream);
    cudaStreamDestroy(ctx->c.copy_stream);
  }
  if (ctx->c.decode_stream) cudaStreamDestroy(ctx->c.decode_stream);
  cudaStreamDestroy(ctx->c.stream);
  delete ctx;
}

int tqp_sync(tqp_ctx* ctx, tqp_status* st) {
  return guard(st, [&] {
    C_(ctx).sync();
    return 0;
  });
}
void* tqp_stream(tqp_ctx* ctx) { return ctx ? ctx->c.stream : nullptr; }
const char* tqp_backend_name(tqp_ctx*) { return "b200"; }
int tqp_device(tqp_ctx* ctx) { return ctx ? ctx->c.device : -1; }
int64_t tqp_launch_count(tqp_ctx* ctx) { return ctx ? ctx->c.launches.load() : 0; }
int tqp_jit_nvrtc_version(void) {
  try {
    return tqp::jit_nvrtc_version();
  } catch (...) {
    return -1;
  }
}

size_t tqp_dtype_size(int dtype) { return dtype_size(dtype); }

tqp_tensor* tqp_tensor_from_host(tqp_ctx* ctx, int dtype, int64_t rows, int64_t cols, const void* host,
                                 tqp_status* st) {
  return guard(st, [&] {
    if (dtype < TQP_BOOL || dtype > TQP_STR8) throw Error(TQP_ERR_ARG, "bad dtype");
    return wrap(upload(C_(ctx), dtype, rows, cols, host));
  });
}

tqp_tensor* tqp_tensor_from_host_utf8_i32(tqp_ctx* ctx, int64_t rows, int64_t cols, const int32_t* host,
                                          tqp_status* st) {
  return guard(st, [&] {
    Ctx& c = C_(ctx);
    if (rows < 0 || cols < 1) kernel_fail("tensor: buffer length does not match shape");
    // narrowed to 1 byte per UTF-8 byte on the host (the reference keeps one
    // Int32 per byte, columnar.cpp:161-175): a quarter of the PCIe bytes;
    // large columns are narrowed by several host threads
    const int64_t n = rows * cols;
    std::vector<uint8_t> bytes(static_cast<size_t>(n));
    const int nt = n >= (int64_t{1} << 22) ? static_cast<int>(std::min<unsigned>(8, std::max(1u, std::thread::hardware_concurrency()))) : 1;
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        const int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
        for (int64_t i = lo; i < hi; ++i) bytes[static_cast<size_t>(i)] = static_cast<uint8_t>(host[i]);
      });
    for (auto& x : th) x.join();
    Tensor o = upload(c, TQP_STR8, rows, cols, bytes.data());
    c.sync();  // `bytes` is a pageable host buffer: the copy has read it
    return wrap(std::move(o));
  });
}

int64_t tqp_codec_bound(int dtype, int64_t rows, int64_t cols) {
  if (dtype < TQP_BOOL || dtype > TQP_STR8 || rows < 0 || cols < 1) return -1;
  return tqp::codec_bound(dtype, rows, cols);
}

int64_t tqp_codec_encode(int dtype, int64_t rows, int64_t cols, const void* host, void* out, int64_t cap,
                         tqp_codec* codec, tqp_status* st) {
  int64_t n = -1;
  guard(st, [&] {
    if (!out || !codec || (!host && rows * cols)) throw Error(TQP_ERR_ARG, "codec: null argument");
    n = tqp::codec_encode(dtype, rows, cols, host, out, cap, codec);
    return 0;
  });
  return n;
}

tqp_tensor* tqp_tensor_from_encoded(tqp_ctx* ctx, int dtype, int64_t rows, int64_t cols, const tqp_codec* codec,
                                    const void* payload, int64_t bytes, tqp_status* st) {
  return guard(st, [&] {
    if (!codec || (!payload && bytes)) throw Error(TQP_ERR_ARG, "codec: null argument");
    if (dtype < TQP_BOOL || dtype > TQP_STR8) throw Error(TQP_ERR_ARG, "bad dtype");
    return wrap(tqp::decode_column(C_(ctx), dtype, rows, cols, *codec, payload, bytes));
  });
}

int tqp_tensor_wait(const tqp_tensor* t, tqp_status* st) {
  return guard(st, [&] {
    T_(t);
    return 0;
  });
}

tqp_tensor* tqp_tensor_from_device(tqp_ctx* ctx, int dtype, int64_t rows, int64_t cols, const void* dev,
                                   tqp_status* st) {
  return guard(st, [&] {
    Ctx& c = C_(ctx);
    Tensor t = c.alloc(dtype, rows, cols);
    if (t.bytes()) TQP_CUDA(cudaMemcpyAsync(t.data(), dev, t.bytes(), cudaMemcpyDeviceToDevice, c.stream));
    return wrap(t);
  });
}

int tqp_tensor_dtype(const tqp_tensor* t) { return t ? t->t.dtype : -1; }
int64_t tqp_tensor_rows(const tqp_tensor* t) { return t ? t->t.rows : -1; }
int64_t tqp_tensor_cols(const tqp_tensor* t) { return t ? t->t.cols : -1; }
const void* tqp_tensor_data(const tqp_tensor* t) {
  if (!t) return nullptr;
  try {
    T_(t);  // ordered after a pending decode on the context stream
  } catch (...) {
  }
  return t->t.data();
}

int tqp_tensor_to_host(tqp_ctx* ctx, const tqp_tensor* t, void* host, tqp_status* st) {
  return guard(st, [&] {
    download(C_(ctx), T_(t), host);
    return 0;
  });
}

int tqp_tensor_to_host_utf8_i32(tqp_ctx* ctx, const tqp_tensor* t, int32_t* host, tqp_status* st) {
  return guard(st, [&] {
    Ctx& c = C_(ctx);
    const Tensor& x = T_(t);
    if (x.dtype == TQP_STR8) download(c, k::str8_to_i32(c, x), host);
    else download(c, x, host);
    return 0;
  });
}

tqp_tensor* tqp_tensor_retain(tqp_tensor* t) {
  if (t) t->refs++;
  return t;
}
void tqp_tensor_free(tqp_tensor* t) {
  if (t && --t->refs == 0) delete t;
}

// ---- kernels -----------------------------------------------------------------
#define TQP_K2(NAME, CALL)                                                                                   \
  tqp_tensor* NAME(tqp_ctx* ctx, const tqp_tensor* a, const tqp_tensor* b, int op, tqp_status* st) {       \
    return guard(st, [&] { return wrap(CALL); });                                                          \
  }
TQP_K2(tqp_compare, k::compare(C_(ctx), T_(a), T_(b), op))
TQP_K2(tqp_arith, k::arith(C_(ctx), T_(a), T_(b), op))
TQP_K2(tqp_logical, k::logical(C_(ctx), T_(a), T_(b), op))
TQP_K2(tqp_string_compare, k::string_compare(C_(ctx), T_(a), T_(b), op))
#undef TQP_K2

tqp_tensor* tqp_logical_not(tqp_ctx* ctx, const tqp_tensor* v, tqp_status* st) {
  return guard(st, [&] { return wrap(k::logical_not(C_(ctx), T_(v))); });
}
tqp_tensor* tqp_select_where(tqp_ctx* ctx, const tqp_tensor* cond, const tqp_tensor* a, const tqp_tensor* b,
                             tqp_status* st) {
  return guard(st, [&] { return wrap(k::select_where(C_(ctx), T_(cond), T_(a), T_(b))); });
}
tqp_tensor* tqp_prefix_sum_exclusive(tqp_ctx* ctx, const tqp_tensor* x, tqp_status* st) {
  return guard(st, [&] { return wrap(k::prefix_sum_exclusive(C_(ctx), T_(x))); });
}
tqp_tensor* tqp_compact(tqp_ctx* ctx, const tqp_tensor* v, const tqp_tensor* m, tqp_status* st) {
  return guard(st, [&] { return wrap(k::compact(C_(ctx), T_(v), T_(m))); });
}
tqp_tensor* tqp_argsort_stable(tqp_ctx* ctx, const tqp_tensor* keys, tqp_status* st) {
  return guard(st, [&] { return wrap(k::argsort_stable(C_(ctx), T_(keys))); });
}
tqp_tensor* tqp_gather(tqp_ctx* ctx, const tqp_tensor* v, const tqp_tensor* idx, tqp_status* st) {
  return guard(st, [&] { return wrap(k::gather(C_(ctx), T_(v), T_(idx))); });
}
tqp_tensor* tqp_searchsorted(tqp_ctx* ctx, const tqp_tensor* s, const tqp_tensor* p, int side, tqp_status* st) {
  return guard(st, [&] { return wrap(k::searchsorted(C_(ctx), T_(s), T_(p), side)); });
}
tqp_tensor* tqp_expand_segments(tqp_ctx* ctx, const tqp_tensor* s, const tqp_tensor* c, tqp_status* st) {
  return guard(st, [&] { return wrap(k::expand_segments(C_(ctx), T_(s), T_(c))); });
}
tqp_tensor* tqp_segment_starts(tqp_ctx* ctx, const tqp_tensor* k_, tqp_status* st) {
  return guard(st, [&] { return wrap(k::segment_starts(C_(ctx), T_(k_))); });
}
tqp_tensor* tqp_segmented_reduce(tqp_ctx* ctx, const tqp_tensor* v, const tqp_tensor* ids, int64_t num, int op,
                                 tqp_status* st) {
  return guard(st, [&] { return wrap(k::segmented_reduce(C_(ctx), T_(v), T_(ids), num, op)); });
}
tqp_tensor* tqp_matmul(tqp_ctx* ctx, const tqp_tensor* a, const tqp_tensor* b, tqp_status* st) {
  return guard(st, [&] { return wrap(k::matmul(C_(ctx), T_(a), T_(b))); });
}
tqp_tensor* tqp_substring_match(tqp_ctx* ctx, const tqp_tensor* chars, const char* pattern, int64_t plen, int anchor,
                                tqp_status* st) {
  return guard(st, [&] {
    return wrap(k::substring_match(C_(ctx), T_(chars), std::string(pattern ? pattern : "", plen), anchor));
  });
}
tqp_tensor* tqp_iota(tqp_ctx* ctx, int64_t n, tqp_status* st) {
  return guard(st, [&] { return wrap(k::iota(C_(ctx), n)); });
}
tqp_tensor* tqp_cast(tqp_ctx* ctx, const tqp_tensor* t, int to, tqp_status* st) {
  return guard(st, [&] { return wrap(k::cast(C_(ctx), T_(t), to)); });
}
tqp_tensor* tqp_exp_f64(tqp_ctx* ctx, const tqp_tensor* t, tqp_status* st) {
  return guard(st, [&] { return wrap(k::exp_f64(C_(ctx), T_(t))); });
}
tqp_tensor* tqp_last_or_zero(tqp_ctx* ctx, const tqp_tensor* t, tqp_status* st) {
  return guard(st, [&] { return wrap(k::last_or_zero(C_(ctx), T_(t))); });
}
tqp_tensor* tqp_pack_cols(tqp_ctx* ctx, const tqp_tensor* const* cols, int n, tqp_status* st) {
  return guard(st, [&] {
    std::vector<Tensor> v;
    for (int i = 0; i < n; ++i) v.push_back(T_(cols[i]));
    return wrap(k::pack_cols(C_(ctx), v));
  });
}
tqp_tensor* tqp_broadcast_rows(tqp_ctx* ctx, const tqp_tensor* v, int64_t n, tqp_status* st) {
  return guard(st, [&] { return wrap(k::broadcast_rows(C_(ctx), T_(v), n)); });
}
tqp_tensor* tqp_pad_width_like(tqp_ctx* ctx, const tqp_tensor* t, const tqp_tensor* like, tqp_status* st) {
  return guard(st, [&] { return wrap(k::pad_width_like(C_(ctx), T_(t), T_(like))); });
}
tqp_tensor* tqp_sort_perm_rows(tqp_ctx* ctx, const tqp_tensor* key, const tqp_tensor* perm, int asc, tqp_status* st) {
  return guard(st, [&] { return wrap(k::sort_perm_rows(C_(ctx), T_(key), T_(perm), asc != 0)); });
}

// ---- tables ------------------------------------------------------------------
tqp_table* tqp_table_create(tqp_ctx* ctx, tqp_status* st) {
  return guard(st, [&] {
    auto* t = new tqp_table;
    t->ctx = &C_(ctx);
    return t;
  });
}

int tqp_table_add_column(tqp_table* tab, const char* name, int lt, tqp_tensor* t, tqp_status* st) {
  return guard(st, [&] {
    if (!tab || !name) throw Error(TQP_ERR_ARG, "null table or name");
    const Tensor& x = TH_(t);
    if (tab->t.find(name)) throw Error(TQP_ERR_ENCODING, std::string("table: duplicate column name '") + name + "'");
    if (!tab->t.cols.empty() && x.rows != tab->t.rows) {
      throw Error(TQP_ERR_ENCODING, std::string("table: column '") + name + "' has " + std::to_string(x.rows) +
                                        " rows, expected " + std::to_string(tab->t.rows));
    }
    int want = physical_dtype(lt);
    if (x.dtype != want || (lt != TQP_LT_UTF8 && x.cols != 1)) {
      throw Error(TQP_ERR_ENCODING, std::string("table: column '") + name + "' tensor dtype does not match logical type");
    }
    if (tab->t.cols.empty()) tab->t.rows = x.rows;
    tab->t.cols.push_back({name, lt, x});
    return 0;
  });
}
int tqp_table_declare_column(tqp_table* tab, const char* name, int lt, int64_t rows, tqp_status* st) {
  return guard(st, [&] {
    if (!tab || !name) throw Error(TQP_ERR_ARG, "null table or name");
    if (lt < TQP_LT_INT64 || lt > TQP_LT_BOOL) throw Error(TQP_ERR_ARG, "bad logical type");
    if (tab->t.find(name)) throw Error(TQP_ERR_ENCODING, std::string("table: duplicate column name '") + name + "'");
    if (!tab->t.cols.empty() && rows != tab->t.rows)
      throw Error(TQP_ERR_ENCODING, std::string("table: column '") + name + "' has " + std::to_string(rows) +
                                        " rows, expected " + std::to_string(tab->t.rows));
    Tensor x;  // no device buffer: a column the plan binds but never loads
    x.dtype = physical_dtype(lt);
    x.rows = rows;
    x.cols = 1;
    if (tab->t.cols.empty()) tab->t.rows = rows;
    tab->t.cols.push_back({name, lt, x});
    return 0;
  });
}

int64_t tqp_table_rows(const tqp_table* tab) { return tab ? tab->t.rows : -1; }
int tqp_table_num_columns(const tqp_table* tab) { return tab ? static_cast<int>(tab->t.cols.size()) : -1; }
const char* tqp_table_column_name(const tqp_table* tab, int i) { return tab->t.cols.at(i).name.c_str(); }
int tqp_table_column_type(const tqp_table* tab, int i) { return tab->t.cols.at(i).type; }
tqp_tensor* tqp_table_column(const tqp_table* tab, int i) {
  // borrowed handle cached on the table is not needed: hand out a fresh one
  // owned by the caller through tqp_tensor_free
  return wrap(tab->t.cols.at(i).t);
}
void tqp_table_free(tqp_table* tab) { delete tab; }

// ---- plans -------------------------------------------------------------------
tqp_plan* tqp_plan_create(int num_slots, tqp_status* st) {
  return guard(st, [&] {
    auto* p = new tqp_plan;
    p->p.num_slots = num_slots;
    return p;
  });
}
int tqp_plan_begin_step(tqp_plan* p, const char* id, const char* kind, tqp_status* st) {
  return guard(st, [&] {
    Step s;
    s.id = id;
    s.kind = kind;
    p->p.steps.push_back(std::move(s));
    return 0;
  });
}
int tqp_plan_add_instr(tqp_plan* p, const tqp_instr_desc* d, tqp_status* st) {
  return guard(st, [&] {
    if (p->p.steps.empty()) throw Error(TQP_ERR_ARG, "tqp_plan_add_instr before tqp_plan_begin_step");
    Instr in;
    if (!op_from_name(d->op ? d->op : "", &in.op)) throw Error(TQP_ERR_PLAN, std::string("unknown instruction ") + d->op);
    if (d->num_inputs < 0 || (d->num_inputs > 0 && !d->inputs)) throw Error(TQP_ERR_ARG, "tqp_plan_add_instr: bad inputs");
    in.inputs.assign(d->inputs, d->inputs + d->num_inputs);
    in.output = d->output;
    in.cmp = d->cmp;
    in.arith = d->arith;
    in.logic = d->logic;
    in.side = d->side;
    in.reduce = d->reduce;
    in.anchor = d->anchor;
    in.cast_to = d->cast_to;
    if (d->pattern) in.pattern.assign(d->pattern, d->pattern_len);
    if (d->table) in.table = d->table;
    if (d->column) in.column = d->column;
    in.param = d->param;
    if (in.op == Op::ConstTensor) {
      if (d->const_dtype < TQP_BOOL || d->const_dtype > TQP_STR8 || d->const_rows < 0 || d->const_cols < 0)
        throw Error(TQP_ERR_ARG, "tqp_plan_add_instr: bad constant dtype or shape");
      in.const_dtype = d->const_dtype;
      in.const_rows = d->const_rows;
      in.const_cols = d->const_cols;
      size_t bytes = static_cast<size_t>(d->const_rows * d->const_cols) * dtype_size(d->const_dtype);
      if (bytes && !d->const_data) throw Error(TQP_ERR_ARG, "tqp_plan_add_instr: null constant data");
      in.const_host.resize(bytes);
      if (bytes) std::memcpy(in.const_host.data(), d->const_data, bytes);
    }
    p->p.steps.back().instrs.push_back(std::move(in));
    return 0;
  });
}
int tqp_plan_set_step_outputs(tqp_plan* p, const int* slots, int n, tqp_status* st) {
  return guard(st, [&] {
    if (p->p.steps.empty()) throw Error(TQP_ERR_ARG, "tqp_plan_set_step_outputs before tqp_plan_begin_step");
    if (n < 0 || (n > 0 && !slots)) throw Error(TQP_ERR_ARG, "tqp_plan_set_step_outputs: bad slot array");
    p->p.steps.back().output_slots.assign(slots, slots + n);
    return 0;
  });
}
int tqp_plan_add_output(tqp_plan* p, const char* name, int lt, int slot, tqp_status* st) {
  return guard(st, [&] {
    p->p.outputs.push_back({name, lt, slot});
    return 0;
  });
}
int tqp_plan_add_input_column(tqp_plan* p, const char* table, const char* column, int lt, tqp_status* st) {
  return guard(st, [&] {
    for (auto& it : p->p.input_tables) {
      if (iequals(it.name, table)) {
        it.schema.push_back({column, lt});
        return 0;
      }
    }
    p->p.input_tables.push_back({table, {{column, lt}}});
    return 0;
  });
}
void tqp_plan_free(tqp_plan* p) { delete p; }

// ---- executor ----------------------------------------------------------------
tqp_executor* tqp_executor_create(tqp_ctx* ctx, const tqp_plan* p, unsigned flags, tqp_status* st) {
  return guard(st, [&] {
    auto* e = new tqp_executor;
    e->ctx = &C_(ctx);
    try {
      e->ex = std::make_unique<Executor>(*e->ctx, p->p, flags);
    } catch (...) {
      delete e;
      throw;
    }
    e->explain = e->ex->explain();
    return e;
  });
}

static tqp_result* run_exec(tqp_executor* ex, const char* const* names, tqp_table* const* tables, int n,
                            ProfileTrace* trace) {
  TableSet ts;
  for (int i = 0; i < n; ++i) ts.push_back({names[i], &tables[i]->t});
  wait_tables(ts);
  auto* r = new tqp_result;
  try {
    r->r = ex->ex->execute(ts, trace);
  } catch (...) {
    delete r;
    throw;
  }
  for (auto& c : r->r.cols) r->handles.push_back(wrap(c.t));
  return r;
}

tqp_result* tqp_executor_execute(tqp_executor* ex, const char* const* names, tqp_table* const* tables, int n,
                                 tqp_status* st) {
  return guard(st, [&] { return run_exec(ex, names, tables, n, nullptr); });
}

tqp_pending* tqp_executor_execute_async(tqp_executor* ex, const char* const* names, tqp_table* const* tables, int n,
                                        tqp_status* st) {
  return guard(st, [&] {
    if (!ex) throw Error(TQP_ERR_ARG, "null executor");
    TableSet ts;
    for (int i = 0; i < n; ++i) ts.push_back({names[i], &tables[i]->t});
    wait_tables(ts);
    auto* p = new tqp_pending;
    p->ex = ex;
    try {
      p->a = ex->ex->execute_async(ts);
    } catch (...) {
      delete p;
      throw;
    }
    return p;
  });
}

tqp_result* tqp_pending_wait(tqp_pending* p, tqp_status* st) {
  return guard(st, [&] {
    if (!p) throw Error(TQP_ERR_ARG, "null pending execution");
    std::unique_ptr<tqp_pending> own(p);
    auto* r = new tqp_result;
    try {
      r->r = p->ex->ex->wait(p->a);
    } catch (...) {
      delete r;
      throw;
    }
    for (auto& c : r->r.cols) r->handles.push_back(wrap(c.t));
    return r;
  });
}

void tqp_pending_free(tqp_pending* p) {
  if (!p) return;
  if (p->a.done) {
    cudaEventSynchronize(p->a.done);  // the slot is written by the queued copy
    cudaEventDestroy(p->a.done);
  }
  delete p;
}

tqp_result* tqp_executor_profile(tqp_executor* ex, const char* const* names, tqp_table* const* tables, int n,
                                 char** trace_json, tqp_status* st) {
  return guard(st, [&] {
    ProfileTrace trace;
    tqp_result* r = run_exec(ex, names, tables, n, &trace);
    if (trace_json) *trace_json = strdup(trace.to_chrome_json().c_str());
    return r;
  });
}

tqp_tensor* tqp_executor_execute_partial(tqp_executor* ex, const char* const* names, tqp_table* const* tables, int n,
                                         tqp_status* st) {
  return guard(st, [&] {
    if (!ex) throw Error(TQP_ERR_ARG, "null executor");
    TableSet ts;
    for (int i = 0; i < n; ++i) ts.push_back({names[i], &tables[i]->t});
    wait_tables(ts);
    Partial p = ex->ex->execute_partial(ts);
    Tensor t;
    t.dtype = TQP_I64;
    t.rows = p.words;
    t.cols = 1;
    t.buf = p.buf;
    return wrap(std::move(t));
  });
}

tqp_result* tqp_executor_finish(tqp_executor* ex, const void* const* parts, const int64_t* words, int nparts,
                                tqp_status* st) {
  return guard(st, [&] {
    if (!ex) throw Error(TQP_ERR_ARG, "null executor");
    if (nparts < 1 || !parts || !words) throw Error(TQP_ERR_ARG, "finish needs at least one partial");
    std::vector<PartRef> refs;
    for (int i = 0; i < nparts; ++i) refs.push_back({parts[i], words[i]});
    auto* r = new tqp_result;
    try {
      r->r = ex->ex->finish(refs);
    } catch (...) {
      delete r;
      throw;
    }
    for (auto& c : r->r.cols) r->handles.push_back(wrap(c.t));
    return r;
  });
}

struct tqp_comm {
  std::unique_ptr<Comm> c;
};

int tqp_comm_nccl_unique_id(void* out128, tqp_status* st) {
  return guard(st, [&] {
    if (!out128) throw Error(TQP_ERR_ARG, "null id buffer");
    nccl_unique_id(out128);
    return 0;
  });
}

tqp_comm* tqp_comm_init_nccl(tqp_ctx* ctx, const void* id128, int nranks, int rank, tqp_status* st) {
  return guard(st, [&]() -> tqp_comm* {
    if (!ctx || !id128) throw Error(TQP_ERR_ARG, "null context or id");
    auto* h = new tqp_comm;
    try {
      h->c = make_nccl_comm(ctx->c, id128, nranks, rank);
    } catch (...) {
      delete h;
      throw;
    }
    return h;
  });
}

int tqp_comm_init_local(int n, tqp_comm** out, tqp_status* st) {
  return guard(st, [&] {
    if (!out) throw Error(TQP_ERR_ARG, "null output array");
    auto g = make_local_group(n);
    for (int i = 0; i < n; ++i) {
      out[i] = new tqp_comm;
      out[i]->c = std::move(g[i]);
    }
    return 0;
  });
}

int tqp_comm_rank(const tqp_comm* comm) { return comm ? comm->c->rank : -1; }
int tqp_comm_size(const tqp_comm* comm) { return comm ? comm->c->size : -1; }
const char* tqp_comm_kind(const tqp_comm* comm) { return comm ? comm->c->kind() : ""; }
void tqp_comm_free(tqp_comm* comm) { delete comm; }

tqp_result* tqp_executor_execute_sharded(tqp_executor* ex, tqp_comm* comm, const char* const* names,
                                         tqp_table* const* tables, const int* kinds, int n, tqp_status* st) {
  return guard(st, [&] {
    if (!ex || !comm) throw Error(TQP_ERR_ARG, "null executor or communicator");
    if (n < 0 || (n > 0 && (!names || !tables || !kinds))) throw Error(TQP_ERR_ARG, "bad table arrays");
    TableSet ts;
    ShardEnv env;
    env.comm = comm->c.get();
    for (int i = 0; i < n; ++i) {
      if (kinds[i] < TQP_SHARD_REPLICATED || kinds[i] > TQP_SHARD_ROWS) throw Error(TQP_ERR_ARG, "bad shard kind");
      ts.push_back({names[i], &tables[i]->t});
      std::string lower = names[i];
      for (auto& ch : lower) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
      env.kinds[lower] = kinds[i];
    }
    wait_tables(ts);
    auto* r = new tqp_result;
    try {
      r->r = ex->ex->execute_sharded(ts, env);
    } catch (...) {
      delete r;
      throw;
    }
    for (auto& c : r->r.cols) r->handles.push_back(wrap(c.t));
    return r;
  });
}

const char* tqp_executor_shard_stats(tqp_executor* ex) { return ex ? ex->ex->shard_stats().c_str() : "{}"; }

int tqp_executor_shardable(tqp_executor* ex, const char** why) {
  static thread_local std::string msg;
  msg.clear();
  const bool ok = ex && ex->ex->shardable(&msg);
  if (!ex) msg = "null executor";
  if (why) *why = msg.c_str();
  return ok ? 1 : 0;
}

const char* tqp_executor_explain(tqp_executor* ex) { return ex ? ex->explain.c_str() : ""; }
int64_t tqp_executor_fallbacks(tqp_executor* ex) { return ex ? ex->ex->fallbacks() : 0; }
void tqp_executor_free(tqp_executor* ex) { delete ex; }
void tqp_free_str(char* s) { std::free(s); }

int64_t tqp_result_rows(const tqp_result* r) { return r ? r->r.rows : -1; }
int tqp_result_num_columns(const tqp_result* r) { return r ? static_cast<int>(r->r.cols.size()) : -1; }
const char* tqp_result_column_name(const tqp_result* r, int i) { return r->r.cols.at(i).name.c_str(); }
int tqp_result_column_type(const tqp_result* r, int i) { return r->r.cols.at(i).type; }
tqp_tensor* tqp_result_column(const tqp_result* r, int i) { return r->handles.at(i); }
void tqp_result_free(tqp_result* r) {
  if (!r) return;
  for (auto* h : r->handles) tqp_tensor_free(h);
  delete r;
}

}  // extern "C"

namespace tqp {
Table gen_table(Ctx& c, const std::string& name, double sf, uint64_t seed, int shard, int nshards);
}

extern "C" tqp_table* tqp_gen_table(tqp_ctx* ctx, const char* table, double sf, uint64_t seed, int shard, int nshards,
                                    tqp_status* st) {
  return guard(st, [&] {
    auto* t = new tqp_table;
    t->ctx = &C_(ctx);
    try {
      t->t = tqp::gen_table(*t->ctx, table ? table : "", sf, seed, shard, nshards);
    } catch (...) {
      delete t;
      throw;
    }
    return t;
  });
}

extern "C" void tqp_executor_set_timing(tqp_executor* ex, int on) {
  if (ex) ex->ex->set_timing(on < 0 || on > 2 ? 1 : on);
}

extern "C" const char* tqp_executor_timings(tqp_executor* ex) {
  static thread_local std::string s;
  try {
    s = ex ? ex->ex->timings_json() : "{}";
  } catch (const std::exception& e) {
    s = "{}";
  }
  return s.c_str();
}

extern "C" void tqp_executor_reset_timings(tqp_executor* ex) {
  if (ex) ex->ex->reset_timings();
}

// Fusion decisions for a plan without a device (the planner is host code).
extern "C" const char* tqp_plan_fusion_explain(const tqp_plan* p) {
  static thread_local std::string s;
  try {
    tqp::Ctx dummy;
    auto units = tqp::plan_fusion(dummy, p->p);
    std::ostringstream os;
    os << "{\"fused\": [";
    for (size_t i = 0; i < units.size(); ++i) {
      const auto& u = units[i];
      os << (i ? ", " : "") << "{\"name\": \"" << u.name << "\", \"steps\": [\"" << p->p.steps[u.first_step].id << "\", \""
         << p->p.steps[u.last_step].id << "\"], \"detail\": \"" << u.explain << "\"}";
    }
    os << "]}";
    s = os.str();
  } catch (const std::exception& e) {
    s = std::string("{\"error\": \"") + e.what() + "\"}";
  }
  return s.c_str();
}

// ---- CSV loader -----------------------------------------------
namespace tqp {
Table csv_parse(Ctx& c, const unsigned char* text, int64_t len, const std::vector<std::pair<std::string, int>>& schema,
                char delimiter, const std::string& origin);
Table csv_load(Ctx& c, const std::string& path, const std::vector<std::pair<std::string, int>>& schema, char delimiter);
}

namespace {
std::vector<std::pair<std::string, int>> csv_schema(const char* const* names, const int* types, int ncols) {
  std::vector<std::pair<std::string, int>> s;
  for (int i = 0; i < ncols; ++i) {
    if (!names || !names[i] || !types) throw Error(TQP_ERR_ARG, "csv: null schema entry");
    if (types[i] < TQP_LT_INT64 || types[i] > TQP_LT_BOOL) throw Error(TQP_ERR_ARG, "csv: bad logical type");
    s.push_back({names[i], types[i]});
  }
  return s;
}
}  // namespace

extern "C" tqp_table* tqp_csv_parse(tqp_ctx* ctx, const char* text, int64_t len, const char* const* names,
                                    const int* logical_types, int ncols, char delimiter, const char* origin,
                                    tqp_status* st) {
  return guard(st, [&] {
    if (!text && len) throw Error(TQP_ERR_ARG, "csv: null text");
    auto schema = csv_schema(names, logical_types, ncols);
    auto* t = new tqp_table;
    t->ctx = &C_(ctx);
    try {
      t->t = tqp::csv_parse(*t->ctx, reinterpret_cast<const unsigned char*>(text), len, schema, delimiter,
                            origin ? origin : "<csv>");
    } catch (...) {
      delete t;
      throw;
    }
    return t;
  });
}

extern "C" tqp_table* tqp_csv_load(tqp_ctx* ctx, const char* path, const char* const* names, const int* logical_types,
                                   int ncols, char delimiter, tqp_status* st) {
  return guard(st, [&] {
    if (!path) throw Error(TQP_ERR_ARG, "csv: null path");
    auto schema = csv_schema(names, logical_types, ncols);
    auto* t = new tqp_table;
    t->ctx = &C_(ctx);
    try {
      t->t = tqp::csv_load(*t->ctx, path, schema, delimiter);
    } catch (...) {
      delete t;
      throw;
    }
    return t;
  });
}
