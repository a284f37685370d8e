/* tqp_b200.h — the C-ABI drop-in boundary of the B200 (sm_100a) hot path.
 *
 * This library replaces the execution half of the reference (tensql,
 * /root/reference/proj): the kernel set (include/tensql/kernels.hpp:28-78),
 * the executor's plumbing ops and dispatch loop (src/executor.cpp:190-429),
 * the host Tensor/EncodedTable value carriers (include/tensql/tensor.hpp:49-122,
 * include/tensql/columnar.hpp:33-54) and the thread-pool backend
 * (include/tensql/backend.hpp:22-70). The reference's frontend, optimizer
 * and lowering (plan_operators, operator_plan.hpp:96) stay unchanged: a
 * caller lowers a plan with the reference and hands the resulting
 * OperatorPlan to tqp_executor_create through the tqp_plan_* builder below
 * (INTEGRATION.md shows the 60-line adapter a maintainer adds to tensql).
 *
 * Conventions
 *  - Plain C: opaque handles, plain pointers and sizes. No torch types.
 *  - Every fallible call takes a tqp_status* (may be NULL). On failure it
 *    returns NULL / nonzero and fills status with a code, the reference's
 *    message text and the first offending row (FirstBadIndex semantics,
 *    kernels.cpp:31-45).
 *  - Tensors are device-resident, immutable, row-major (rows, cols), like
 *    tensql::Tensor (tensor.hpp:46-48). Utf8 columns are stored on device as
 *    one byte per UTF-8 byte (TQP_STR8) instead of the reference's Int32 per
 *    byte; uploads accept either and downloads can widen back to Int32.
 *  - All work is enqueued on the context's CUDA stream; calls that return a
 *    data-dependent shape synchronise that stream.
 */
#ifndef TQP_B200_H
#define TQP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TQP_ABI_VERSION 1

/* Physical dtypes: mirrors tensql::DType (tensor.hpp:13) plus STR8. */
typedef enum {
  TQP_BOOL = 0, /* uint8 0/1 */
  TQP_I32 = 1,
  TQP_I64 = 2,
  TQP_F64 = 3,
  TQP_STR8 = 4 /* Utf8 rows, one byte per byte, zero padded (device only) */
} tqp_dtype;

/* Logical column types: mirrors tensql::LogicalType (columnar.hpp:13). */
typedef enum {
  TQP_LT_INT64 = 0,
  TQP_LT_FLOAT64 = 1,
  TQP_LT_DATE = 2,
  TQP_LT_UTF8 = 3,
  TQP_LT_BOOL = 4
} tqp_logical_type;

/* Enum values mirror kernels.hpp:11-16 exactly. */
typedef enum { TQP_EQ = 0, TQP_NE, TQP_LT, TQP_LE, TQP_GT, TQP_GE } tqp_compare_op;
typedef enum { TQP_ADD = 0, TQP_SUB, TQP_MUL, TQP_DIV } tqp_arith_op;
typedef enum { TQP_AND = 0, TQP_OR } tqp_logical_op;
typedef enum { TQP_LEFT = 0, TQP_RIGHT } tqp_search_side;
typedef enum { TQP_SUM = 0, TQP_COUNT, TQP_MIN, TQP_MAX } tqp_reduce_op;
typedef enum { TQP_START = 0, TQP_END, TQP_ANY, TQP_EXACT } tqp_match_anchor;

/* Error classes: the reference's exception types. */
typedef enum {
  TQP_OK = 0,
  TQP_ERR_KERNEL = 1,   /* tensql::KernelError   (tensor.hpp:20-23)     */
  TQP_ERR_EXEC = 2,     /* tensql::ExecError     (interpreter.hpp:11-14) */
  TQP_ERR_PLAN = 3,     /* tensql::PlanError     (expr.hpp:14-17)       */
  TQP_ERR_ENCODING = 4, /* tensql::EncodingError (columnar.hpp:23-26)   */
  TQP_ERR_CUDA = 5,     /* CUDA runtime / device failure               */
  TQP_ERR_ARG = 6       /* bad argument at the C boundary              */
} tqp_error_code;

typedef struct tqp_status {
  int code;        /* tqp_error_code */
  int64_t bad_row; /* first offending row, or -1 */
  char msg[1024];  /* reference message text */
} tqp_status;

typedef struct tqp_ctx tqp_ctx;
typedef struct tqp_tensor tqp_tensor;
typedef struct tqp_table tqp_table;
typedef struct tqp_plan tqp_plan;
typedef struct tqp_executor tqp_executor;
typedef struct tqp_result tqp_result;
typedef struct tqp_pending tqp_pending;

/* ---- context (replaces KernelBackend/backend_by_name, backend.hpp:22-70) -- */
int tqp_abi_version(void);
tqp_ctx* tqp_init(int device, tqp_status* st);
void tqp_shutdown(tqp_ctx* ctx);
int tqp_sync(tqp_ctx* ctx, tqp_status* st);
void* tqp_stream(tqp_ctx* ctx);          /* the cudaStream_t work is enqueued on */
const char* tqp_backend_name(tqp_ctx* ctx); /* "b200" (KernelBackend::name)  */
int tqp_device(tqp_ctx* ctx);
/* Number of this library's kernels launched on ctx since creation. */
int64_t tqp_launch_count(tqp_ctx* ctx);
/* NVRTC the run-time specialised kernels compile with (major * 1000 + minor
 * 10, e.g. 12090), bound from the build's toolkit whatever else the process
 * loaded; < 0 when it cannot be loaded. */
int tqp_jit_nvrtc_version(void);

/* ---- tensors (tensql::Tensor, tensor.hpp:49-122) ------------------------ */
size_t tqp_dtype_size(int dtype);
tqp_tensor* tqp_tensor_from_host(tqp_ctx* ctx, int dtype, int64_t rows, int64_t cols,
                                 const void* host, tqp_status* st);
/* Utf8 upload: host is (rows, cols) Int32 byte values (the reference layout,
 * columnar.cpp:161-175); stored as TQP_STR8. */
tqp_tensor* tqp_tensor_from_host_utf8_i32(tqp_ctx* ctx, int64_t rows, int64_t cols,
                                          const int32_t* host, tqp_status* st);
/* Wraps an existing device buffer (copied; the caller keeps ownership). */
tqp_tensor* tqp_tensor_from_device(tqp_ctx* ctx, int dtype, int64_t rows, int64_t cols,
                                   const void* dev, tqp_status* st);

/* ---- compressed columnar host format (the loader) -------
 * The reference loads columns only from CSV text (columnar.cpp:453-527).
 * This binary host format keeps a column losslessly compressed in (pinned)
 * host memory, so an upload moves fewer bytes over PCIe and the device
 * decodes at HBM speed. Codecs (one per column, chosen by tqp_codec_encode):
 *   RAW   the reference layout as is (any dtype / shape)
 *   FOR   int64/date or one-byte (STR8/BOOL, one column) vector:
 *         v = base + scale * u (frame of reference; scale = gcd of v - min,
 *         e.g. one day in ns for dates)
 *   DICT  float64 vector with <= 256 distinct bit patterns: dict_n patterns
 *         (8 B each, ascending) then the codes
 *   DEC   float64 vector whose every value is exactly (base + u) / scale
 *         for an integer u and scale = 10^d (d <= 4): the decode (an IEEE
 *         division) reproduces the original bits; -0.0, NaN, inf excluded.
 *   DELTA int64 vector in non-decreasing order (sorted keys): code i is
 *         (v_i - v_(i-1)) / scale (code 0 is 0), base = v_0; decoded by a
 *         device prefix sum
 *   ROWDICT STR8 / BOOL rows of any width with <= 256 distinct rows: the
 *         dict_n rows (ascending bytes, padded to 8 B) then the codes
 * Codes u are bit-packed, `width` bits each (1..32), little endian in
 * 32-bit words, plus one spare word: 4 * (ceil(rows * width / 32) + 1) B.
 * Lossless by construction: the encoder verifies every value. */
typedef enum { TQP_CODEC_RAW = 0, TQP_CODEC_FOR = 1, TQP_CODEC_DICT = 2, TQP_CODEC_DEC = 3, TQP_CODEC_DELTA = 4,
               TQP_CODEC_ROWDICT = 5 } tqp_codec_kind;
typedef struct {
  int32_t codec;  /* tqp_codec_kind */
  int32_t width;  /* bits per code (1..32), FOR / DICT / DEC */
  int64_t base;   /* FOR: value of code 0; DEC: integer numerator of code 0; DELTA: v_0 */
  int64_t scale;  /* FOR / DELTA: value step of one code; DEC: the denominator 10^d */
  int32_t dict_n; /* DICT: dictionary entries at the start of the payload */
  int32_t reserved;
} tqp_codec;
/* Upper bound of an encoded payload's bytes (the RAW size plus a dictionary). */
int64_t tqp_codec_bound(int dtype, int64_t rows, int64_t cols);
/* Encodes a host column (device dtype layout: int64/date and float64 8 B
 * per row, STR8 one byte per byte) into `out` (cap bytes); returns the
 * payload bytes and fills *codec, or -1 (status set). Runs on the host's
 * cores. */
int64_t tqp_codec_encode(int dtype, int64_t rows, int64_t cols, const void* host, void* out, int64_t cap,
                         tqp_codec* codec, tqp_status* st);
/* Uploads an encoded payload (pinned host memory for an asynchronous copy)
 * and decodes it on the device into a new tensor of the original dtype and
 * shape, bit-identical to the encoded column. Returns at once: the copy runs
 * on the context's copy stream and the decode on its decode stream, so the
 * payload must stay alive and unchanged until the tensor has been used on
 * the context stream (every entry point taking the tensor, or a table
 * holding it, orders the context stream after the decode) or
 * tqp_tensor_wait + tqp_ctx_sync. Replaces the load step of
 * columnar.cpp:453-527 (EncodedTable columns from host memory). */
tqp_tensor* tqp_tensor_from_encoded(tqp_ctx* ctx, int dtype, int64_t rows, int64_t cols, const tqp_codec* codec,
                                    const void* payload, int64_t bytes, tqp_status* st);
/* Orders the context stream after the tensor's producer (a decode still
 * running on the decode stream); no-op otherwise. 0 or -1 (status set). */
int tqp_tensor_wait(const tqp_tensor* t, tqp_status* st);
int tqp_tensor_dtype(const tqp_tensor* t);
int64_t tqp_tensor_rows(const tqp_tensor* t);
int64_t tqp_tensor_cols(const tqp_tensor* t);
const void* tqp_tensor_data(const tqp_tensor* t); /* device pointer */
/* Copies to a host buffer of rows*cols*dtype_size bytes (STR8 -> bytes). */
int tqp_tensor_to_host(tqp_ctx* ctx, const tqp_tensor* t, void* host, tqp_status* st);
/* STR8 -> Int32 per byte (reference layout). */
int tqp_tensor_to_host_utf8_i32(tqp_ctx* ctx, const tqp_tensor* t, int32_t* host,
                                tqp_status* st);
tqp_tensor* tqp_tensor_retain(tqp_tensor* t);
void tqp_tensor_free(tqp_tensor* t);

/* ---- the kernel set (kernels.hpp:28-78), one entry point per kernel ----- */
tqp_tensor* tqp_compare(tqp_ctx*, const tqp_tensor* a, const tqp_tensor* b, int op, tqp_status*);   /* kernels.hpp:30 */
tqp_tensor* tqp_arith(tqp_ctx*, const tqp_tensor* a, const tqp_tensor* b, int op, tqp_status*);     /* kernels.hpp:34 */
tqp_tensor* tqp_logical(tqp_ctx*, const tqp_tensor* a, const tqp_tensor* b, int op, tqp_status*);   /* kernels.hpp:37 */
tqp_tensor* tqp_logical_not(tqp_ctx*, const tqp_tensor* v, tqp_status*);                           /* kernels.hpp:38 */
tqp_tensor* tqp_select_where(tqp_ctx*, const tqp_tensor* cond, const tqp_tensor* a,
                             const tqp_tensor* b, tqp_status*);                                     /* kernels.hpp:41 */
tqp_tensor* tqp_prefix_sum_exclusive(tqp_ctx*, const tqp_tensor* x, tqp_status*);                   /* kernels.hpp:44 */
tqp_tensor* tqp_compact(tqp_ctx*, const tqp_tensor* values, const tqp_tensor* mask, tqp_status*);   /* kernels.hpp:47 */
tqp_tensor* tqp_argsort_stable(tqp_ctx*, const tqp_tensor* keys, tqp_status*);                      /* kernels.hpp:50 */
tqp_tensor* tqp_gather(tqp_ctx*, const tqp_tensor* values, const tqp_tensor* idx, tqp_status*);     /* kernels.hpp:53 */
tqp_tensor* tqp_searchsorted(tqp_ctx*, const tqp_tensor* sorted, const tqp_tensor* probes,
                             int side, tqp_status*);                                                /* kernels.hpp:57 */
tqp_tensor* tqp_expand_segments(tqp_ctx*, const tqp_tensor* starts, const tqp_tensor* counts,
                                tqp_status*);                                                       /* kernels.hpp:61 */
tqp_tensor* tqp_segment_starts(tqp_ctx*, const tqp_tensor* sorted_keys, tqp_status*);               /* kernels.hpp:64 */
tqp_tensor* tqp_segmented_reduce(tqp_ctx*, const tqp_tensor* values, const tqp_tensor* ids,
                                 int64_t num_segments, int op, tqp_status*);                        /* kernels.hpp:69 */
tqp_tensor* tqp_matmul(tqp_ctx*, const tqp_tensor* a, const tqp_tensor* b, tqp_status*);            /* kernels.hpp:73 */
tqp_tensor* tqp_substring_match(tqp_ctx*, const tqp_tensor* chars, const char* pattern,
                                int64_t pattern_len, int anchor, tqp_status*);                      /* kernels.hpp:79 */

/* ---- executor plumbing ops (executor.cpp:190-278) ----------------------- */
tqp_tensor* tqp_iota(tqp_ctx*, int64_t n, tqp_status*);                                 /* IotaRows/IotaLen :223-236 */
tqp_tensor* tqp_cast(tqp_ctx*, const tqp_tensor* t, int to_dtype, tqp_status*);         /* Cast :137-146 */
tqp_tensor* tqp_exp_f64(tqp_ctx*, const tqp_tensor* t, tqp_status*);                    /* ExpF64 :171-178 */
tqp_tensor* tqp_last_or_zero(tqp_ctx*, const tqp_tensor* t, tqp_status*);               /* LastOrZero :239-242 */
tqp_tensor* tqp_pack_cols(tqp_ctx*, const tqp_tensor* const* cols, int n, tqp_status*); /* PackCols :243-255 */
tqp_tensor* tqp_broadcast_rows(tqp_ctx*, const tqp_tensor* value, int64_t n, tqp_status*); /* BroadcastScalar :256-261 */
tqp_tensor* tqp_pad_width_like(tqp_ctx*, const tqp_tensor* t, const tqp_tensor* like,
                               tqp_status*);                                            /* PadWidthLike :262-273 */
tqp_tensor* tqp_sort_perm_rows(tqp_ctx*, const tqp_tensor* key, const tqp_tensor* perm,
                               int ascending, tqp_status*);                             /* SortPermRows :44-68 */
tqp_tensor* tqp_string_compare(tqp_ctx*, const tqp_tensor* a, const tqp_tensor* b, int op,
                               tqp_status*);                                            /* StringCompare :72-108 */

/* ---- tables (EncodedTable, columnar.hpp:41-54) -------------------------- */
tqp_table* tqp_table_create(tqp_ctx* ctx, tqp_status* st);
/* Adds a column; takes a reference to t (the caller may free its handle). */
int tqp_table_add_column(tqp_table* tab, const char* name, int logical_type, tqp_tensor* t,
                         tqp_status* st);
/* A column the plan's input schema names (the reference binds every catalog
 * column, executor.cpp:355-371) but no LoadColumn reads: name, logical type
 * and row count only, no device data (a drop-in upload skips the bytes). A
 * plan that does load it fails with an ExecError. */
int tqp_table_declare_column(tqp_table* tab, const char* name, int logical_type, int64_t rows, tqp_status* st);
int64_t tqp_table_rows(const tqp_table* tab);
int tqp_table_num_columns(const tqp_table* tab);
const char* tqp_table_column_name(const tqp_table* tab, int i);
int tqp_table_column_type(const tqp_table* tab, int i);
tqp_tensor* tqp_table_column(const tqp_table* tab, int i); /* new handle: tqp_tensor_free */
void tqp_table_free(tqp_table* tab);

/* Device-side TPC-H generator (include/tqp_gen.h, bit-identical to the host
 * one): table in {"lineitem","orders","customer","part"}; rows of shard
 * `shard` of `nshards` (lineitem/orders split on order boundaries). */
tqp_table* tqp_gen_table(tqp_ctx* ctx, const char* table, double sf, uint64_t seed, int shard,
                         int nshards, tqp_status* st);

/* ---- CSV loader ---------------------------------------
 * tensql::parse_csv_text (columnar.cpp:453-519): the header line of `text`
 * must name the schema's columns (case-insensitive); every data line is split
 * on `delimiter` and parsed on the device into a table with the schema's names
 * and logical types (TQP_LT_*). Field syntax, rounding and every error message
 * are the reference's (std::from_chars, encode_date, valid_utf8); errors come
 * back as EncodingError ("<origin>:<line>: column '<c>' (field k): ..."). */
tqp_table* tqp_csv_parse(tqp_ctx* ctx, const char* text, int64_t len, const char* const* names,
                         const int* logical_types, int ncols, char delimiter, const char* origin,
                         tqp_status* st);
/* tensql::load_csv (columnar.cpp:521-527): the file is read into pinned host
 * memory and copied to HBM once; origin = path. */
tqp_table* tqp_csv_load(tqp_ctx* ctx, const char* path, const char* const* names,
                        const int* logical_types, int ncols, char delimiter, tqp_status* st);

/* ---- OperatorPlan builder (operator_plan.hpp:16-92) ----------------------
 * op names are the reference's instr_op_name strings (operator_plan.cpp:11-42):
 * "compare", "arith", ..., "load_column", "const", "iota_rows", ... */
typedef struct tqp_instr_desc {
  const char* op;
  const int* inputs;
  int num_inputs;
  int output;
  int cmp, arith, logic, side, reduce, anchor; /* enum values above */
  int cast_to;                                 /* tqp_dtype (BOOL..F64) */
  const char* pattern;                         /* SubstringMatch */
  int64_t pattern_len;
  const char* table;                           /* LoadColumn */
  const char* column;
  int64_t param;                               /* Instr::param */
  /* ConstTensor: host data in the reference layout (Int32 for strings) */
  int const_dtype;
  int64_t const_rows, const_cols;
  const void* const_data;
} tqp_instr_desc;

tqp_plan* tqp_plan_create(int num_slots, tqp_status* st);
int tqp_plan_begin_step(tqp_plan* p, const char* id, const char* kind, tqp_status* st);
int tqp_plan_add_instr(tqp_plan* p, const tqp_instr_desc* d, tqp_status* st);
int tqp_plan_set_step_outputs(tqp_plan* p, const int* slots, int n, tqp_status* st);
int tqp_plan_add_output(tqp_plan* p, const char* name, int logical_type, int slot,
                        tqp_status* st);
int tqp_plan_add_input_column(tqp_plan* p, const char* table, const char* column,
                              int logical_type, tqp_status* st);
void tqp_plan_free(tqp_plan* p);
/* Fused pipelines the executor would choose for this plan (JSON; needs no
 * device; the string is owned by the library, valid until the next call). */
const char* tqp_plan_fusion_explain(const tqp_plan* p);

/* ---- executor (tensql::Executor, executor.hpp:43-59) --------------------- */
#define TQP_EXEC_FUSE 1u      /* pattern-match steps into fused pipelines */
#define TQP_EXEC_NO_FUSE 0u   /* every instruction on its own device kernel */
/* Validates SSA form and computes last use (Executor::Executor,
 * executor.cpp:314-344); PlanError on violation. */
tqp_executor* tqp_executor_create(tqp_ctx* ctx, const tqp_plan* p, unsigned flags,
                                  tqp_status* st);
/* Executor::execute (executor.cpp:346,354-429). tables[i] is bound to names[i]
 * (case-insensitive). Result stays on device until downloaded. */
tqp_result* tqp_executor_execute(tqp_executor* ex, const char* const* names,
                                 tqp_table* const* tables, int ntables, tqp_status* st);
/* Executor::execute without its final host synchronisation (an extension of
 * executor.cpp:346: a serving loop submits the next query while this one
 * runs). When the plan's last fused unit can defer its precondition check
 * (only instruction-free steps follow it), returns with the work queued on
 * the context stream; otherwise the run completes first. tqp_pending_wait
 * finishes it: the unit's check word is read, a unit that met data outside
 * its contract re-runs the plan on the checked path (the tables must stay
 * alive until then), and the completed result is returned - the same
 * result and errors as tqp_executor_execute. */
tqp_pending* tqp_executor_execute_async(tqp_executor* ex, const char* const* names,
                                        tqp_table* const* tables, int ntables, tqp_status* st);
/* Completes and frees `p`; returns the result (or NULL, status set). */
tqp_result* tqp_pending_wait(tqp_pending* p, tqp_status* st);
/* Frees a pending execution without waiting for its result. */
void tqp_pending_free(tqp_pending* p);
/* Same run with a ProfileTrace (executor.hpp:12-38) rendered as Chrome
 * trace-event JSON into a malloc'd string the caller frees with tqp_free_str. */
tqp_result* tqp_executor_profile(tqp_executor* ex, const char* const* names,
                                 tqp_table* const* tables, int ntables, char** trace_json,
                                 tqp_status* st);
/* Per-unit device time (CUDA events on the context stream, no host sync
 * until read): unit = fused pipeline name or "step:<kind>". JSON owned by
 * the library, valid until the next call on this thread. on: 0 off, 1 units,
 * steps and every kernel, 2 the fused fact-scan kernels only. */
void tqp_executor_set_timing(tqp_executor* ex, int on);
const char* tqp_executor_timings(tqp_executor* ex);
void tqp_executor_reset_timings(tqp_executor* ex);
/* ---- sharded execution (the reference runs one process,
 * so there is no reference entry point: executor.cpp:346 is the unsharded
 * equivalent). Each shard runs phase 1 over its rows of the fact table
 * (lineitem cut on order boundaries, dimension tables whole or co-partitioned)
 * and gets an opaque partial: a device I64 tensor of `rows` words, moved
 * between GPUs as rows*8 bytes (NCCL all-gather). Phase 2 merges the partials
 * of all shards, in shard order, on any one GPU and runs the remaining steps;
 * the result equals the unsharded run (bit-exact for integers and
 * build-grouped sums, fp64 scan sums within 1e-9 relative). */
/* 1 if the plan can run sharded; else 0 and *why (thread-local string). */
int tqp_executor_shardable(tqp_executor* ex, const char** why);
tqp_tensor* tqp_executor_execute_partial(tqp_executor* ex, const char* const* names,
                                         tqp_table* const* tables, int ntables, tqp_status* st);
/* parts[i]: device pointer to partial i's words, words[i] its word count. */
tqp_result* tqp_executor_finish(tqp_executor* ex, const void* const* parts, const int64_t* words,
                                int nparts, tqp_status* st);

/* ---- communicators and one-call sharded execution ----
 * One rank per GPU. tqp_executor_execute_sharded runs phase 1 on this rank's
 * tables with the build-side exchanges their layout needs (row-shard
 * dimension tables: presence / flag bitmaps all-gathered over the global key
 * range; row-shard tables whose rows the scan reads: rows re-aligned to the
 * fact shards' key ranges with a grouped send/recv all-to-all), all-gathers
 * the partials and merges them on every rank: every rank returns the whole
 * result. Plans that cannot shard, or shards whose data leave the fused
 * contract, run on the tables all-gathered to every rank, so the result and
 * errors are the reference's either way (executor.cpp:346 is the unsharded
 * equivalent; the reference has no sharded entry point). */
typedef struct tqp_comm tqp_comm;
typedef enum { TQP_SHARD_REPLICATED = 0, TQP_SHARD_COPARTITIONED = 1, TQP_SHARD_ROWS = 2 } tqp_shard_kind;
/* 128-byte NCCL unique id, made on one rank and sent to the others by the
 * caller (e.g. torch.distributed broadcast); NCCL is bound at run time. */
int tqp_comm_nccl_unique_id(void* out128, tqp_status* st);
tqp_comm* tqp_comm_init_nccl(tqp_ctx* ctx, const void* id128, int nranks, int rank, tqp_status* st);
/* n ranks that are threads of this process (out[0..n)); each thread uses its
 * own context. For single-GPU tests of the sharded paths (NCCL needs one
 * GPU per rank). */
int tqp_comm_init_local(int n, tqp_comm** out, tqp_status* st);
int tqp_comm_rank(const tqp_comm* comm);
int tqp_comm_size(const tqp_comm* comm);
const char* tqp_comm_kind(const tqp_comm* comm);
void tqp_comm_free(tqp_comm* comm);
/* kinds[i]: tqp_shard_kind of tables[i] (lineitem / orders cut on order
 * boundaries: COPARTITIONED; part / customer row-sharded: ROWS) */
tqp_result* tqp_executor_execute_sharded(tqp_executor* ex, tqp_comm* comm, const char* const* names,
                                         tqp_table* const* tables, const int* kinds, int ntables, tqp_status* st);
/* JSON of this executor's last sharded run: {"path": "fused" | "gathered" |
 * "unsharded", "ranks", "bitmap_merges", "shuffled_tables", "exchange_bytes"} */
const char* tqp_executor_shard_stats(tqp_executor* ex);

/* Description of the fused pipelines chosen for this plan (JSON). */
const char* tqp_executor_explain(tqp_executor* ex);
/* Fused units that met data outside their contract (duplicate build keys,
 * too many groups, fixed-point or int64 range, ...) and ran the exact
 * per-instruction path instead, since the executor was created. */
int64_t tqp_executor_fallbacks(tqp_executor* ex);
void tqp_executor_free(tqp_executor* ex);
void tqp_free_str(char* s);

int64_t tqp_result_rows(const tqp_result* r);
int tqp_result_num_columns(const tqp_result* r);
const char* tqp_result_column_name(const tqp_result* r, int i);
int tqp_result_column_type(const tqp_result* r, int i);
tqp_tensor* tqp_result_column(const tqp_result* r, int i); /* borrowed */
void tqp_result_free(tqp_result* r);

#ifdef __cplusplus
}
#endif
#endif /* TQP_B200_H */
