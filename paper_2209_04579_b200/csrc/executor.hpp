// B200 executor: device-side counterpart of tensql::Executor
// (executor.hpp:43-59, executor.cpp:314-429) over the reference's lowered
// OperatorPlan (operator_plan.hpp:16-92), with pattern-matched fused
// pipelines (fused.cu) for the relational shapes TPC-H Q1/Q3/Q6/Q14 lower to.
#pragma once

#include <chrono>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <vector>

#include "tqp_internal.hpp"

namespace tqp {

enum class Op : uint8_t {
  Compare, Arith, Logical, Not, SelectWhere, PrefixSum, Compact, ArgsortStable, Gather, SearchSorted,
  ExpandSegments, SegmentStarts, SegmentedReduce, MatMul, SubstringMatch,
  LoadColumn, ConstTensor, IotaRows, IotaLen, Cast, ExpF64, LastOrZero, PackCols, BroadcastScalar,
  PadWidthLike, SortPermRows, StringCompare,
};
bool op_from_name(const std::string& name, Op* out);
const char* op_name(Op op);

struct Instr {
  Op op{};
  std::vector<int> inputs;
  int output = -1;
  int cmp = 0, arith = 0, logic = 0, side = 0, reduce = 0, anchor = 0, cast_to = 0;
  std::string pattern, table, column;
  int64_t param = -1;
  // ConstTensor: host copy (reference layout) + device copy
  int const_dtype = TQP_I64;
  int64_t const_rows = 0, const_cols = 1;
  std::vector<uint8_t> const_host;
  Tensor constant;
};

struct Step {
  std::string id, kind;
  std::vector<Instr> instrs;
  std::vector<int> output_slots;
};

struct OutputCol {
  std::string name;
  int type;
  int slot;
};

struct InputTable {
  std::string name;
  std::vector<std::pair<std::string, int>> schema;
};

struct Plan {
  int num_slots = 0;
  std::vector<Step> steps;
  std::vector<OutputCol> outputs;
  std::vector<InputTable> input_tables;
};

// Min/max of an int64 column, computed on the device the first time a build
// side keys on it and kept with the column: table columns are immutable once
// on the device (the reference never mutates an input), so the
// range is table metadata like its row count, not a per-query result.
struct KeyRange {
  std::mutex mu;
  bool ready = false;
  long long mn = 0, mx = 0;
  int day = -1;  // Date keys: 1 every value is a whole day in ns, 0 not, -1 not computed
  // 1: no value repeats (checked once, on the device, the first time a
  // direct-addressed build keys on the column), 0: some value repeats,
  // -1: not checked
  int unique = -1;
};

// Dictionary of an int64 key column (MODE_HASH keys whose value range is too
// wide to pack): the distinct values ascending, and an open-addressing map
// value -> rank; cached with the (immutable) column like its KeyRange.
struct KeyDict {
  std::mutex mu;
  bool ready = false;
  long long d = 0;                      // distinct values
  Tensor vals;                          // (d, 1) int64, ascending
  std::shared_ptr<DevBuf> hkeys, hranks;
  unsigned long long mask = 0;
  long long empty = 0;                  // marker of an empty map slot (column min - 1)
};

struct Column {
  std::string name;
  int type;  // logical
  Tensor t;
  std::shared_ptr<KeyRange> range = std::make_shared<KeyRange>();
  std::shared_ptr<KeyDict> dict = std::make_shared<KeyDict>();
};

struct Table {
  std::vector<Column> cols;
  int64_t rows = 0;
  const Column* find(const std::string& name) const;
};

using TableSet = std::vector<std::pair<std::string, const Table*>>;

struct KernelTrace {
  std::string op_id, kernel;
  int64_t start_ns, wall_ns, rows, bytes;
};
struct OperatorTrace {
  std::string id, kind;
  int64_t start_ns, wall_ns, rows_out, bytes;
};
struct ProfileTrace {
  std::string backend = "b200";
  std::vector<OperatorTrace> operators;
  std::vector<KernelTrace> kernels;
  std::string to_chrome_json() const;
};

struct Result {
  std::vector<Column> cols;
  int64_t rows = 0;
};

// Phase-1 state of a sharded run (fused.cu describes the word layout).
struct Comm;
// How a sharded run's tables are laid out across the ranks: 0 replicated
// (every rank holds the whole table), 1 co-partitioned with the fact table
// (rows cut on the join key's boundaries, e.g. orders with lineitem: joins
// stay local), 2 row shard (any rows: dimension build sides are exchanged -
// presence / flag bitmaps all-gathered, or rows re-aligned to the fact shards).
enum ShardKind : int { SHARD_REPLICATED = 0, SHARD_COPARTITIONED = 1, SHARD_ROWS = 2 };
struct ShardEnv {
  Comm* comm = nullptr;
  std::map<std::string, int> kinds;  // lower-case table name -> ShardKind (default SHARD_REPLICATED)
  int kind_of(const std::string& table) const;
  // what the run did (reported by Executor::shard_stats)
  mutable long long bitmap_merges = 0, shuffled_tables = 0, exchange_bytes = 0;
  mutable bool gathered = false;
};
struct Partial {
  std::shared_ptr<DevBuf> buf;
  int64_t words = 0;
  const ShardEnv* env = nullptr;  // set by execute_sharded: exchanges inside phase 1
};
// a partial as handed back for the merge (device pointer, any owner)
struct PartRef {
  const void* ptr = nullptr;
  int64_t words = 0;
};

// A fused pipeline replaces a contiguous range of steps [first, last] and
// writes the slots later instructions (or the plan outputs) read.
// A fused unit whose outputs go straight to the result (only instruction-free
// steps follow it) need not wait for its error/row-count word before the
// executor moves on: the word is copied to pinned memory with the outputs
// and checked at the result's one synchronisation (Executor::execute).
struct UnitPending {
  bool active = false;
  long long nrows = -1;            // host-known row count, or -1: err[2]
  std::vector<const void*> outs;   // device buffers of the unit's outputs
  std::shared_ptr<DevBuf> err;     // the device word (kept until read)
  long long* host = nullptr;       // pinned destination of the 4 words (null: Ctx::kPinnedUnitErr)
};

// An execution whose last fused unit's check is still on the device
// (Executor::execute_async): the outputs are queued on the context stream,
// the unit's error words travel to `host` (a pinned slot of the context) and
// an event marks their arrival. wait() checks them and either finishes the
// result (row count patched) or, when the unit met data outside its
// contract, runs the plan again on the checked path over the same tables
// (the caller keeps them alive until then).
struct AsyncResult {
  Result r;
  UnitPending pend;
  TableSet tables;
  cudaEvent_t done = nullptr;
  std::shared_ptr<long long> slot;  // pinned, 4 words
  bool complete = false;            // r is final already (nothing deferred)
};

struct FusedUnit {
  int first_step = 0, last_step = 0;
  std::string name;  // e.g. "scan_filter_aggregate"
  std::string explain;
  // returns false when the data violates the fused path's preconditions
  // (e.g. a fixed-point overflow or a non-unique build key); the executor
  // then runs the covered steps through the per-instruction path.
  // pend != nullptr: deferred check (see UnitPending); returns true
  std::function<bool(Ctx&, std::vector<std::optional<Tensor>>& slots, const TableSet& tables, UnitPending* pend)> run;
  // sharded runs: phase 1 writes this shard's partial state (false: the data
  // violates the preconditions); phase 2 merges the parts of every shard
  std::function<bool(Ctx&, const TableSet& tables, Partial* out)> partial;
  std::function<void(Ctx&, std::vector<std::optional<Tensor>>& slots, const std::vector<PartRef>& parts)> finish;
};

class Executor {
 public:
  Executor(Ctx& ctx, Plan plan, unsigned flags);
  Result execute(const TableSet& tables, ProfileTrace* trace = nullptr, bool allow_defer = true);
  // execute() without the final synchronisation when the plan's last fused
  // unit can defer its check (only instruction-free steps after it); else
  // the completed result. wait() finishes it (see AsyncResult).
  AsyncResult execute_async(const TableSet& tables);
  Result wait(AsyncResult& a);

  // Sharded execution: every shard runs phase 1 over its
  // rows of the fact table; the concatenated partials of all shards (rank
  // order) go through finish() on any one of them. Requires the plan to be a
  // single fused unit over the fact table plus steps that only read its
  // outputs; shardable() says why not otherwise.
  Partial execute_partial(const TableSet& tables);
  Result finish(const std::vector<PartRef>& parts);
  // One call per rank (every rank gets the whole result): phase 1 with the
  // build-side exchanges the table layout needs, an all-gather of the
  // partials, phase 2 on every rank. Plans that cannot shard, or shards that
  // leave the fused contract, run on the tables gathered to every rank (the
  // reference's result and errors either way).
  Result execute_sharded(const TableSet& tables, const ShardEnv& env);
  // JSON of the last execute_sharded: path ("fused" or "gathered"), build
  // sides merged as bitmaps, tables re-aligned, bytes this rank exchanged
  const std::string& shard_stats() const { return shard_stats_; }
  bool shardable(std::string* why = nullptr) const;
  const Plan& plan() const { return plan_; }
  std::string explain() const;

  // Device-time accounting per unit (fused pipeline or generic step) with
  // CUDA events on the context stream; no host synchronisation until read.
  // mode 1: units, steps and every kernel; 2: the fused fact-scan kernels
  // only (an event pair costs a few us of host time per launch, so a timed
  // benchmark region records just the kernel its roofline is quoted on).
  void set_timing(int mode) {
    timing_ = mode == 1;
    ctx_.time_kernels = mode;
  }
  std::string timings_json();
  // fused units that met data outside their contract and ran the exact
  // per-instruction path instead (since creation)
  int64_t fallbacks() const { return fallbacks_; }
  void reset_timings();

 private:
  struct UnitTiming {
    int64_t calls = 0;
    double total_ms = 0.0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
  };
  void time_begin(cudaEvent_t* ev);
  void time_end(const std::string& name, cudaEvent_t start);
  void drain_timings();
  void collect_kernel_events();
  bool timing_ = false;
  int64_t fallbacks_ = 0;
  std::string shard_stats_ = "{}";
  std::map<std::string, UnitTiming> timings_;

  Tensor exec_instr(const Instr& in, std::vector<std::optional<Tensor>>& slots, const TableSet& tables);
  void run_step(int s, std::vector<std::optional<Tensor>>& slots, const TableSet& tables, ProfileTrace* trace,
                int64_t run_start);
  void release_after(int s, std::vector<std::optional<Tensor>>& slots);
  void check_inputs(const TableSet& tables) const;
  Result collect_outputs(std::vector<std::optional<Tensor>>& slots, bool check_rows = true, bool sync = true);
  Result run_units(const TableSet& tables, ProfileTrace* trace, bool allow_defer, UnitPending& pend, bool sync);
  Result gather_and_execute(const TableSet& tables, const ShardEnv& env);

  Ctx& ctx_;
  Plan plan_;
  unsigned flags_;
  std::vector<int64_t> last_use_;          // per slot: global instruction ordinal of last read
  std::vector<int64_t> step_first_ordinal_;
  std::vector<FusedUnit> units_;
};

// fused.cu: recognises fusable step patterns
std::vector<FusedUnit> plan_fusion(Ctx& ctx, const Plan& plan);

const Table* bind_table(const TableSet& tables, const std::string& name);
bool iequals(const std::string& a, const std::string& b);

}  // namespace tqp
