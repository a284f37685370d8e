// Executor: SSA validation + last-use analysis (executor.cpp:314-344), the
// instruction dispatch loop (executor.cpp:354-429) and exec_instr
// (executor.cpp:190-278), over device tensors. Steps covered by a fused
// pipeline (fused.cu) run as one unit; everything else dispatches one device
// kernel per instruction. There is no CPU fallback: every InstrOp has a
// device implementation.
#include <algorithm>
#include <cctype>
#include <cstring>
#include <limits>
#include <set>
#include <sstream>

#include "comm.hpp"
#include "executor.hpp"

namespace tqp {

namespace {
const char* kOpNames[] = {"compare",       "arith",         "logical",          "not",
                          "select_where",  "prefix_sum_exclusive", "compact",   "argsort_stable",
                          "gather",        "searchsorted",  "expand_segments",  "segment_starts",
                          "segmented_reduce", "matmul",     "substring_match",  "load_column",
                          "const",         "iota_rows",     "iota_len",         "cast",
                          "exp",           "last_or_zero",  "pack_cols",        "broadcast_scalar",
                          "pad_width_like", "sort_perm_rows", "string_compare"};
constexpr int kNumOps = sizeof(kOpNames) / sizeof(kOpNames[0]);

int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

std::string json_escape(const std::string& s) {
  std::string o;
  for (char ch : s) {
    if (ch == '"' || ch == '\\') o += '\\';
    o += ch;
  }
  return o;
}
void check_result_rows(Result& res) {
  res.rows = res.cols.empty() ? 0 : res.cols[0].t.rows;
  for (const auto& c : res.cols) {
    if (c.t.rows != res.rows) {
      throw Error(TQP_ERR_ENCODING, "table: column '" + c.name + "' has " + std::to_string(c.t.rows) +
                                        " rows, expected " + std::to_string(res.rows));
    }
  }
}

}  // namespace

bool op_from_name(const std::string& name, Op* out) {
  for (int i = 0; i < kNumOps; ++i) {
    if (name == kOpNames[i]) {
      *out = static_cast<Op>(i);
      return true;
    }
  }
  return false;
}
const char* op_name(Op op) { return kOpNames[static_cast<int>(op)]; }

bool iequals(const std::string& a, const std::string& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i) {
    if (std::tolower(static_cast<unsigned char>(a[i])) != std::tolower(static_cast<unsigned char>(b[i]))) return false;
  }
  return true;
}

const Column* Table::find(const std::string& name) const {
  for (const auto& c : cols)
    if (iequals(c.name, name)) return &c;
  return nullptr;
}

const Table* bind_table(const TableSet& tables, const std::string& name) {
  const Table* t = nullptr;
  for (const auto& [n, tab] : tables)
    if (iequals(n, name)) t = tab;  // last match wins, as the reference's loop does
  return t;
}

std::string ProfileTrace::to_chrome_json() const {
  std::ostringstream os;
  os << "[\n";
  bool first = true;
  auto sep = [&] {
    if (!first) os << ",\n";
    first = false;
  };
  for (const auto& op : operators) {
    sep();
    os << "  {\"name\": \"" << json_escape(op.id) << "\", \"cat\": \"operator\", \"ph\": \"X\", \"ts\": "
       << op.start_ns / 1000.0 << ", \"dur\": " << op.wall_ns / 1000.0
       << ", \"pid\": 0, \"tid\": 0, \"args\": {\"rows\": " << op.rows_out << ", \"bytes\": " << op.bytes
       << ", \"backend\": \"" << backend << "\"}}";
  }
  for (const auto& k : kernels) {
    sep();
    os << "  {\"name\": \"" << json_escape(k.kernel) << "\", \"cat\": \"kernel\", \"ph\": \"X\", \"ts\": "
       << k.start_ns / 1000.0 << ", \"dur\": " << k.wall_ns / 1000.0
       << ", \"pid\": 0, \"tid\": 1, \"args\": {\"operator\": \"" << json_escape(k.op_id) << "\", \"rows\": " << k.rows
       << ", \"bytes\": " << k.bytes << "}}";
  }
  os << "\n]";
  return os.str();
}

Executor::Executor(Ctx& ctx, Plan plan, unsigned flags) : ctx_(ctx), plan_(std::move(plan)), flags_(flags) {
  // SSA validation and last-use analysis (executor.cpp:314-344)
  std::vector<bool> written(plan_.num_slots, false);
  last_use_.assign(plan_.num_slots, -1);
  int64_t ordinal = 0;
  for (const auto& step : plan_.steps) {
    step_first_ordinal_.push_back(ordinal);
    for (const auto& in : step.instrs) {
      for (int s : in.inputs) {
        if (s < 0 || s >= plan_.num_slots || !written[s]) {
          plan_fail("executor: instruction reads slot " + std::to_string(s) + " before it is written");
        }
        last_use_[s] = ordinal;
      }
      if (in.output < 0 || in.output >= plan_.num_slots || written[in.output]) {
        plan_fail("executor: slot " + std::to_string(in.output) + " written twice or out of range");
      }
      written[in.output] = true;
      ++ordinal;
    }
  }
  step_first_ordinal_.push_back(ordinal);
  for (const auto& o : plan_.outputs) {
    if (o.slot < 0 || o.slot >= plan_.num_slots || !written[o.slot]) plan_fail("executor: output slot never written");
    last_use_[o.slot] = std::numeric_limits<int64_t>::max();
  }
  // device-resident constants; Int32 constants are Utf8 literals
  // (lower_literal, operator_plan.cpp:476-490) and live as STR8
  for (auto& step : plan_.steps) {
    for (auto& in : step.instrs) {
      if (in.op != Op::ConstTensor) continue;
      if (in.const_dtype == TQP_I32) {
        Tensor wide = upload(ctx_, TQP_I32, in.const_rows, in.const_cols, in.const_host.data());
        in.constant = k::utf8_i32_to_str8(ctx_, wide);
      } else {
        in.constant = upload(ctx_, in.const_dtype, in.const_rows, in.const_cols, in.const_host.data());
      }
    }
  }
  ctx_.sync();
  if (flags_ & TQP_EXEC_FUSE) units_ = plan_fusion(ctx_, plan_);
}

std::string Executor::explain() const {
  std::ostringstream os;
  os << "{\"fused\": [";
  for (size_t i = 0; i < units_.size(); ++i) {
    const auto& u = units_[i];
    os << (i ? ", " : "") << "{\"name\": \"" << u.name << "\", \"steps\": [\"" << plan_.steps[u.first_step].id
       << "\", \"" << plan_.steps[u.last_step].id << "\"], \"detail\": \"" << json_escape(u.explain) << "\"}";
  }
  os << "]}";
  return os.str();
}

Tensor Executor::exec_instr(const Instr& in, std::vector<std::optional<Tensor>>& slots, const TableSet& tables) {
  auto arg = [&](size_t i) -> const Tensor& {
    int s = in.inputs.at(i);
    if (!slots[s]) exec_fail("internal: slot " + std::to_string(s) + " read after release");
    return *slots[s];
  };
  Ctx& c = ctx_;
  switch (in.op) {
    case Op::Compare: return k::compare(c, arg(0), arg(1), in.cmp);
    case Op::Arith: return k::arith(c, arg(0), arg(1), in.arith);
    case Op::Logical: return k::logical(c, arg(0), arg(1), in.logic);
    case Op::Not: return k::logical_not(c, arg(0));
    case Op::SelectWhere: return k::select_where(c, arg(0), arg(1), arg(2));
    case Op::PrefixSum: return k::prefix_sum_exclusive(c, arg(0));
    case Op::Compact: return k::compact(c, arg(0), arg(1));
    case Op::ArgsortStable: return k::argsort_stable(c, arg(0));
    case Op::Gather: return k::gather(c, arg(0), arg(1));
    case Op::SearchSorted: return k::searchsorted(c, arg(0), arg(1), in.side);
    case Op::ExpandSegments: return k::expand_segments(c, arg(0), arg(1));
    case Op::SegmentStarts: return k::segment_starts(c, arg(0));
    case Op::SegmentedReduce: {
      int64_t num = in.param;
      if (num < 0) {
        const Tensor& t = arg(2);
        if (t.size() != 1) kernel_fail("tensor: item() requires exactly one element");
        check_i64_access(t);
        num = std::max<int64_t>(0, read_scalar<int64_t>(c, t));
      }
      return k::segmented_reduce(c, arg(0), arg(1), num, in.reduce);
    }
    case Op::MatMul: return k::matmul(c, arg(0), arg(1));
    case Op::SubstringMatch: return k::substring_match(c, arg(0), in.pattern, in.anchor);
    case Op::LoadColumn: {
      const Table* t = bind_table(tables, in.table);
      if (!t) exec_fail("no input table named '" + in.table + "'");
      const Column* col = t->find(in.column);
      if (!col) throw Error(TQP_ERR_ENCODING, "table: no column named '" + in.column + "'");
      if (!col->t.buf && col->t.size() > 0)  // tqp_table_declare_column: bound, never uploaded
        exec_fail("column '" + in.column + "' of table '" + in.table + "' was declared without data");
      return col->t;
    }
    case Op::ConstTensor: return in.constant;
    case Op::IotaRows: {
      int64_t n = arg(0).rows;
      if (in.param >= 0) n = std::min(n, in.param);
      return k::iota(c, n);
    }
    case Op::IotaLen: {
      const Tensor& t = arg(0);
      if (t.size() != 1) kernel_fail("tensor: item() requires exactly one element");
      check_i64_access(t);
      return k::iota(c, read_scalar<int64_t>(c, t));
    }
    case Op::Cast: return k::cast(c, arg(0), in.cast_to);
    case Op::ExpF64: return k::exp_f64(c, arg(0));
    case Op::LastOrZero: return k::last_or_zero(c, arg(0));
    case Op::PackCols: {
      std::vector<Tensor> cols;
      for (size_t i = 0; i < in.inputs.size(); ++i) cols.push_back(arg(i));
      return k::pack_cols(c, cols);
    }
    case Op::BroadcastScalar: return k::broadcast_rows(c, arg(0), arg(1).rows);
    case Op::PadWidthLike: return k::pad_width_like(c, arg(0), arg(1));
    case Op::SortPermRows: return k::sort_perm_rows(c, arg(0), arg(1), in.param == 1);
    case Op::StringCompare: return k::string_compare(c, arg(0), arg(1), in.cmp);
  }
  exec_fail("unknown instruction");
}

void Executor::run_step(int s, std::vector<std::optional<Tensor>>& slots, const TableSet& tables, ProfileTrace* trace,
                        int64_t run_start) {
  const Step& step = plan_.steps[s];
  int64_t ordinal = step_first_ordinal_[s];
  int64_t step_start = now_ns(), step_bytes = 0, rows_out = 0;
  // error checks of this step's instructions may be deferred to one readback
  // at its end (Ctx::check_deferred); a synchronous error first reports any
  // earlier deferred failure, so the first failing instruction always wins
  struct DeferScope {
    Ctx& c;
    explicit DeferScope(Ctx& c_) : c(c_) { c.defer_checks = true; }
    ~DeferScope() {
      c.defer_checks = false;
      c.deferred.clear();
    }
  } defer_scope(ctx_);
  auto wrap = [&](const Error& e) -> Error {
    if (e.code == TQP_ERR_KERNEL || e.code == TQP_ERR_ENCODING) return Error(TQP_ERR_EXEC, step.id + ": " + e.what(), e.bad_row);
    return e;
  };
  for (size_t ii = 0; ii < step.instrs.size(); ++ii) {
    const Instr& in = step.instrs[ii];
    int64_t t0 = now_ns();
    Tensor r;
    try {
      r = exec_instr(in, slots, tables);
      if (trace || ii + 1 == step.instrs.size()) ctx_.check_deferred();
    } catch (const Error& e) {
      try {
        ctx_.check_deferred();
      } catch (const Error& first) {
        throw wrap(first);
      }
      throw wrap(e);
    }
    if (trace) ctx_.sync();
    int64_t t1 = now_ns();
    int64_t bytes = static_cast<int64_t>(r.size()) * (r.dtype == TQP_STR8 ? 4 : static_cast<int64_t>(r.elem_size()));
    rows_out = r.rows;
    step_bytes += bytes;
    if (trace) trace->kernels.push_back({step.id, op_name(in.op), t0 - run_start, t1 - t0, r.rows, bytes});
    slots[in.output] = std::move(r);
    for (int x : in.inputs)
      if (last_use_[x] == ordinal) slots[x].reset();
    ++ordinal;
  }
  if (trace) {
    if (!step.output_slots.empty() && slots[step.output_slots.front()]) rows_out = slots[step.output_slots.front()]->rows;
    trace->operators.push_back({step.id, step.kind, step_start - run_start, now_ns() - step_start, rows_out, step_bytes});
  }
}

void Executor::release_after(int s, std::vector<std::optional<Tensor>>& slots) {
  int64_t last = step_first_ordinal_[s + 1] - 1;
  for (int x = 0; x < plan_.num_slots; ++x)
    if (slots[x] && last_use_[x] <= last) slots[x].reset();
}

void Executor::time_begin(cudaEvent_t* ev) {
  *ev = nullptr;
  if (!timing_) return;
  *ev = ctx_.take_event();
  TQP_CUDA(cudaEventRecord(*ev, ctx_.stream));
}

void Executor::time_end(const std::string& name, cudaEvent_t start) {
  if (!start) return;
  cudaEvent_t stop = ctx_.take_event();
  TQP_CUDA(cudaEventRecord(stop, ctx_.stream));
  timings_[name].pending.push_back({start, stop});
}

void Executor::collect_kernel_events() {
  // kernel events recorded on the shared context during this executor's run
  for (auto& [name, ev] : ctx_.kernel_events) timings_["kernel:" + name].pending.push_back(ev);
  ctx_.kernel_events.clear();
}

void Executor::drain_timings() {
  collect_kernel_events();
  for (auto& [name, t] : timings_) {
    for (auto& [a, b] : t.pending) {
      TQP_CUDA(cudaEventSynchronize(b));
      float ms = 0.f;
      TQP_CUDA(cudaEventElapsedTime(&ms, a, b));
      t.total_ms += ms;
      t.calls += 1;
      ctx_.give_event(a);
      ctx_.give_event(b);
    }
    t.pending.clear();
  }
}

std::string Executor::timings_json() {
  drain_timings();
  std::ostringstream os;
  os << "{";
  bool first = true;
  for (const auto& [name, t] : timings_) {
    os << (first ? "" : ", ") << "\"" << json_escape(name) << "\": {\"calls\": " << t.calls
       << ", \"total_ms\": " << t.total_ms << "}";
    first = false;
  }
  os << "}";
  return os.str();
}

void Executor::reset_timings() {
  drain_timings();
  timings_.clear();
}

void Executor::check_inputs(const TableSet& tables) const {
  // bind and type-check the input tables (executor.cpp:355-371)
  for (const auto& it : plan_.input_tables) {
    const Table* t = bind_table(tables, it.name);
    if (!t) exec_fail("no input table named '" + it.name + "'");
    for (const auto& [cname, ctype] : it.schema) {
      const Column* c = t->find(cname);
      if (!c) exec_fail("input table '" + it.name + "' is missing column '" + cname + "'");
      if (c->type != ctype) {
        exec_fail("input table '" + it.name + "': column '" + cname + "' is " + logical_type_name(c->type) +
                  ", the plan expects " + logical_type_name(ctype));
      }
    }
  }
}

Result Executor::execute(const TableSet& tables, ProfileTrace* trace, bool allow_defer) {
  UnitPending pend;
  Result r = run_units(tables, trace, allow_defer, pend, true);
  if (pend.active) {
    // collect_outputs synchronised: the deferred word is on the host
    long long herr[4];
    std::memcpy(herr, ctx_.h_err + Ctx::kPinnedUnitErr, sizeof(herr));
    if (herr[0] || herr[1]) return execute(tables, trace, false);  // the checked path decides (fallback / 8 slots)
    const long long nrows = pend.nrows >= 0 ? pend.nrows : herr[2];
    for (auto& col : r.cols)
      if (std::find(pend.outs.begin(), pend.outs.end(), col.t.data()) != pend.outs.end()) col.t.rows = nrows;
    check_result_rows(r);
  }
  return r;
}

AsyncResult Executor::execute_async(const TableSet& tables) {
  AsyncResult a;
  a.tables = tables;
  a.slot = ctx_.pinned_slot();
  a.pend.host = a.slot.get();
  a.r = run_units(tables, nullptr, true, a.pend, false);
  if (!a.pend.active) {  // nothing deferred: complete it now
    ctx_.sync();
    if (ctx_.time_kernels) collect_kernel_events();
    check_result_rows(a.r);
    a.complete = true;
    return a;
  }
  TQP_CUDA(cudaEventCreateWithFlags(&a.done, cudaEventDisableTiming));
  TQP_CUDA(cudaEventRecord(a.done, ctx_.stream));
  return a;
}

Result Executor::wait(AsyncResult& a) {
  if (a.complete) return a.r;
  TQP_CUDA(cudaEventSynchronize(a.done));
  cudaEventDestroy(a.done);
  a.done = nullptr;
  if (ctx_.time_kernels) collect_kernel_events();
  long long herr[4];
  std::memcpy(herr, a.slot.get(), sizeof(herr));
  a.complete = true;
  if (herr[0] || herr[1]) {
    a.r = execute(a.tables, nullptr, false);  // the checked path decides (fallback / 8 slots)
    return a.r;
  }
  const long long nrows = a.pend.nrows >= 0 ? a.pend.nrows : herr[2];
  for (auto& col : a.r.cols)
    if (std::find(a.pend.outs.begin(), a.pend.outs.end(), col.t.data()) != a.pend.outs.end()) col.t.rows = nrows;
  check_result_rows(a.r);
  return a.r;
}

// the plan over `tables` up to its outputs; `pend` receives a deferred last
// unit's check, `sync` false leaves the context stream running
Result Executor::run_units(const TableSet& tables, ProfileTrace* trace, bool allow_defer, UnitPending& pend, bool sync) {
  HostProf hp("exec");
  check_inputs(tables);
  hp.mark("inputs");
  // the last fused unit defers its check when only instruction-free steps
  // follow it (its outputs are the result)
  int defer_unit = -1;
  if (allow_defer && !trace && !units_.empty()) {
    const FusedUnit& last = units_.back();
    bool tail_free = true;
    for (size_t q = last.last_step + 1; q < plan_.steps.size(); ++q)
      if (!plan_.steps[q].instrs.empty()) tail_free = false;
    if (tail_free) defer_unit = static_cast<int>(units_.size()) - 1;
  }
  std::vector<std::optional<Tensor>> slots(plan_.num_slots);
  int64_t run_start = now_ns();
  size_t u = 0;
  for (int s = 0; s < static_cast<int>(plan_.steps.size());) {
    if (u < units_.size() && units_[u].first_step == s) {
      const FusedUnit& unit = units_[u++];
      int64_t t0 = now_ns();
      cudaEvent_t ev;
      time_begin(&ev);
      bool ok = unit.run(ctx_, slots, tables, static_cast<int>(u) - 1 == defer_unit ? &pend : nullptr);
      hp.mark("unit");
      if (ok) time_end(unit.name, ev);
      else ctx_.give_event(ev);
      if (!ok) ++fallbacks_;
      if (ok) {
        if (trace) {
          ctx_.sync();
          int64_t t1 = now_ns();
          trace->kernels.push_back({plan_.steps[unit.last_step].id, unit.name, t0 - run_start, t1 - t0, 0, 0});
          for (int q = unit.first_step; q <= unit.last_step; ++q) {
            const Step& st = plan_.steps[q];
            int64_t rows = 0;
            if (!st.output_slots.empty() && slots[st.output_slots.front()]) rows = slots[st.output_slots.front()]->rows;
            trace->operators.push_back({st.id, st.kind, t0 - run_start, t1 - t0, rows, 0});
          }
        }
        release_after(unit.last_step, slots);
        s = unit.last_step + 1;
        continue;
      }
      // preconditions failed on this data: run the covered steps per
      // instruction (still on device)
      for (int q = unit.first_step; q <= unit.last_step; ++q) run_step(q, slots, tables, trace, run_start);
      s = unit.last_step + 1;
      continue;
    }
    cudaEvent_t ev;
    time_begin(&ev);
    run_step(s, slots, tables, trace, run_start);
    time_end("step:" + plan_.steps[s].kind, ev);
    hp.mark("step");
    ++s;
  }
  Result r = collect_outputs(slots, !pend.active && sync, sync);
  hp.mark("collect");
  return r;
}

Result Executor::collect_outputs(std::vector<std::optional<Tensor>>& slots, bool check_rows, bool sync) {
  Result res;
  for (const auto& o : plan_.outputs) {
    if (!slots[o.slot]) exec_fail("internal: slot " + std::to_string(o.slot) + " read after release");
    res.cols.push_back({o.name, o.type, *slots[o.slot]});
  }
  if (check_rows) check_result_rows(res);
  if (!sync) return res;
  ctx_.sync();
  if (ctx_.time_kernels) collect_kernel_events();
  return res;
}

// ---- sharded execution -------------------------------------------------------
bool Executor::shardable(std::string* why) const {
  auto no = [&](const std::string& m) {
    if (why) *why = m;
    return false;
  };
  if (units_.empty() || !units_[0].partial) return no("the plan has no fused scan unit (run unsharded, or with fusion on)");
  const FusedUnit& u = units_[0];
  // steps before the unit only load columns or constants (their slots feed
  // the unit alone); steps after it read the unit's outputs, never a table
  std::set<int> before;
  for (int s = 0; s < u.first_step; ++s) {
    for (const auto& in : plan_.steps[s].instrs) {
      if (in.op != Op::LoadColumn && in.op != Op::ConstTensor) return no("step " + plan_.steps[s].id + " runs before the fused unit");
      before.insert(in.output);
    }
  }
  for (size_t s = u.last_step + 1; s < plan_.steps.size(); ++s) {
    for (const auto& in : plan_.steps[s].instrs) {
      if (in.op == Op::LoadColumn) return no("step " + plan_.steps[s].id + " reads a table after the fused unit");
      for (int x : in.inputs)
        if (before.count(x)) return no("step " + plan_.steps[s].id + " reads a slot loaded before the fused unit");
    }
  }
  for (const auto& o : plan_.outputs)
    if (before.count(o.slot)) return no("a plan output is loaded before the fused unit");
  return true;
}

Partial Executor::execute_partial(const TableSet& tables) {
  std::string why;
  if (!shardable(&why)) exec_fail("plan is not shardable: " + why);
  check_inputs(tables);
  const FusedUnit& u = units_[0];
  cudaEvent_t ev;
  time_begin(&ev);
  Partial p;
  if (!u.partial(ctx_, tables, &p)) {
    ctx_.give_event(ev);
    exec_fail(plan_.steps[u.last_step].id + ": this shard violates the fused path's preconditions "
              "(non-unique or sparse build keys, an int64 overflow, or more than 8 groups per block); "
              "run it unsharded");
  }
  time_end(u.name + ":partial", ev);
  ctx_.sync();
  if (ctx_.time_kernels) collect_kernel_events();
  return p;
}

int ShardEnv::kind_of(const std::string& table) const {
  for (const auto& [name, k] : kinds)
    if (iequals(name, table)) return k;
  return SHARD_REPLICATED;
}

// Every row-shard / co-partitioned table all-gathered to every rank (rank
// order), then the plan runs unsharded: the fallback for plans that do not
// shard and for shards that leave the fused contract.
Result Executor::gather_and_execute(const TableSet& tables, const ShardEnv& env) {
  Comm& comm = *env.comm;
  std::vector<std::shared_ptr<Table>> hold;
  TableSet full;
  for (const auto& [name, t] : tables) {
    if (env.kind_of(name) == SHARD_REPLICATED) {
      full.push_back({name, t});
      continue;
    }
    const std::vector<long long> rows = allgather_host(ctx_, comm, {t->rows});
    long long total = 0, mx = 0;
    for (long long r : rows) {
      total += r;
      mx = std::max(mx, r);
    }
    auto g = std::make_shared<Table>();
    g->rows = total;
    for (const Column& col : t->cols) {
      if (!col.t.buf) {  // declared without data (never loaded): declared here too
        Column nc = col;
        nc.t.rows = total;
        g->cols.push_back(std::move(nc));
        continue;
      }
      const size_t rowb = col.t.elem_size() * static_cast<size_t>(col.t.cols);
      auto pad = ctx_.alloc_bytes(std::max<size_t>(1, rowb * mx));
      auto all = ctx_.alloc_bytes(std::max<size_t>(1, rowb * mx * comm.size));
      if (t->rows) TQP_CUDA(cudaMemcpyAsync(pad->ptr, col.t.data(), rowb * t->rows, cudaMemcpyDeviceToDevice, ctx_.stream));
      comm.allgather(ctx_, pad->ptr, all->ptr, rowb * mx);
      Column nc;
      nc.name = col.name;
      nc.type = col.type;
      nc.t = ctx_.alloc(col.t.dtype, total, col.t.cols);
      long long off = 0;
      for (int r = 0; r < comm.size; ++r) {
        if (rows[r])
          TQP_CUDA(cudaMemcpyAsync(static_cast<char*>(nc.t.data()) + rowb * off, static_cast<char*>(all->ptr) + rowb * mx * r,
                                   rowb * rows[r], cudaMemcpyDeviceToDevice, ctx_.stream));
        off += rows[r];
      }
      g->cols.push_back(std::move(nc));
    }
    hold.push_back(g);
    full.push_back({name, g.get()});
  }
  Result r = execute(full);
  ctx_.sync();
  return r;
}

Result Executor::execute_sharded(const TableSet& tables, const ShardEnv& env) {
  if (!env.comm) throw Error(TQP_ERR_ARG, "execute_sharded: no communicator");
  Comm& comm = *env.comm;
  check_inputs(tables);
  bool any_sharded = false;
  for (const auto& [name, t] : tables) any_sharded = any_sharded || env.kind_of(name) != SHARD_REPLICATED;
  shard_stats_ = "{\"path\": \"unsharded\"}";
  env.bitmap_merges = env.shuffled_tables = env.exchange_bytes = 0;
  if (!any_sharded || comm.size == 1) return execute(tables);
  std::string why;
  bool fact_sharded = false;
  if (shardable(&why)) {
    // the fact table of the unit must be sharded (a replicated fact would be
    // counted once per rank)
    const auto& fus = units_[0];
    for (int s = fus.first_step; s <= fus.last_step && !fact_sharded; ++s)
      for (const auto& in : plan_.steps[s].instrs)
        if (in.op == Op::LoadColumn && env.kind_of(in.table) != SHARD_REPLICATED) fact_sharded = true;
  }
  // phase 1 on every rank, then agree: any rank off the fused path -> gather
  Partial p;
  p.env = &env;
  bool ok = false;
  if (fact_sharded && shardable(&why)) {
    cudaEvent_t ev;
    time_begin(&ev);
    ok = units_[0].partial(ctx_, tables, &p);
    if (ok) time_end(units_[0].name + ":partial", ev);
    else ctx_.give_event(ev);
  }
  const std::vector<long long> oks = allgather_host(ctx_, comm, {ok ? 1LL : 0LL, ok ? p.words : 0LL});
  long long maxw = 0;
  bool all_ok = true;
  for (int r = 0; r < comm.size; ++r) {
    all_ok = all_ok && oks[2 * r] == 1;
    maxw = std::max(maxw, oks[2 * r + 1]);
  }
  auto stats = [&](const char* path) {
    std::ostringstream os;
    os << "{\"path\": \"" << path << "\", \"ranks\": " << comm.size << ", \"bitmap_merges\": " << env.bitmap_merges
       << ", \"shuffled_tables\": " << env.shuffled_tables << ", \"exchange_bytes\": " << env.exchange_bytes << "}";
    shard_stats_ = os.str();
  };
  if (!all_ok) {
    if (fact_sharded && shardable()) ++fallbacks_;
    env.gathered = true;
    stats("gathered");
    return gather_and_execute(tables, env);
  }
  // exchange the partials (padded to the longest), merge on every rank
  auto pad = ctx_.alloc_bytes(sizeof(long long) * maxw);
  auto all = ctx_.alloc_bytes(sizeof(long long) * maxw * comm.size);
  TQP_CUDA(cudaMemcpyAsync(pad->ptr, p.buf->ptr, sizeof(long long) * p.words, cudaMemcpyDeviceToDevice, ctx_.stream));
  comm.allgather(ctx_, pad->ptr, all->ptr, sizeof(long long) * maxw);
  env.exchange_bytes += static_cast<long long>(sizeof(long long) * maxw * comm.size);
  stats("fused");
  std::vector<PartRef> refs;
  for (int r = 0; r < comm.size; ++r)
    refs.push_back({static_cast<const long long*>(all->ptr) + maxw * r, oks[2 * r + 1]});
  try {
    Result res = finish(refs);
    ctx_.sync();
    return res;
  } catch (const Error& e) {
    // merged partials outside the fused contract (e.g. more groups than the
    // merge keeps): every rank sees the same parts, so every rank gathers
    if (std::string(e.what()).find("merged partials violate") == std::string::npos) throw;
    ++fallbacks_;
    stats("gathered");
    return gather_and_execute(tables, env);
  }
}

Result Executor::finish(const std::vector<PartRef>& parts) {
  std::string why;
  if (!shardable(&why)) exec_fail("plan is not shardable: " + why);
  const FusedUnit& u = units_[0];
  std::vector<std::optional<Tensor>> slots(plan_.num_slots);
  cudaEvent_t ev;
  time_begin(&ev);
  u.finish(ctx_, slots, parts);
  time_end(u.name + ":merge", ev);
  int64_t run_start = now_ns();
  for (int s = u.last_step + 1; s < static_cast<int>(plan_.steps.size()); ++s) {
    cudaEvent_t e2;
    time_begin(&e2);
    run_step(s, slots, TableSet{}, nullptr, run_start);
    time_end("step:" + plan_.steps[s].kind, e2);
  }
  return collect_outputs(slots);
}

}  // namespace tqp
