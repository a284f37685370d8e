"""TQP hot-path benchmark on B200: TPC-H Q1/Q6/Q14/Q3 at SF10 through the
B200 executor (libtqp_b200.so, C ABI), one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--sf 10] [--impl b200|reference]

A step runs the four queries once over device-resident tables (synthetic,
counter-based generator of include/tqp_gen.h, seed 7). value = lineitem rows
scanned per second over the four queries (4 x rows per step / step time).
Inputs per query are 1.9-2.5 GB, far larger than the 126 MB L2, so no L2
flush is needed between steps. `--impl reference` times the reference's own
CPU executor (oracle/_ref/tqp_ref_runner, built from /root/reference's
sources, `par` backend on every host core) on the same configuration (SF10
suite, same generated tables; --ref-sf overrides), with the step count cut to
fit --ref-budget-s if needed.

Extra legs on the b200 line (rank 0, N=1): `cold_first_execution_ms` (each
query's first execution in the process: NVRTC compile included), `q6_sf1`
(BASELINE config 1), `per_instruction` (the suite with fuse=False),
`e2e.encode_once_ms` (host encode of the compressed columnar format).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
METRIC = "TPC-H Q1/Q6/Q14/Q3 rows/s & latency, % HBM roofline, SF10/SF100 at 1-8 B200"
QUERIES = ("q1", "q6", "q14", "q3")
REF_RUNNER = ROOT / "oracle" / "_ref" / "tqp_ref_runner"

# Compulsory input bytes per query: 8 B per Int64/Float64/
# Date value, 1 B per UTF-8 byte; intermediates not credited.
def algorithmic_bytes(q: str, L: int, P: int, O: int, Cn: int) -> int:
    return {
        "q6": 32 * L,
        "q1": 42 * L,
        "q14": 32 * L + 33 * P,
        "q3": 32 * L + 32 * O + 18 * Cn,
    }[q]


# Bytes the fused fact-scan kernel itself must read (the lineitem columns of
# algorithmic_bytes; build sides are read by their own build kernels).
def scan_bytes(q: str, L: int) -> int:
    return {"q6": 32 * L, "q1": 42 * L, "q14": 32 * L, "q3": 32 * L}[q]


def committed_traffic(kernel: str):
    """dram read+write bytes per launch from the committed ncu --set full
    capture summary (profiles/), or None."""
    p = ROOT / "profiles" / "kernel_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return d.get(kernel)


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled (NVML, every 5 ms, plus one sample
    as the timed region starts and one as it ends) during the timed region;
    falls back to nvidia-smi when NVML is unavailable. NVML is initialised
    before the region so the first sample is not lost to its start-up."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self.max_mhz = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._nvml = pynvml
        except Exception:  # noqa: BLE001
            self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            sm = self._nvml.nvmlDeviceGetClockInfo(self._h, self._nvml.NVML_CLOCK_SM)
            rs = self._nvml.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            self.samples.append((sm, rs))
            return
        out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                              "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip().split(",")
        self.max_mhz = float(out[1])
        self.samples.append((float(out[0]), int(out[2], 16)))

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.005 if self._nvml is not None else 0.2)

    def __enter__(self):
        try:
            self._sample()
        except Exception:  # noqa: BLE001
            pass
        self._t.start()
        return self

    def __exit__(self, *a):
        try:
            self._sample()
        except Exception:  # noqa: BLE001
            pass
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        sm = [s[0] for s in self.samples]
        reasons = sorted({name for _, rs in self.samples for name, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples)}


def run_reference(args, rank: int) -> None:
    """Reference arm: the reference's CPU executor (par backend, all cores) on
    the b200 arm's own configuration (the suite at --sf, same generated
    tables). One SF10 step is ~12 s on 16 cores; if K + W steps would exceed
    --ref-budget-s the timed count is reduced (stated in the line)."""
    if rank != 0:
        return
    sample_sf = args.ref_sf
    cores = os.cpu_count() or 1
    if not REF_RUNNER.exists():
        print(json.dumps({"impl": "reference", "unavailable": f"{REF_RUNNER} not built (make -C oracle)"}))
        return
    steps, warmup = args.steps, args.warmup
    # one untimed probe step sizes the run (its table generation included)
    probe = subprocess.run([str(REF_RUNNER), "run", "--sf", str(sample_sf), "--queries", ",".join(QUERIES),
                            "--backend", "par", "--threads", str(cores), "--repeat", "1", "--warmup", "0"],
                           capture_output=True, text=True, check=True).stdout
    probe_ms = sum(json.loads(x)["median_ms"] for x in probe.splitlines() if x.startswith("{"))
    fit = max(2, int(args.ref_budget_s * 1e3 / max(probe_ms, 1.0)))
    if steps + warmup > fit:
        warmup = min(warmup, max(1, fit // 4))
        steps = max(1, fit - warmup)
    cmd = [str(REF_RUNNER), "run", "--sf", str(sample_sf), "--queries", ",".join(QUERIES), "--backend", "par",
           "--threads", str(cores), "--repeat", str(steps), "--warmup", str(warmup)]
    out = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
    lines = [json.loads(x) for x in out.splitlines() if x.startswith("{")]
    per_q = {d["query"]: d for d in lines}
    L = lines[0]["lineitem_rows"]
    step_ms = [sum(per_q[q]["times_ms"][i] for q in QUERIES) for i in range(steps)]
    ms = statistics.median(step_ms)
    value = len(QUERIES) * L / (ms / 1e3)
    same = sample_sf == args.sf
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64+int64", "data": "synthetic",
        "config": {"workload": (f"TPC-H Q1+Q6+Q14+Q3 suite, SF{args.sf:g}" if same else
                                f"TPC-H Q1+Q6+Q14+Q3 suite, SF{args.sf:g} (reference timed on an SF{sample_sf:g} sample)"),
                   "sf": args.sf, "sample_sf": sample_sf, "same_config": same, "queries": list(QUERIES),
                   "lineitem_rows": L, "requested_steps": args.steps, "requested_warmup": args.warmup,
                   "budget_s": args.ref_budget_s},
        "queries": {q: {"latency_ms": per_q[q]["median_ms"], "rows_per_s": L / (per_q[q]["median_ms"] / 1e3)}
                    for q in QUERIES},
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": cores, "kind": "reference",
                         "sample": f"tensql Executor(par, {cores} threads) on SF{sample_sf:g} ({L} lineitem rows), "
                                   f"median of {steps} after {warmup} warmups"},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def cpu_baseline_sample(sf: float):
    """Bounded sample of the reference CPU path for the b200 arm's line."""
    cores = os.cpu_count() or 1
    if not REF_RUNNER.exists():
        return None
    cmd = [str(REF_RUNNER), "run", "--sf", str(sf), "--queries", ",".join(QUERIES), "--backend", "par",
           "--threads", str(cores), "--repeat", "1", "--warmup", "1"]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, check=True, timeout=600).stdout
    except Exception as e:  # noqa: BLE001
        return {"value": None, "unit": "rows/s", "cores": cores, "kind": "reference", "sample": f"failed: {e}"}
    lines = [json.loads(x) for x in out.splitlines() if x.startswith("{")]
    L = lines[0]["lineitem_rows"]
    ms = sum(d["median_ms"] for d in lines)
    return {"value": len(QUERIES) * L / (ms / 1e3), "unit": "rows/s", "cores": cores, "kind": "reference",
            "sample": f"tensql Executor(par, {cores} threads), Q1+Q6+Q14+Q3 on SF{sf:g} ({L} lineitem rows), "
                      f"one timed run after 1 warmup (about 25 s of CPU work at SF10)",
            "queries_ms": {d["query"]: d["median_ms"] for d in lines}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--sf", type=float, default=10.0)
    ap.add_argument("--ref-sf", type=float, default=None, help="reference arm / cpu_baseline SF (default: --sf)")
    ap.add_argument("--ref-budget-s", type=float, default=900.0)
    ap.add_argument("--no-extra", action="store_true", help="skip the cold, Q6@SF1 and per-instruction legs")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-fuse", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-async", action="store_true", help="throughput steps with the synchronous execute()")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-csv", action="store_true")
    ap.add_argument("--csv-sf", type=float, default=1.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    if args.ref_sf is None:
        args.ref_sf = args.sf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    # TQP_BENCH_SHARE_GPU=1: every rank on cuda:0 with a gloo exchange - a
    # functional check of the N-rank flow on a one-GPU box (not a measurement)
    share = os.environ.get("TQP_BENCH_SHARE_GPU") == "1"
    if share:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dist = None
    red_dev = "cuda"
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
            red_dev = "cpu"
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    from paper_2209_04579_b200 import tqp
    ctx = tqp.Context(local_rank)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local_rank))
    seed = 7
    # weak scaling: the dataset is SF(sf x N); lineitem and orders are cut on order
    # boundaries (co-partitioned, so Q3's groups stay on one rank); part and
    # customer are cut by rows (row shards: their build sides are exchanged as
    # presence / flag bitmaps through the library's NCCL communicator). The
    # shared-GPU functional mode keeps them whole (the torch/gloo exchange).
    sharded = ("lineitem", "orders") if share else ("lineitem", "orders", "customer", "part")
    tables = {n: tqp.Table.generate(n, args.sf * world, seed,
                                    shard=rank if n in sharded else 0, nshards=world if n in sharded else 1, ctx=ctx)
              for n in ("lineitem", "orders", "customer", "part")}
    L, O, P, Cn = (tables[n].rows for n in ("lineitem", "orders", "part", "customer"))
    L_total = L
    if dist:
        t = torch.tensor([L], device=red_dev, dtype=torch.int64)
        dist.all_reduce(t)
        L_total = int(t.item())
    execs = {}
    for q in QUERIES:
        plan = json.loads((ROOT / "paper_2209_04579_b200" / "plans" / f"{q}.opplan.json").read_text())
        execs[q] = tqp.Executor(plan, fuse=not args.no_fuse, ctx=ctx)
        # inside the timed region only the fused fact-scan launches carry
        # CUDA events (the roofline kernel); per-query latencies and the
        # per-unit breakdown come from separate passes after it
        execs[q].set_timing("scan")
    comm = None
    if dist and not share:
        # NCCL inside the library (tqp_comm_init_nccl): the unique id travels
        # over torch.distributed, every exchange runs on the library's stream
        uid = [tqp.Comm.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = tqp.Comm.nccl(uid[0], world, rank, ctx)

        def run_query(q, tabs):
            return execs[q].execute_sharded(tabs, comm, tqp.TPCH_SHARD_KINDS)
    elif dist:
        from paper_2209_04579_b200.distributed import execute_sharded

        def run_query(q, tabs):
            return execute_sharded(execs[q], tabs)
    else:
        def run_query(q, tabs):
            return execs[q].execute(tabs)

    # Single GPU: a throughput step submits the four queries with
    # execute_async (the next query's host preparation overlaps the running
    # one) and then takes every result (each checked as execute() checks it);
    # the per-query latencies below are measured with the synchronous
    # execute(), one query at a time.
    pipelined = not dist and not args.no_async

    def step(timing=None):
        if timing is None and pipelined:
            pend = [execs[q].execute_async(tables) for q in QUERIES]
            for p in pend:
                p.result()
            return
        for q in QUERIES:
            if timing is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            run_query(q, tables)
            if timing is not None:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(stream)
                timing[q].append((e0, e1))

    # cold latency: each query's first execution in this process (NVRTC
    # compile of its specialised kernels, key ranges, allocations), wall clock
    cold = {}
    for q in QUERIES:
        ctx.sync()
        t0 = time.perf_counter()
        run_query(q, tables)
        ctx.sync()
        cold[q] = (time.perf_counter() - t0) * 1e3
    for _ in range(args.warmup):
        step()
    for ex in execs.values():
        ex.reset_timings()
    ctx.sync()

    launches0 = ctx.launches
    with ClockSampler(local_rank) as clocks:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ctx.sync()
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for _ in range(args.steps):
            step()
        end.record(stream)
        end.synchronize()
        ctx.sync()
        torch.cuda.synchronize()
    launches = ctx.launches - launches0
    fallbacks = sum(ex.fallbacks for ex in execs.values())
    total_ms = start.elapsed_time(end)
    if dist:
        t = torch.tensor([total_ms], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps

    # roofline of the dominant kernel: largest device time over the timed
    # region among the fused fact-scan kernels (CUDA events recorded by the
    # library on its own stream around each launch)
    peak_gbs, peak_kind = measured_peaks()
    timings = {q: execs[q].timings() for q in QUERIES}
    # per-query latency (events around each query, no library events) and
    # the per-unit device-time breakdown: separate passes, after the timed one
    per_q = {q: [] for q in QUERIES}
    for ex in execs.values():
        ex.set_timing(False)
    for _ in range(args.steps):
        step(per_q)
    q_ms = {q: statistics.median([a.elapsed_time(b) for a, b in per_q[q]]) for q in QUERIES}
    for ex in execs.values():
        ex.set_timing(True)
        ex.reset_timings()
    step()
    ctx.sync()
    units = {q: execs[q].timings() for q in QUERIES}
    for ex in execs.values():
        ex.set_timing(False)
    kern = []
    for q in QUERIES:
        for name, t in timings[q].items():
            if name.startswith("kernel:"):
                kern.append((t["total_ms"], q, name[len("kernel:"):], t["calls"]))
    kern.sort(reverse=True)
    if kern:
        dom_ms, dom_q, dom_name, dom_calls = kern[0]
        dom_avg_ms = dom_ms / max(1, dom_calls)
        dom_bytes = scan_bytes(dom_q, L)
        achieved = dom_bytes / (dom_avg_ms / 1e3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak_gbs, "unit": "GB/s",
                    "frac": achieved / peak_gbs, "traffic": committed_traffic(f"{dom_q}:{dom_name}"),
                    "kernel": f"{dom_q}:{dom_name}", "peak_kind": peak_kind, "bytes_per_launch": dom_bytes,
                    "avg_launch_ms": dom_avg_ms,
                    "all_kernels": {f"{q}:{n}": {"avg_ms": ms / max(1, c),
                                                 "achieved_gbs": scan_bytes(q, L) / (ms / max(1, c) / 1e3) / 1e9}
                                    for ms, q, n, c in kern}}
    else:
        roofline = {"bound": "hbm", "achieved": None, "peak": peak_gbs, "unit": "GB/s", "frac": None,
                    "traffic": None, "kernel": None, "peak_kind": peak_kind}

    rows_total = len(QUERIES) * L_total
    value = rows_total / (ms_per_step / 1e3)
    queries = {}
    for q in QUERIES:
        b = algorithmic_bytes(q, L, P, O, Cn)
        queries[q] = {"latency_ms": q_ms[q], "rows_per_s": L_total / (q_ms[q] / 1e3),
                      "algorithmic_bytes": b, "hbm_frac": b / (q_ms[q] / 1e3) / 1e9 / peak_gbs,
                      "units": units[q], "explain": execs[q].explain()}

    # e2e: host (pinned) columns -> device -> four queries -> result to host
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, tqp, torch, ctx, stream, tables, run_query, L_total, dist, red_dev, encoded=True)
        e2e["raw_layout"] = run_e2e(args, tqp, torch, ctx, stream, tables, run_query, L_total, dist, red_dev,
                                    encoded=False)

    extra = {}
    if rank == 0 and world == 1 and not args.no_extra:
        extra["q6_sf1"] = run_q6_sf1(args, tqp, torch, ctx, stream)
        extra["per_instruction"] = run_per_instruction(args, tqp, torch, ctx, stream, tables, L)
        extra["hash_group"] = run_hash_group(args, tqp, torch, ctx, stream, tables, L)
        extra["dropin_e2e"] = run_dropin_leg()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(args.ref_sf)

    csv_leg = None
    if rank == 0 and not args.no_csv:
        csv_leg = run_csv_leg(tqp, ctx, args.csv_sf)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64+int64", "data": "synthetic (counter-based TPC-H generator, seed 7)",
            "config": {"workload": f"TPC-H Q1+Q6+Q14+Q3 suite, SF{args.sf:g} per GPU (SF{args.sf * world:g} total), device-resident columns",
                       "sf": args.sf, "queries": list(QUERIES), "lineitem_rows_per_gpu": L,
                       "cold_ms": cold,
                       "fused": not args.no_fuse,
                       "submission": ("execute_async x4 then every result (host preparation of the next query "
                                      "overlaps the running one); query latencies with synchronous execute()")
                                     if pipelined else "synchronous execute() per query",
                       "l2": "inputs larger than L2 (1.9-2.5 GB per query vs 126 MB)",
                       "parallelism": ((f"lineitem+orders cut on order boundaries x{world}, part/customer row "
                                        f"shards (build bitmaps all-gathered), partials all-gathered; NCCL in "
                                        f"the library (tqp_executor_execute_sharded)") if world > 1 and not share
                                       else (f"x{world} ranks sharing cuda:0 (functional check, gloo)" if world > 1
                                             else "single GPU"))},
            "queries": queries, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clocks.summary(), "gpu_launches": launches, "fused_fallbacks": fallbacks, "csv_load": csv_leg,
            "shard_stats": {q: execs[q].shard_stats() for q in QUERIES} if comm is not None else None,
            "cold_first_execution_ms": cold,
        }
        line.update(extra)
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def timed_queries(torch, stream, run, queries, steps):
    """median device latency (CUDA events on the library's stream) per query"""
    per = {q: [] for q in queries}
    for _ in range(steps):
        for q in queries:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run(q)
            e1.record(stream)
            per[q].append((e0, e1))
    torch.cuda.synchronize()
    return {q: statistics.median([a.elapsed_time(b) for a, b in v]) for q, v in per.items()}


def run_q6_sf1(args, tqp, torch, ctx, stream):
    """BASELINE.json config 1: TPC-H Q6 at SF1 (6 M lineitem rows), fused,
    device-resident, median of K after W warmups."""
    plan = json.loads((ROOT / "paper_2209_04579_b200" / "plans" / "q6.opplan.json").read_text())
    li = tqp.Table.generate("lineitem", 1.0, 7, ctx=ctx)
    ex = tqp.Executor(plan, ctx=ctx)
    for _ in range(args.warmup):
        ex.execute({"lineitem": li})
    ms = timed_queries(torch, stream, lambda q: ex.execute({"lineitem": li}), ["q6"], max(5, args.steps))["q6"]
    peak, _ = measured_peaks()
    return {"workload": "TPC-H Q6 at SF1 (BASELINE config 1), fused, device-resident", "latency_ms": ms,
            "rows_per_s": li.rows / (ms / 1e3), "algorithmic_bytes": 32 * li.rows,
            "hbm_frac": 32 * li.rows / (ms / 1e3) / 1e9 / peak, "fallbacks": ex.fallbacks}


def run_per_instruction(args, tqp, torch, ctx, stream, tables, L):
    """The per-instruction device path (fuse=False: one kernel family per
    InstrOp, the reference's lowering executed as written - radix sorts,
    compactions, sort joins, segmented reductions) on the same SF tables: the
    path every plan outside the fused contract takes."""
    execs = {}
    for q in QUERIES:
        plan = json.loads((ROOT / "paper_2209_04579_b200" / "plans" / f"{q}.opplan.json").read_text())
        execs[q] = tqp.Executor(plan, fuse=False, ctx=ctx)
    for _ in range(3):  # the pool grows to the path's working set during the first runs
        for q in QUERIES:
            execs[q].execute(tables)
    ctx.sync()
    ms = timed_queries(torch, stream, lambda q: execs[q].execute(tables), list(QUERIES), 5)
    launches0 = ctx.launches
    for q in QUERIES:
        execs[q].execute(tables)
    ctx.sync()
    return {"workload": f"suite per instruction (fuse=False), SF{args.sf:g}", "latency_ms": ms,
            "rows_per_s": {q: L / (v / 1e3) for q, v in ms.items()}, "suite_ms": sum(ms.values()),
            "launches_per_suite": ctx.launches - launches0}


def run_hash_group(args, tqp, torch, ctx, stream, tables, L):
    """queries/qg.sql: GROUP BY l_partkey (200 k groups per SF) with a date
    filter, SUM(price*(1-disc)), SUM(qty), COUNT(*) - the fused hash-group
    unit (direct-address group table, exact Q64.64 limb sums), and the same
    plan per instruction (the reference's sort-based lowering on the device).
    Algorithmic bytes: l_shipdate, l_partkey, l_extendedprice, l_discount,
    l_quantity = 40 B per lineitem row."""
    plan = json.loads((ROOT / "paper_2209_04579_b200" / "plans" / "qg.opplan.json").read_text())
    ex = tqp.Executor(plan, ctx=ctx)
    li = {"lineitem": tables["lineitem"]}
    t0 = time.perf_counter()
    ex.execute(li)
    ctx.sync()
    cold = (time.perf_counter() - t0) * 1e3
    for _ in range(args.warmup):
        ex.execute(li)
    ms = timed_queries(torch, stream, lambda q: ex.execute(li), ["qg"], max(5, args.steps))["qg"]
    ex.set_timing(True)
    ex.reset_timings()
    ex.execute(li)
    ctx.sync()
    units = ex.timings()
    ex.set_timing(False)
    res = ex.execute(li).to_numpy()
    groups = res[0][2].shape[0]
    passing = int(res[-1][2].sum())  # COUNT(*) per group
    nf = tqp.Executor(plan, fuse=False, ctx=ctx)
    nf.execute(li)
    ms_nf = timed_queries(torch, stream, lambda q: nf.execute(li), ["qg"], 3)["qg"]
    peak, _ = measured_peaks()
    b = 40 * L
    kern = {k: v["total_ms"] / max(1, v["calls"]) for k, v in units.items() if k.startswith("kernel:")}
    scan_ms = max(kern.values()) if kern else None
    return {"workload": f"qg: GROUP BY l_partkey, SF{args.sf:g} ({groups} groups), fused hash-group, device-resident",
            "latency_ms": ms, "rows_per_s": L / (ms / 1e3), "algorithmic_bytes": b,
            "hbm_frac": b / (ms / 1e3) / 1e9 / peak, "scan_kernel_ms": scan_ms,
            "scan_kernel_hbm_frac": (b / (scan_ms / 1e3) / 1e9 / peak) if scan_ms else None,
            "units": units, "explain": ex.explain(), "cold_ms": cold, "fallbacks": ex.fallbacks,
            "per_instruction_ms": ms_nf, "speedup_vs_per_instruction": ms_nf / ms,
            # the scan's real bound: per passing row one RED for the group's
            # count, two for revenue (fp64: 2-limb exact sum) and one for
            # sum_qty (int64: one word), against the measured ceiling of
            # random 64-bit REDs (profiles/r2_red_probe.txt)
            "atomic_roofline": ({"bound": "l2_atomics", "reds_per_launch": passing * 4,
                                 "achieved": passing * 4 / (scan_ms / 1e3) / 1e9, "peak": RED_PEAK_GOPS,
                                 "unit": "G RED/s", "frac": passing * 4 / (scan_ms / 1e3) / 1e9 / RED_PEAK_GOPS,
                                 "peak_source": "tools/red_probe.cu on a B200 (profiles/r2_red_probe.txt)"}
                                if scan_ms else None)}


RED_PEAK_GOPS = 188.0  # random 64-bit REDs per second, measured (profiles/r2_red_probe.txt)


def run_dropin_leg(sf: float = 1.0):
    """The path a tensql caller gets, timed from C++ (oracle/tools/
    dropin_bench.cpp): host EncodedTables in the reference's layout ->
    tqp_integration::B200Executor::execute(TableSet) (columns the plan loads,
    page-locked in place once and DMA'd every call; Utf8 narrowed on the host)
    -> EncodedTable, median wall ms per query, beside tensql::Executor (par) on
    the same tables and host cores."""
    exe = ROOT / "oracle" / "_ref" / "tqp_dropin_bench"
    if not exe.exists():
        return {"unavailable": "oracle/_ref/tqp_dropin_bench not built"}
    r = subprocess.run([str(exe), "--sf", str(sf), "--reps", "5"], capture_output=True, text=True, timeout=600)
    if r.returncode != 0:
        return {"error": r.stderr[-500:]}
    d = json.loads(r.stdout.strip().splitlines()[-1])
    d["path"] = ("host EncodedTable (reference layout) -> B200Executor::execute(TableSet): H2D of the loaded columns "
                 "(registered host memory), device run, D2H of the result; wall clock per query")
    return d


def run_csv_leg(tqp, ctx, sf):
    """lineitem as a CSV file -> device table through the
    loader's public call (Table.load_csv: pinned read, one copy to HBM, device
    parse), against the reference's own load_csv (columnar.cpp:521-527, one
    host thread) on the same file. The file is written by the oracle's
    generator (oracle/_ref/csv_cases lineitem)."""
    tool = ROOT / "oracle" / "_ref" / "csv_cases"
    if not tool.exists():
        return {"skipped": "oracle/_ref/csv_cases not built"}
    path = Path(f"/tmp/tqp_bench_lineitem_sf{sf:g}.csv")
    if not path.exists():
        subprocess.run([str(tool), "lineitem", str(sf), str(path)], check=True)
    nbytes = path.stat().st_size
    schema = [("l_orderkey", "int64"), ("l_partkey", "int64"), ("l_quantity", "int64"),
              ("l_extendedprice", "float64"), ("l_discount", "float64"), ("l_tax", "float64"),
              ("l_returnflag", "utf8"), ("l_linestatus", "utf8"), ("l_shipdate", "date")]
    for _ in range(2):
        t = tqp.Table.load_csv(path, schema, ctx=ctx)
    times = []
    for _ in range(5):
        t0 = time.perf_counter()
        t = tqp.Table.load_csv(path, schema, ctx=ctx)
        ctx.sync()
        times.append((time.perf_counter() - t0) * 1e3)
    ms = statistics.median(times)
    rows = t.rows
    ref = subprocess.run([str(tool), "time", str(path), "1"], capture_output=True, text=True, timeout=600)
    ref_ms = json.loads(ref.stdout.strip().splitlines()[-1])["ms"] if ref.returncode == 0 else None
    return {"workload": f"lineitem SF{sf:g} CSV file ({nbytes} B, {rows} rows) -> device table (Table.load_csv)",
            "ms": ms, "rows_per_s": rows / (ms / 1e3), "gb_per_s": nbytes / (ms / 1e3) / 1e9,
            "reference_ms": ref_ms, "reference_rows_per_s": rows / (ref_ms / 1e3) if ref_ms else None,
            "reference": "tensql::load_csv (one host thread), same file"}


def run_e2e(args, tqp, torch, ctx, stream, tables, run_query, L_total, dist, red_dev="cuda", encoded=True):
    """Same suite through the public C ABI with HOST inputs: every step
    uploads the columns from pinned host memory, runs the queries and reads
    the results back; all inside the timed region. encoded: the host columns
    are in the compressed columnar format (tqp_codec_encode, once, when the
    host copy is made - the loader's storage format); each step copies the
    encoded bytes and decodes them on the device (tqp_tensor_from_encoded).
    Otherwise the reference's layout is copied as is (tqp_tensor_from_host)."""
    host = {}
    h2d = 0
    codecs = {}
    encode_s = 0.0
    for name, t in tables.items():
        cols = []
        for cname, lt in t.columns():
            dev = t.column(cname)
            arr = dev.numpy(widen_strings=False)
            if encoded:
                t0 = time.perf_counter()
                codec, payload = tqp.encode_column(arr, dev.dtype)
                encode_s += time.perf_counter() - t0
                pin = torch.from_numpy(payload).pin_memory()
                codecs[f"{name}.{cname}"] = f"{codec.name}{codec.width if codec.name in ('for', 'dec') else ''}"
                cols.append((cname, lt, dev.dtype, arr.shape, codec, pin))
            else:
                pin = torch.from_numpy(arr).pin_memory()
                cols.append((cname, lt, dev.dtype, arr.shape, None, pin))
            h2d += pin.numel() * pin.element_size()
        host[name] = cols

    def upload():
        out = {}
        for name, cols in host.items():
            tab = tqp.Table.create(ctx)
            for cname, lt, dt, shape, codec, pin in cols:
                if codec is not None:
                    # asynchronous: the pinned payloads stay alive and unchanged
                    # (`host`), the copies run back to back on the copy stream
                    # and the queries wait for the decodes on the context stream
                    t = tqp.Tensor.from_encoded(codec, pin, dt, shape[0], shape[1], ctx=ctx, sync=False)
                else:
                    st = tqp.Status()
                    h = tqp.lib.tqp_tensor_from_host(ctx.h, dt, shape[0], shape[1], pin.data_ptr(), tqp.C.byref(st))
                    tqp._check(st, bool(h))
                    t = tqp.Tensor(h, ctx)
                tab.add_column(cname, lt, t)
            out[name] = tab
        return out

    def queries(tabs):
        d2h = 0
        for q in QUERIES:
            res = run_query(q, tabs)
            for _, _, arr in res.to_numpy():
                d2h += arr.nbytes
        return d2h

    def run(steps):
        # every step uploads its own columns; with the encoded format the
        # next step's upload (copy stream + decode stream) is issued before
        # this step's queries run, so the copies overlap them (the queries
        # wait only for their own columns' decodes)
        d2h = 0
        tabs = upload()
        for s in range(steps):
            nxt = upload() if encoded and s + 1 < steps else None
            d2h = queries(tabs)
            tabs = nxt if nxt is not None else (upload() if s + 1 < steps else None)
        return d2h

    run(2)
    if dist:
        dist.barrier()
    ctx.sync()
    t0 = time.perf_counter()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    steps = max(2, args.steps // 2)
    d2h = run(steps)
    end.record(stream)
    end.synchronize()
    wall_ms = (time.perf_counter() - t0) * 1e3
    ev_ms = start.elapsed_time(end)
    ms = max(ev_ms, wall_ms) / steps
    if dist:
        t = torch.tensor([ms], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    out = {"value": len(QUERIES) * L_total / (ms / 1e3), "unit": "rows/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": ms, "steps": steps,
           "device_ms_per_step": ev_ms / steps, "wall_ms_per_step": wall_ms / steps}
    if encoded:
        out["path"] = ("pinned host columns in the compressed columnar format -> tqp_tensor_from_encoded (C ABI: "
                       "H2D of the encoded bytes on the copy stream + decode on the decode stream) -> "
                       "tqp_executor_execute x4 -> results to host; step k+1's upload is issued before step k's "
                       "queries, so its copies overlap them")
        out["codecs"] = codecs
        out["encode_once_ms"] = encode_s * 1e3
        out["encode_note"] = ("host-side encode of every column, done once when the host copy is made (the "
                              "loader's storage format), outside the timed region; tqp_codec_encode on the "
                              "host cores")
    else:
        out["path"] = "pinned host columns (reference layout) -> tqp_tensor_from_host (C ABI) -> tqp_executor_execute x4 -> results to host"
    return out


if __name__ == "__main__":
    main()
