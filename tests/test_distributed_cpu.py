"""Host logic of the sharded path (paper_2209_04579_b200/distributed.py) on
CPU: world_size-2 gloo process group, a stand-in executor whose partials are
plain word buffers. Checks rank order, variable lengths, the empty partial and
the failure consensus (no rank left waiting in a collective)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class FakeExecutor:
    def __init__(self, rank, fail_rank=-1):
        self.rank = rank
        self.fail_rank = fail_rank

    def execute_partial(self, tables):
        if self.rank == self.fail_rank:
            raise RuntimeError("phase 1 failed here")
        n = tables["n"]
        return torch.arange(n, dtype=torch.int64) + 1000 * (self.rank + 1)

    def finish(self, parts):
        return [p.tolist() for p in parts]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    from paper_2209_04579_b200.distributed import ShardError, execute_sharded
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        if case == "lengths":
            out = execute_sharded(FakeExecutor(rank), {"n": [3, 0][rank]})
            q.put((rank, "ok", out))
        elif case == "fail":
            try:
                execute_sharded(FakeExecutor(rank, fail_rank=1), {"n": 2})
                q.put((rank, "no error", None))
            except ShardError as e:
                q.put((rank, "ShardError", e.ranks))
            except RuntimeError as e:
                q.put((rank, "own error", str(e)))
    finally:
        dist.destroy_process_group()


def _run(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, status, val = q.get(timeout=120)
        out[r] = (status, val)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_all_gather_rank_order_and_lengths():
    out = _run("lengths")
    want = [[1000, 1001, 1002], []]
    assert out[0] == ("ok", want)
    assert out[1] == ("ok", want)


def test_phase1_failure_reaches_every_rank():
    out = _run("fail")
    assert out[0] == ("ShardError", [1])
    assert out[1] == ("own error", "phase 1 failed here")
