"""Sharded execution over torch.distributed.

One process per GPU. Every rank holds its shard of the fact table (lineitem,
cut on order boundaries by ``Table.generate(..., shard=r, nshards=N)``);
orders may be co-partitioned the same way or whole, part/customer are whole
(the build sides are small and are rebuilt on each rank from its own copy).

A query is one fused unit over the fact table followed by steps that only read
its outputs (``Executor.shardable()``), so the exchange is one small
all-gather (NCCL over NVLink on GPUs, gloo for the host-logic tests on CPU):

  phase 1  ``Executor.execute_partial(tables)`` on every rank: per-CTA partial
           sums / group tables / touched-group records (a few KB to a few MB)
  exchange ``all_gather_words``: lengths first, then the padded word buffers
  phase 2  ``Executor.finish(parts)`` on every rank, parts in rank order, so
           every rank returns the same result

The reference runs in one process and has no counterpart; the unsharded
equivalent is ``Executor.execute`` (executor.cpp:346).
"""
from __future__ import annotations

from typing import List, Mapping, Optional

import torch
import torch.distributed as dist


def _device_for(group) -> torch.device:
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def all_gather_words(words: Optional[torch.Tensor], group=None) -> List[torch.Tensor]:
    """All-gather variable-length int64 word buffers; returns one tensor per
    rank, in rank order, on the backend's device. ``words=None`` marks a
    rank whose phase 1 failed: every rank then raises (no rank is left
    waiting in a collective)."""
    dev = _device_for(group)
    world = dist.get_world_size(group)
    n = -1 if words is None else int(words.numel())
    lens = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(lens, torch.tensor([n], dtype=torch.int64, device=dev), group=group)
    lens = [int(x.item()) for x in lens]
    bad = [r for r, x in enumerate(lens) if x < 0]
    if bad:
        raise ShardError(bad)
    width = max(1, max(lens))
    buf = torch.zeros(width, dtype=torch.int64, device=dev)
    if n:
        buf[:n] = words.reshape(-1).to(device=dev, dtype=torch.int64)
    out = [torch.empty(width, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    return [o[:x] for o, x in zip(out, lens)]


class ShardError(RuntimeError):
    def __init__(self, ranks):
        super().__init__(f"phase 1 failed on rank(s) {ranks}; the query cannot run sharded")
        self.ranks = ranks


def _words_of(part) -> torch.Tensor:
    if isinstance(part, torch.Tensor):
        return part.reshape(-1)
    if hasattr(part, "__cuda_array_interface__"):
        return torch.as_tensor(part, device="cuda").reshape(-1)
    return torch.as_tensor(part, dtype=torch.int64).reshape(-1)


def execute_sharded(executor, tables: Mapping, group=None):
    """Run ``executor``'s plan over this rank's shard and return the merged
    result of all ranks (identical on every rank)."""
    err = None
    words = None
    part = None
    try:
        part = executor.execute_partial(tables)
        words = _words_of(part)
    except Exception as e:  # noqa: BLE001 - re-raised after the consensus step
        err = e
    try:
        parts = all_gather_words(words, group)
    except ShardError:
        if err is not None:
            raise err
        raise
    if parts and not parts[0].is_cuda and hasattr(executor, "ctx") and torch.cuda.is_available():
        parts = [p.cuda() for p in parts]  # a gloo exchange: the device executor merges device words
    if parts and parts[0].is_cuda:
        torch.cuda.current_stream().synchronize()  # NCCL done before the library stream reads
    del part
    return executor.finish(parts)
