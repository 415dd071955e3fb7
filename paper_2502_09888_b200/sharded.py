"""Multi-GPU candidate sharding for one request (latency mode).

The paper's serving statement has one exchange step when a
request is spread over G GPUs: the user's multi-layer K/V cache must reach the
GPUs that score its candidates.  Protocol (one process per GPU, torch.distributed
process group = NCCL over NVLink on a B200 box, gloo in the CPU tests):

  1. the owner rank encodes the user (climber_encode_user) and exports the
     handle's K/V pages into one contiguous device slab (climber_kv_export);
  2. the slab is replicated with one broadcast;
  3. every other rank imports it into its own page pool (climber_kv_import);
  4. candidate m is scored by rank floor(m * G / M) — contiguous shards — and
     the per-rank scores are gathered to the owner.

Every GPU runs the same kernels on its shard, so the gathered scores are
bitwise identical to the 1-GPU scores (candidates are independent: P:L255).
The collective is the process group's; everything else is libclimber.
"""
from __future__ import annotations

import math
from typing import Sequence, Tuple


def shard_bounds(M: int, G: int, rank: int) -> Tuple[int, int]:
    """Candidates [lo, hi) owned by `rank`: exactly the m with floor(m G / M) == rank."""
    lo = -(-rank * M // G)            # ceil(rank * M / G)
    hi = -(-(rank + 1) * M // G)
    return lo, min(hi, M)


class ClimberBackend:
    """libclimber adapter for `rank_request_sharded`."""

    def __init__(self, cl):
        import torch
        self.cl = cl
        self.torch = torch
        self.device = cl.arena.device

    @property
    def slab_bytes(self) -> int:
        return self.cl.slab_bytes

    def encode(self, events, r):
        item, action, scenario, ts = events
        return self.cl.encode_user(item, action, scenario, ts, r)

    def export(self, handle, slab):
        self.cl.kv_export(handle, slab)

    def import_(self, slab, r):
        return self.cl.kv_import(slab, r)

    def score(self, handle, items):
        return self.cl.score_items(handle, items)

    def release(self, handle):
        self.cl.release(handle)


def rank_request_sharded(backend, dist, events, r: int, items, root: int = 0):
    """Score one request's candidates across the process group.

    events: the user's events as `backend.encode` expects (used on `root` only);
    items: the M candidate ids, a tensor on backend.device (every rank).
    Returns the M scores on `root` (a tensor on backend.device), None elsewhere.
    """
    torch = backend.torch
    G, rank = dist.get_world_size(), dist.get_rank()
    M = int(items.numel())
    slab = torch.empty(backend.slab_bytes, dtype=torch.uint8, device=backend.device)
    handle = None
    if rank == root:
        handle = backend.encode(events, r)
        backend.export(handle, slab)
    dist.broadcast(slab, src=root)
    if rank != root:
        handle = backend.import_(slab, r)
    lo, hi = shard_bounds(M, G, rank)
    width = -(-M // G)
    part = torch.full((width,), float("nan"), dtype=torch.float32, device=backend.device)
    if hi > lo:
        part[:hi - lo] = backend.score(handle, items[lo:hi])
    parts = [torch.empty_like(part) for _ in range(G)]
    dist.all_gather(parts, part)
    backend.release(handle)
    if rank != root:
        return None
    out = torch.empty(M, dtype=torch.float32, device=backend.device)
    for g in range(G):
        a, b = shard_bounds(M, G, g)
        out[a:b] = parts[g][:b - a]
    return out
