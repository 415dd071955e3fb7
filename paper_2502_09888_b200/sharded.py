"""Multi-GPU serving of one request (latency mode): candidate sharding
 and block-parallel serving.

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

    # block-parallel
    @property
    def n_blocks(self) -> int:
        return self.cl.cfg.N_b

    def encode_blocks(self, events, r, k0, k1):
        import numpy as np
        item, action, scenario, ts = events
        n = int(item.numel())
        return self.cl.encode_users_blocks(np.array([0, n], np.int64), item, action, scenario, ts,
                                           np.array([r], np.int32), k0, k1)[0]

    def score_blocks(self, handle, items, k0, k1, out=None):
        import numpy as np
        return self.cl.score_blocks([handle], np.array([0, int(items.numel())], np.int64), items, k0, k1, E=out)

    def fuse(self, E_all, r, n_slices):
        import numpy as np
        M = int(E_all.shape[1])
        return self.cl.fuse_scores(np.array([0, M], np.int64), np.array([r], np.int32), E_all, n_slices=n_slices)


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


def rank_request_sharded_lib(cl, dist, events, r: int, items, root: int = 0):
    """Candidate sharding with the K/V replicated by the library itself
    (climber_kv_broadcast: export, ncclBroadcast on the ctx's communicator,
    import) instead of the process group.  `cl` is a Climber created with this
    rank's (rank, world, nccl_uid).  Same return convention as
    rank_request_sharded."""
    torch = cl.torch
    G, rank = dist.get_world_size(), dist.get_rank()
    M = int(items.numel())
    handle = cl.encode_user(*events, r) if rank == root else None
    handle = cl.kv_broadcast(handle, root)
    lo, hi = shard_bounds(M, G, rank)
    width = -(-M // G)
    part = torch.full((width,), float("nan"), dtype=torch.float32, device=items.device)
    if hi > lo:
        part[:hi - lo] = cl.score_items(handle, items[lo:hi])
    parts = [torch.empty_like(part) for _ in range(G)]
    dist.all_gather(parts, part)
    cl.release(handle)
    if rank != root:
        return None
    out = torch.empty(M, dtype=torch.float32, device=items.device)
    for g in range(G):
        a, b = shard_bounds(M, G, g)
        out[a:b] = parts[g][:b - a]
    return out


def rank_request_sharded_pipelined(cl, dist, events, r: int, items, root: int = 0):
    """Candidate sharding with the K/V replicated WHILE it is encoded
    (climber_encode_user_bcast: the root broadcasts each layer's pages as soon
    as its QKV GEMM wrote them, receivers unpack section by section, no host
    sync).  Same return convention as rank_request_sharded."""
    torch = cl.torch
    G, rank = dist.get_world_size(), dist.get_rank()
    M = int(items.numel())
    handle = cl.encode_user_bcast(events if rank == root else None, r, root)
    lo, hi = shard_bounds(M, G, rank)
    width = -(-M // G)
    part = torch.full((width,), float("nan"), dtype=torch.float32, device=items.device)
    if hi > lo:
        part[:hi - lo] = cl.score_items(handle, items[lo:hi])
    parts = [torch.empty_like(part) for _ in range(G)]
    dist.all_gather(parts, part)
    cl.release(handle)
    if rank != root:
        return None
    out = torch.empty(M, dtype=torch.float32, device=items.device)
    for g in range(G):
        a, b = shard_bounds(M, G, g)
        out[a:b] = parts[g][:b - a]
    return out


def rank_request_layered_protocol(backend, dist, events, r: int, items, root: int = 0):
    """The section protocol of climber_encode_user_bcast written against a
    backend (for the gloo tests): the root produces a header section and one
    section per layer, every rank takes part in 1 + L broadcasts in that order,
    receivers rebuild the cache from the sections, then candidates are
    sharded and gathered as in rank_request_sharded."""
    torch = backend.torch
    G, rank = dist.get_world_size(), dist.get_rank()
    M = int(items.numel())
    n_layers, sec_bytes = backend.layered_shape()
    if rank == root:
        handle, sections = backend.encode_layered(events, r)    # [header] + [layer 0 .. L-1]
    else:
        handle, sections = None, [torch.empty(n, dtype=torch.uint8, device=backend.device) for n in sec_bytes]
    for sec in sections:                                         # header first, then layer by layer
        dist.broadcast(sec, src=root)
    if rank != root:
        handle = backend.import_layered(sections, r)
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


# ---------------------------------------------------------------------------
# block-parallel serving ("block-parallel
# KV cache", L203: the N_b blocks are independent until the fusion step)
# ---------------------------------------------------------------------------
def block_bounds(N_b: int, G: int, rank: int) -> Tuple[int, int]:
    """Blocks [k0, k1) of `rank` (G must divide N_b)."""
    if N_b % G:
        raise ValueError(f"G={G} must divide N_b={N_b}")
    n = N_b // G
    return rank * n, (rank + 1) * n


def rank_request_block_parallel(backend, dist, events, r: int, items, root: int = 0):
    """Score one request with its N_b blocks spread over the process group.

    Every rank encodes and scores only its blocks (no K/V moves at all); the
    block outputs E [M][N_b / G][d] are all-gathered rank-major into one
    [G][M][N_b / G][d] buffer, which is exactly the layout the fusion call
    reads; `root` fuses (BGF + head).  events: the user's events on `root`
    (broadcast here, ~14 B per event); items: the M candidates (every rank).
    Returns the M scores on `root`, None elsewhere."""
    torch = backend.torch
    G, rank = dist.get_world_size(), dist.get_rank()
    k0, k1 = block_bounds(backend.n_blocks, G, rank)
    # the request's events reach every rank: one broadcast of n_s, one of the packed arrays
    n = torch.zeros(1, dtype=torch.int64, device=backend.device)
    if rank == root:
        n[0] = int(events[0].numel())
    dist.broadcast(n, src=root)
    n_s = int(n.item())
    packed = torch.empty((4, n_s), dtype=torch.int64, device=backend.device)
    if rank == root:
        for i, a in enumerate(events):
            packed[i] = a.to(torch.int64)
    dist.broadcast(packed, src=root)
    ev = (packed[0].to(torch.int32), packed[1].to(torch.uint8), packed[2].to(torch.uint8), packed[3].contiguous())
    handle = backend.encode_blocks(ev, r, k0, k1)
    E = backend.score_blocks(handle, items, k0, k1)                   # [M][N_b / G][d]
    E_all = torch.empty((G,) + tuple(E.shape), dtype=E.dtype, device=E.device)
    dist.all_gather(list(E_all.unbind(0)), E)
    backend.release(handle)
    if rank != root:
        return None
    return backend.fuse(E_all, r, G)
