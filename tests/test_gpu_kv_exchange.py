"""K/V slab export/import (the multi-GPU candidate-sharding exchange) on one
GPU: a user encoded in ctx A and imported into ctx B scores bit-identically;
a slab from another config is rejected; the sharded driver runs on a
world-size-1 NCCL group."""
import os
import socket

import numpy as np
import pytest

import synth
from helpers import make_gpu, to_dev

pytestmark = pytest.mark.gpu


def test_export_import_bitwise():
    import torch
    cfg = synth.preset("small")
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 5, B=1)
    a = make_gpu(cfg, w, 1, kv_users=2)
    b = make_gpu(cfg, w, 1, kv_users=2)
    item, action, scenario, ts, cand = to_dev(batch)
    ha = a.encode_user(item, action, scenario, ts, int(batch.r[0]))
    sa = a.score_items(ha, cand).cpu().numpy()
    slab = a.kv_export(ha)
    hb = b.kv_import(slab, int(batch.r[0]))
    sb = b.score_items(hb, cand).cpu().numpy()
    torch.cuda.synchronize()
    a.stream_status()
    b.stream_status()
    assert np.array_equal(sa, sb)
    # the imported cache equals the original page by page
    ia, va = a.debug_extract(ha)
    for k in range(cfg.N_b):
        for l in range(cfg.L):
            Ka, Va = a.debug_kv(ha, l, k, int(va[k]))
            Kb, Vb = b.debug_kv(hb, l, k, int(va[k]))
            assert np.array_equal(Ka, Kb) and np.array_equal(Va, Vb)
    a.release(ha)
    b.release(hb)


def test_slab_from_another_config_is_rejected():
    from paper_2502_09888_b200 import ClimberError
    cfg = synth.preset("small")
    w = synth.make_weights(cfg, 0)
    cl = make_gpu(cfg, w, 1)
    other = make_gpu(synth.preset("small", L=1), synth.make_weights(synth.preset("small", L=1), 0), 1)
    batch = synth.make_batch(cfg, 5, B=1)
    item, action, scenario, ts, cand = to_dev(batch)
    h = other.encode_user(item, action, scenario, ts, int(batch.r[0]))
    slab = other.kv_export(h)
    import torch
    big = torch.zeros(cl.slab_bytes, dtype=torch.uint8, device="cuda")
    big[:slab.numel()] = slab[:big.numel()]
    h2 = cl.kv_import(big, int(batch.r[0]))
    with pytest.raises(ClimberError) as ei:
        cl.stream_status()
    assert ei.value.name == "E_CONFIG"
    cl.release(h2)


def test_sharded_driver_world1_nccl():
    import torch
    import torch.distributed as dist
    from paper_2502_09888_b200.sharded import ClimberBackend, rank_request_sharded
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        cfg = synth.preset("small")
        w = synth.make_weights(cfg, 0)
        batch = synth.make_batch(cfg, 6, B=1)
        cl = make_gpu(cfg, w, 1, kv_users=2)
        item, action, scenario, ts, cand = to_dev(batch)
        out = rank_request_sharded(ClimberBackend(cl), dist, (item, action, scenario, ts), int(batch.r[0]), cand)
        h = cl.encode_user(item, action, scenario, ts, int(batch.r[0]))
        ref = cl.score_items(h, cand)
        assert torch.equal(out, ref)
        cl.release(h)
    finally:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# block-parallel serving (NEXT-2): every block range run in-process, block
# outputs stacked rank-major, fused: bit-identical to the single-GPU path
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,G,rel_bias", [("medium", 2, 0), ("medium", 4, 1), ("large", 2, 0)])
def test_block_parallel_bitwise(name, G, rel_bias):
    import torch
    from paper_2502_09888_b200 import ClimberError
    from paper_2502_09888_b200.sharded import block_bounds
    cfg = synth.preset(name, rel_bias=rel_bias)
    B = 3
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 8, B=B)
    cl = make_gpu(cfg, w, B, kv_users=B * (G + 1))
    item, action, scenario, ts, cand = to_dev(batch)
    hs = cl.encode_users(batch.ev_offsets, item, action, scenario, ts, batch.r)
    ref = cl.score_batched(hs, batch.cand_offsets, cand)
    P = int(batch.cand_offsets[-1])
    E_all = torch.empty((G, P, cfg.N_b // G, cfg.d), dtype=torch.float32, device=cand.device)
    parts = []
    for g in range(G):
        k0, k1 = block_bounds(cfg.N_b, G, g)
        hg = cl.encode_users_blocks(batch.ev_offsets, item, action, scenario, ts, batch.r, k0, k1)
        cl.score_blocks(hg, batch.cand_offsets, cand, k0, k1, E=E_all[g])
        parts.append(hg)
    got = cl.fuse_scores(batch.cand_offsets, batch.r, E_all, n_slices=G)
    cl.stream_status()
    assert torch.equal(got, ref)
    # a partial handle cannot be scored outside its blocks
    with pytest.raises(ClimberError) as ei:
        cl.score_batched(parts[0], batch.cand_offsets, cand)
    assert ei.value.name == "E_INVALID_ARG"
    for hg in parts:
        cl.release(hg)
    cl.release(hs)


def test_block_parallel_driver_world1_nccl():
    import torch
    import torch.distributed as dist
    from paper_2502_09888_b200.sharded import ClimberBackend, rank_request_block_parallel
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        cfg = synth.preset("medium")
        w = synth.make_weights(cfg, 0)
        batch = synth.make_batch(cfg, 6, B=1)
        cl = make_gpu(cfg, w, 1, kv_users=2)
        item, action, scenario, ts, cand = to_dev(batch)
        out = rank_request_block_parallel(ClimberBackend(cl), dist, (item, action, scenario, ts),
                                          int(batch.r[0]), cand)
        h = cl.encode_user(item, action, scenario, ts, int(batch.r[0]))
        ref = cl.score_items(h, cand)
        assert torch.equal(out, ref)
        cl.release(h)
    finally:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# serving cache store (NEXT-4): hits, staleness, LRU eviction, pinning
# ---------------------------------------------------------------------------
def test_cache_store_hits_staleness_and_lru():
    import torch
    from paper_2502_09888_b200 import ClimberError
    cfg = synth.preset("small")
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 9, B=3)
    cl = make_gpu(cfg, w, 3, kv_users=2)           # room for two cached users
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    ev = [tuple(dv(a) for a in batch.user_events(b)) for b in range(3)]
    cands = [dv(batch.user_cands(b)) for b in range(3)]
    def score(h, b):
        return cl.score_items(h, cands[b]).cpu().numpy()

    fresh = []
    for b in range(3):                              # one user at a time (the pool holds two)
        h = cl.encode_user(*ev[b], int(batch.r[b]))
        fresh.append(score(h, b))
        cl.release(h)
    fresh = np.concatenate(fresh)
    off = batch.cand_offsets

    h0, res = cl.cache_acquire(100, int(batch.r[0]), 7, *ev[0])
    assert res == "encoded" and np.array_equal(score(h0, 0), fresh[off[0]:off[1]])
    h0b, res = cl.cache_acquire(100, int(batch.r[0]), 7, *ev[0])
    assert res == "hit" and h0b == h0                               # same K/V, no encode
    cl.cache_release(h0b)
    cl.cache_release(h0)
    h1, res = cl.cache_acquire(101, int(batch.r[1]), 7, *ev[1])
    assert res == "encoded"
    cl.cache_release(h1)
    # a third user: the pool holds two handles -> the LRU unpinned entry (user 100) goes
    h2, res = cl.cache_acquire(102, int(batch.r[2]), 7, *ev[2])
    assert res == "encoded" and np.array_equal(score(h2, 2), fresh[off[2]:off[3]])
    cl.cache_release(h2)
    st = cl.cache_stats()
    assert st["entries"] == 2 and st["evictions"] == 1 and st["hits"] == 1
    # user 101 is still cached; a new digest (the log changed) while the old
    # K/V is pinned builds an uncached handle (evicting the unpinned user 102)
    h1b, res = cl.cache_acquire(101, int(batch.r[1]), 7, *ev[1])
    assert res == "hit"
    h1c, res = cl.cache_acquire(101, int(batch.r[1]), 8, *ev[1])
    assert res == "uncached"
    assert np.array_equal(score(h1c, 1), fresh[off[1]:off[2]])
    cl.cache_release(h1c)
    cl.cache_release(h1b)
    assert cl.cache_stats()["evictions"] == 2
    h2b, res = cl.cache_acquire(102, int(batch.r[2]), 7, *ev[2])
    assert res == "encoded"
    h1d, res = cl.cache_acquire(101, int(batch.r[1]), 8, *ev[1])   # stale, unpinned: rebuilt in place
    assert res == "encoded"
    # every handle pinned -> capacity error, nothing evicted
    with pytest.raises(ClimberError) as ei:
        cl.cache_acquire(100, int(batch.r[0]), 7, *ev[0])
    assert ei.value.name == "E_CAPACITY"
    with pytest.raises(ClimberError):
        cl.cache_release(12345)
    cl.cache_release(h2b)
    cl.cache_release(h1d)
    assert cl.cache_stats()["pinned"] == 0
    cl.stream_status()


@pytest.mark.parametrize("rel_bias", [0, 1])
def test_cache_incremental_append_bitwise(rel_bias):
    # the log grows by appending; only the blocks whose strategy matches an
    # appended event are recomputed, and the scores equal a full re-encode
    import torch
    cfg = synth.preset("medium", rel_bias=rel_bias)      # N_b = 4: {play_full}, {like}, {share, comment}, {click}
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 12, B=1)
    cl = make_gpu(cfg, w, 1, kv_users=3)
    item, action, scenario, ts = (np.array(a) for a in batch.user_events(0))
    r = int(batch.r[0])
    cand = torch.from_numpy(batch.user_cands(0).copy()).cuda()
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    n1 = len(item)
    n0 = n1 - 12
    action = action.copy()
    action[n0:] = synth.A_SKIP                            # matches no strategy

    def fresh(n, act):
        h = cl.encode_user(dv(item[:n]), dv(act[:n]), dv(scenario[:n]), dv(ts[:n]), r)
        s = cl.score_items(h, cand).cpu().numpy()
        cl.release(h)
        return s

    h, res = cl.cache_acquire(7, r, 1000, dv(item[:n0]), dv(action[:n0]), dv(scenario[:n0]), dv(ts[:n0]))
    assert res == "encoded"
    cl.cache_release(h)
    steps = [(n0 + 4, None, 0),                      # only skips appended: no block changes
             (n0 + 8, (n0 + 5, synth.A_LIKE), 1),    # one 'like': block 1 only
             (n1, (n1 - 1, synth.A_PLAY), 1)]        # one 'play_full': block 0 (full -> its window slides)
    dig = 1000
    for n, change, expect in steps:
        if change:
            action[change[0]] = change[1]
        h, res, nb = cl.cache_append(7, r, dig, dig + 1, dv(item[:n]), dv(action[:n]), dv(scenario[:n]),
                                     dv(ts[:n]))
        dig += 1
        assert res == "appended" and nb == expect, (res, nb)
        got = cl.score_items(h, cand).cpu().numpy()
        cl.cache_release(h)
        assert np.array_equal(got, fresh(n, action)), n
    # a digest that is not the cached one falls back to a full build
    h, res, nb = cl.cache_append(7, r, 999, 5000, dv(item), dv(action), dv(scenario), dv(ts))
    assert res == "encoded" and nb == cfg.N_b
    cl.cache_release(h)
    cl.stream_status()


def test_kv_broadcast_in_library_nccl():
    # climber_kv_broadcast over the ctx's own NCCL communicator (world 1 on one
    # GPU): the root keeps its handle; with CLIMBER_DEBUG_BCAST_SELF (a
    # subprocess, the knob is read once) the root also runs the receiver path
    # (export -> ncclBroadcast -> header scenario -> import): bitwise scores
    import subprocess
    import sys
    import torch
    from paper_2502_09888_b200 import nccl_unique_id
    cfg = synth.preset("small")
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 5, B=1)
    cl = make_gpu(cfg, w, 1, kv_users=2, rank=0, world=1, nccl_uid=nccl_unique_id())
    item, action, scenario, ts, cand = to_dev(batch)
    h = cl.encode_user(item, action, scenario, ts, int(batch.r[0]))
    ref = cl.score_items(h, cand)
    assert cl.kv_broadcast(h, root=0) == h
    assert torch.equal(cl.score_items(h, cand), ref)
    cl.release(h)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r"""
import sys, torch; sys.path[:0] = [%r, %r]
import synth
from helpers import make_gpu, to_dev
from paper_2502_09888_b200 import nccl_unique_id
cfg = synth.preset("small"); w = synth.make_weights(cfg, 0); batch = synth.make_batch(cfg, 5, B=1)
cl = make_gpu(cfg, w, 1, kv_users=2, rank=0, world=1, nccl_uid=nccl_unique_id())
item, action, scenario, ts, cand = to_dev(batch)
h = cl.encode_user(item, action, scenario, ts, int(batch.r[0]))
ref = cl.score_items(h, cand)
h2 = cl.kv_broadcast(h, root=0)
assert h2 != h
assert torch.equal(cl.score_items(h2, cand), ref)
cl.stream_status()
print("ok")
""" % (root, os.path.join(root, "tests"))
    env = dict(os.environ, CLIMBER_DEBUG_BCAST_SELF="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_export_import_carries_relative_bias_state():
    # rel_bias = 1 slabs carry the handle's token ages and candidate-row bias
    # (version-2 slab): the imported handle scores bit-identically
    cfg = synth.preset("medium", rel_bias=1)
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 5, B=1)
    a = make_gpu(cfg, w, 1, kv_users=2)
    b = make_gpu(cfg, w, 1, kv_users=2)
    item, action, scenario, ts, cand = to_dev(batch)
    ha = a.encode_user(item, action, scenario, ts, int(batch.r[0]))
    sa = a.score_items(ha, cand).cpu().numpy()
    hb = b.kv_import(a.kv_export(ha), int(batch.r[0]))
    sb = b.score_items(hb, cand).cpu().numpy()
    a.stream_status()
    b.stream_status()
    assert np.array_equal(sa, sb)
    # a ctx without the bias rejects the slab (header flag)
    c0 = synth.preset("medium")
    c = make_gpu(c0, synth.make_weights(c0, 0), 1, kv_users=2)
    import torch
    from paper_2502_09888_b200 import ClimberError
    slab = a.kv_export(ha)
    big = torch.zeros(c.slab_bytes, dtype=torch.uint8, device="cuda")
    big[:] = slab[:big.numel()]
    c.kv_import(big, int(batch.r[0]))
    with pytest.raises(ClimberError) as ei:
        c.stream_status()
    assert ei.value.name == "E_CONFIG"


def test_export_rejects_block_range_handle_and_broadcast_failure_is_symmetric():
    # a block-range handle holds K/V only for its blocks -> export
    # refuses; a failed root export still joins the broadcast (world-1
    # communicator) and the communicator stays usable afterwards
    import torch
    from paper_2502_09888_b200 import ClimberError, nccl_unique_id
    cfg = synth.preset("medium")
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 5, B=1)
    cl = make_gpu(cfg, w, 1, kv_users=3, rank=0, world=1, nccl_uid=nccl_unique_id())
    item, action, scenario, ts, cand = to_dev(batch)
    hp = cl.encode_users_blocks(batch.ev_offsets, item, action, scenario, ts, batch.r, 0, 2)[0]
    with pytest.raises(ClimberError) as ei:
        cl.kv_export(hp)
    assert ei.value.name == "E_INVALID_ARG"
    with pytest.raises(ClimberError) as ei:
        cl.kv_broadcast(hp, root=0)
    assert ei.value.name == "E_INVALID_ARG"
    cl.release([hp])
    with pytest.raises(ClimberError) as ei:
        cl.kv_broadcast(hp, root=0)               # released: stale
    assert ei.value.name == "E_STALE"
    h = cl.encode_user(item, action, scenario, ts, int(batch.r[0]))
    ref = cl.score_items(h, cand)
    assert cl.kv_broadcast(h, root=0) == h        # the communicator still works
    assert torch.equal(cl.score_items(h, cand), ref)
    cl.release(h)
    cl.stream_status()


@pytest.mark.parametrize("name,rel_bias", [("small", 0), ("medium", 1)])
def test_encode_user_bcast_pipelined(name, rel_bias):
    # climber_encode_user_bcast over a world-1 NCCL communicator: the root's
    # handle scores exactly like a plain encode; with CLIMBER_DEBUG_BCAST_SELF
    # (subprocess: the knob is read once) the root also runs the receiver path
    # (header + per-layer unpack from the slab sections) into a second handle,
    # which must score bit-identically
    import subprocess
    import sys
    import torch
    from paper_2502_09888_b200 import nccl_unique_id
    cfg = synth.preset(name, rel_bias=rel_bias)
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 5, B=1)
    cl = make_gpu(cfg, w, 1, kv_users=3, rank=0, world=1, nccl_uid=nccl_unique_id())
    item, action, scenario, ts, cand = to_dev(batch)
    r = int(batch.r[0])
    h = cl.encode_user(item, action, scenario, ts, r)
    ref = cl.score_items(h, cand)
    cl.release(h)
    h2 = cl.encode_user_bcast((item, action, scenario, ts), r, root=0)
    assert torch.equal(cl.score_items(h2, cand), ref)
    cl.release(h2)
    cl.stream_status()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r"""
import sys, torch; sys.path[:0] = [%r, %r]
import synth
from helpers import make_gpu, to_dev
from paper_2502_09888_b200 import nccl_unique_id
cfg = synth.preset(%r, rel_bias=%d); w = synth.make_weights(cfg, 0); batch = synth.make_batch(cfg, 5, B=1)
cl = make_gpu(cfg, w, 1, kv_users=3, rank=0, world=1, nccl_uid=nccl_unique_id())
item, action, scenario, ts, cand = to_dev(batch)
r = int(batch.r[0])
h = cl.encode_user(item, action, scenario, ts, r)
ref = cl.score_items(h, cand)
cl.release(h)
h2 = cl.encode_user_bcast((item, action, scenario, ts), r, root=0)   # the received copy
assert torch.equal(cl.score_items(h2, cand), ref)
cl.stream_status()
print("ok")
""" % (root, os.path.join(root, "tests"), name, rel_bias)
    env = dict(os.environ, CLIMBER_DEBUG_BCAST_SELF="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
