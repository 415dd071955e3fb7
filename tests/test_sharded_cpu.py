"""Candidate sharding + K/V slab exchange protocol (paper_2502_09888_b200.sharded)
with the gloo backend, world_size 2, on CPU.  The per-rank compute is the fp64
oracle behind the same backend interface the libclimber adapter implements;
the gathered scores must equal single-process oracle scores."""
import os
import pickle
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shard_bounds_match_floor_rule():
    from paper_2502_09888_b200.sharded import shard_bounds
    for M in (1, 2, 7, 100, 1000, 1001):
        for G in (1, 2, 3, 4, 8):
            owner = [m * G // M for m in range(M)]
            cover = []
            for g in range(G):
                lo, hi = shard_bounds(M, G, g)
                assert all(owner[m] == g for m in range(lo, hi))
                cover += list(range(lo, hi))
            assert cover == list(range(M))


class OracleBackend:
    """The oracle behind the libclimber adapter's interface (CPU tensors)."""
    SLAB = 1 << 22

    def __init__(self, cfg, w, strats):
        import torch
        self.torch, self.cfg, self.w, self.strats = torch, cfg, w, strats
        self.device = torch.device("cpu")
        self.slab_bytes = self.SLAB

    def encode(self, events, r):
        import oracle as O
        item, action, scenario = events
        return O.encode_user(self.cfg, self.w, self.strats, item, action, scenario, r)

    def export(self, cache, slab):
        blob = pickle.dumps(cache)
        slab[:8] = self.torch.tensor(list(len(blob).to_bytes(8, "little")), dtype=self.torch.uint8)
        slab[8:8 + len(blob)] = self.torch.tensor(list(blob), dtype=self.torch.uint8)

    def import_(self, slab, r):
        n = int.from_bytes(bytes(slab[:8].tolist()), "little")
        return pickle.loads(bytes(slab[8:8 + n].tolist()))

    def score(self, cache, items):
        import oracle as O
        return self.torch.tensor(O.score_user(self.cfg, self.w, cache, items.numpy()), dtype=self.torch.float32)

    def release(self, cache):
        pass


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import synth
    from paper_2502_09888_b200.sharded import rank_request_sharded
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.preset("tiny", L=2, M=7)
    w = synth.make_weights(cfg, 0)
    u = synth.make_user(cfg, np.random.default_rng(3), n_s=120, M=7)
    item, action, scenario, _ = u.user_events(0)
    be = OracleBackend(cfg, w, synth.strategies_for(cfg.N_b, cfg.R))
    events = (item, action, scenario) if rank == 0 else None
    out = rank_request_sharded(be, dist, events, int(u.r[0]), torch.from_numpy(u.user_cands(0)))
    q.put((rank, None if out is None else out.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_candidate_sharding_matches_single_process():
    sys.path.insert(0, ROOT)
    import oracle as O
    import synth
    port = socket.socket()
    port.bind(("127.0.0.1", 0))
    p = port.getsockname()[1]
    port.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, p, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=180) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res[1] is None
    cfg = synth.preset("tiny", L=2, M=7)
    w = synth.make_weights(cfg, 0)
    u = synth.make_user(cfg, np.random.default_rng(3), n_s=120, M=7)
    ref = O.sumi_scores(cfg, w, synth.strategies_for(cfg.N_b, cfg.R), u, 0)
    np.testing.assert_allclose(res[0], ref, rtol=0, atol=1e-6)   # fp32 transport of fp64 scores


# ---------------------------------------------------------------------------
# block-parallel serving (NEXT-2): blocks [k0, k1) per rank, E all-gathered
# ---------------------------------------------------------------------------
def test_block_bounds():
    from paper_2502_09888_b200.sharded import block_bounds
    for N_b in (1, 2, 4, 8):
        for G in (1, 2, 4, 8):
            if N_b % G:
                with pytest.raises(ValueError):
                    block_bounds(N_b, G, 0)
                continue
            cover = []
            for g in range(G):
                k0, k1 = block_bounds(N_b, G, g)
                cover += list(range(k0, k1))
            assert cover == list(range(N_b))


class OracleBlockBackend:
    """The oracle behind the block-parallel interface: block outputs E(S_k)
    of the rank's blocks only, fusion = BGF + head."""

    def __init__(self, cfg, w, strats):
        import torch
        self.torch, self.cfg, self.w, self.strats = torch, cfg, w, strats
        self.device = torch.device("cpu")
        self.n_blocks = cfg.N_b

    def encode_blocks(self, events, r, k0, k1):
        import oracle as O
        item, action, scenario, ts = (a.numpy() for a in events)
        return (O.encode_user(self.cfg, self.w, self.strats, item, action, scenario, r, ts), k0, k1)

    def score_blocks(self, handle, items, k0, k1):
        import oracle as O
        cache, a, b = handle
        assert (a, b) == (k0, k1)
        E = O.block_outputs(self.cfg, self.w, cache, items.numpy())
        return self.torch.tensor(E[:, k0:k1, :], dtype=self.torch.float64).contiguous()

    def fuse(self, E_all, r, n_slices):
        import oracle as O
        G, M, nb, d = E_all.shape
        E = E_all.permute(1, 0, 2, 3).reshape(M, G * nb, d).numpy()
        return self.torch.tensor(O.head(self.cfg, self.w, O.bgf(self.cfg, self.w, E, r)))

    def release(self, handle):
        pass


def _block_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import synth
    from paper_2502_09888_b200.sharded import rank_request_block_parallel
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.preset("tiny", N_b=4, L=2, M=5, rel_bias=1)
    w = synth.make_weights(cfg, 1)
    u = synth.make_user(cfg, np.random.default_rng(4), n_s=150, M=5)
    item, action, scenario, ts = u.user_events(0)
    be = OracleBlockBackend(cfg, w, synth.strategies_for(cfg.N_b, cfg.R))
    t = torch.from_numpy
    events = (t(item), t(action), t(scenario), t(ts)) if rank == 0 else None
    out = rank_request_block_parallel(be, dist, events, int(u.r[0]), torch.from_numpy(u.user_cands(0)))
    q.put((rank, None if out is None else out.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_block_parallel_matches_single_process():
    sys.path.insert(0, ROOT)
    import oracle as O
    import synth
    port = socket.socket()
    port.bind(("127.0.0.1", 0))
    p = port.getsockname()[1]
    port.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_block_worker, args=(r, 2, p, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=180) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res[1] is None
    cfg = synth.preset("tiny", N_b=4, L=2, M=5, rel_bias=1)
    w = synth.make_weights(cfg, 1)
    u = synth.make_user(cfg, np.random.default_rng(4), n_s=150, M=5)
    ref = O.sumi_scores(cfg, w, synth.strategies_for(cfg.N_b, cfg.R), u, 0)
    np.testing.assert_allclose(res[0], ref, rtol=0, atol=1e-12)     # fp64 transport: exact


# ---------------------------------------------------------------------------
# the section protocol of climber_encode_user_bcast (header, then one section
# per layer, 1 + L broadcasts in that order) with the oracle behind it
# ---------------------------------------------------------------------------
class OracleLayeredBackend(OracleBackend):
    """Sections as length-prefixed pickles: the header carries the extraction
    result, request scenario and times; layer section l the K/V of layer l of
    every block (the library's layout: [N_b][pages] of layer l)."""
    SEC = 1 << 20

    def layered_shape(self):
        return self.cfg.L, [self.SEC] * (1 + self.cfg.L)

    def _pack(self, obj):
        blob = pickle.dumps(obj)
        t = self.torch.zeros(self.SEC, dtype=self.torch.uint8)
        t[:8] = self.torch.tensor(list(len(blob).to_bytes(8, "little")), dtype=self.torch.uint8)
        t[8:8 + len(blob)] = self.torch.tensor(list(blob), dtype=self.torch.uint8)
        return t

    def _unpack(self, t):
        n = int.from_bytes(bytes(t[:8].tolist()), "little")
        return pickle.loads(bytes(t[8:8 + n].tolist()))

    def encode_layered(self, events, r):
        cache = self.encode(events, r)
        head = self._pack((cache.idx, cache.vlen, cache.r, cache.t_hist, cache.t_req))
        layers = [self._pack([(cache.K[k][l], cache.V[k][l]) for k in range(self.cfg.N_b)])
                  for l in range(self.cfg.L)]
        return cache, [head] + layers

    def import_layered(self, sections, r):
        import oracle as O
        idx, vlen, rr, t_hist, t_req = self._unpack(sections[0])
        assert rr == r
        per_layer = [self._unpack(s) for s in sections[1:]]
        K = [[per_layer[l][k][0] for l in range(self.cfg.L)] for k in range(self.cfg.N_b)]
        V = [[per_layer[l][k][1] for l in range(self.cfg.L)] for k in range(self.cfg.N_b)]
        return O.Cache(idx, vlen, K, V, rr, t_hist, t_req)


def _layered_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import synth
    from paper_2502_09888_b200.sharded import rank_request_layered_protocol
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.preset("tiny", L=3, M=9)
    w = synth.make_weights(cfg, 2)
    u = synth.make_user(cfg, np.random.default_rng(5), n_s=130, M=9)
    item, action, scenario, _ = u.user_events(0)
    be = OracleLayeredBackend(cfg, w, synth.strategies_for(cfg.N_b, cfg.R))
    events = (item, action, scenario) if rank == 0 else None
    out = rank_request_layered_protocol(be, dist, events, int(u.r[0]), torch.from_numpy(u.user_cands(0)))
    q.put((rank, None if out is None else out.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_layered_replication_protocol():
    sys.path.insert(0, ROOT)
    import oracle as O
    import synth
    port = socket.socket()
    port.bind(("127.0.0.1", 0))
    p = port.getsockname()[1]
    port.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_layered_worker, args=(r, 2, p, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=180) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res[1] is None
    cfg = synth.preset("tiny", L=3, M=9)
    w = synth.make_weights(cfg, 2)
    u = synth.make_user(cfg, np.random.default_rng(5), n_s=130, M=9)
    ref = O.sumi_scores(cfg, w, synth.strategies_for(cfg.N_b, cfg.R), u, 0)
    np.testing.assert_allclose(res[0], ref, rtol=0, atol=1e-6)   # fp32 transport of fp64 scores
