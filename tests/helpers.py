"""Shared test helpers: run the CUDA path and the oracle on the same seeded inputs."""
import numpy as np

import oracle as O
import synth


def tolerance(cfg):
    """North star: bf16 max abs 2e-2 and max rel 2e-2 (rel floored at 1, G20);
    fp32 verification build 1e-4."""
    return 2e-2 if cfg.dtype == "bf16" else 1e-4


def parity_err(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    ab = np.abs(got - ref)
    return float(ab.max()), float((ab / np.maximum(np.abs(ref), 1.0)).max())


def make_gpu(cfg, w, B, M_max=None, **kw):
    from paper_2502_09888_b200 import Climber, ModelConfig
    mc = ModelConfig.from_any(cfg, M_max=M_max or cfg.M)
    return Climber(mc, w, synth.strategies_for(cfg.N_b, cfg.R), max_users=max(B, 1), **kw)


def to_dev(batch):
    import torch
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t(batch.item), t(batch.action), t(batch.scenario), t(batch.ts), t(batch.cand)


def gpu_scores(cl, batch, release=True):
    import torch
    item, action, scenario, ts, cand = to_dev(batch)
    hs = cl.encode_users(batch.ev_offsets, item, action, scenario, ts, batch.r)
    s = cl.score_batched(hs, batch.cand_offsets, cand)
    torch.cuda.synchronize()
    out = s.cpu().numpy()
    if release:
        cl.release(hs)
        return out
    return out, hs, (item, action, scenario, ts, cand)


def oracle_scores(cfg, w, batch, users=None):
    strats = synth.strategies_for(cfg.N_b, cfg.R)
    users = range(batch.B) if users is None else users
    return {b: O.sumi_scores(cfg, w, strats, batch, b) for b in users}
