"""Parity report: CUDA path (through the C ABI) vs the fp64 oracle on every
BASELINE config, max abs / max rel (rel floored at 1) errors; JSON to stdout."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import synth
from helpers import gpu_scores, make_gpu, oracle_scores, parity_err, tolerance

cases = [("tiny", synth.preset("tiny"), 1, [0], {}),
         ("tiny-L2-bidir", synth.preset("tiny", L=2, hist_causal=0), 2, [0, 1], {}),
         ("small-fp32", synth.preset("small", dtype="fp32"), 4, [0, 1, 2, 3], {}),
         ("small", synth.preset("small"), 32, [0, 5, 17, 31], {}),
         ("medium", synth.preset("medium"), 16, [0, 7, 15], {}),
         ("large", synth.preset("large"), 4, [0, 3], {"max_wave_pairs": 4000}),
         ("sweep-L2-n512-M100", synth.preset("sweep", L=2, n_k=64, M=100, n_s=1536), 4, [0, 3], {}),
         ("sweep-L4-n8192-M500", synth.preset("sweep", L=4, n_k=1024, M=500, n_s=24576), 2, [0], {})]
out = []
for name, cfg, B, users, kw in cases:
    t0 = time.time()
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 1, B=B)
    cl = make_gpu(cfg, w, B, **kw)
    got = gpu_scores(cl, batch)
    cl.stream_status()
    ref = oracle_scores(cfg, w, batch, users)
    ab = rel = 0.0
    for b, r in ref.items():
        a_, r_ = parity_err(got[batch.cand_offsets[b]:batch.cand_offsets[b + 1]], r)
        ab, rel = max(ab, a_), max(rel, r_)
    cl.close()
    rec = {"config": name, "dtype": cfg.dtype, "users_checked": len(users), "pairs_checked": int(sum(len(v) for v in ref.values())),
           "max_abs": ab, "max_rel": rel, "tol": tolerance(cfg), "pass": ab <= tolerance(cfg) and rel <= tolerance(cfg),
           "seconds": round(time.time() - t0, 1)}
    print(json.dumps(rec), flush=True)
    out.append(rec)
