"""Determinism / block-parallel check at `large` (debug helper): scores of the
same batch encoded + scored twice, and via two block ranges, compared bitwise."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np, torch
import synth
from helpers import make_gpu, to_dev
from paper_2502_09888_b200.sharded import block_bounds
name = sys.argv[1] if len(sys.argv) > 1 else "large"
cfg = synth.preset(name); B = 3; G = 2
w = synth.make_weights(cfg, 0)
batch = synth.make_batch(cfg, 8, B=B)
cl = make_gpu(cfg, w, B, kv_users=B * (G + 2))
item, action, scenario, ts, cand = to_dev(batch)
refs = []
for rep in range(3):
    hs = cl.encode_users(batch.ev_offsets, item, action, scenario, ts, batch.r)
    refs.append(cl.score_batched(hs, batch.cand_offsets, cand).clone())
    if rep == 0:
        h0 = hs
    else:
        cl.release(hs)
for r in refs[1:]:
    print("repeat equal", torch.equal(r, refs[0]), float((r - refs[0]).abs().max()))
# score the same handle again
s2 = cl.score_batched(h0, batch.cand_offsets, cand)
print("rescore equal", torch.equal(s2, refs[0]), float((s2 - refs[0]).abs().max()))
P = int(batch.cand_offsets[-1])
E_all = torch.empty((G, P, cfg.N_b // G, cfg.d), dtype=torch.float32, device=cand.device)
for g in range(G):
    k0, k1 = block_bounds(cfg.N_b, G, g)
    hg = cl.encode_users_blocks(batch.ev_offsets, item, action, scenario, ts, batch.r, k0, k1)
    cl.score_blocks(hg, batch.cand_offsets, cand, k0, k1, E=E_all[g])
got = cl.fuse_scores(batch.cand_offsets, batch.r, E_all, n_slices=G)
cl.stream_status()
d = (got - refs[0]).abs()
print("block-parallel equal", torch.equal(got, refs[0]), float(d.max()), int((d > 0).sum()), "of", d.numel())
