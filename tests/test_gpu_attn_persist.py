"""The persistent tcgen05 attention kernel (k_attn_pers, the default without
the relative bias) against the one-tile-per-CTA kernel (k_attn_fa,
CLIMBER_ATTN_PERSIST=0).  History rows do the same arithmetic in the same
order in both; SUMI rows merge the self term at the end in the persistent
kernel instead of starting from it, so the scores agree within the
north-star tolerance (2e-2 abs / rel, rel floored at 1) rather than bit for
bit; the other parity tests bound the default path against the fp64 oracle.
Cases cover d_h 32 and 64, ragged candidate counts (tiles without
candidates, partial tiles), history tiles past v (no keys), blocks with
v_k = 0 (self term only), M = 1, causal and bidirectional history.  A
repeat-launch test checks bitwise reproducibility.  P:L255 (SUMI masks),
Eq. 3 (f_b = 0).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CODE = r"""
import sys, numpy as np
sys.path[:0] = [{root!r}, {tests!r}]
import synth
from helpers import gpu_scores, make_gpu
case = {case!r}
if case == "small":
    cfg = synth.preset("small"); B = 5
    batch = synth.make_batch(cfg, 3, B=B)
elif case in ("medium", "medium_bidir"):
    cfg = synth.preset("medium", hist_causal=0 if case == "medium_bidir" else 1); B = 6
    batch = synth.make_batch(cfg, 4, B=B, M=200)
elif case == "medium_empty":
    cfg = synth.preset("medium"); B = 1
    batch = synth.make_user(cfg, np.random.default_rng(8), n_s=1500, M=1,
                            action_probs=(0.93, 0.0, 0.0, 0.07, 0.0, 0.0))
else:  # large: d_h 64, two candidate tiles + a partial one, ragged candidate counts
    cfg = synth.preset("large", L=2); B = 3
    batch = synth.make_batch(cfg, 5, B=B, M=300)
w = synth.make_weights(cfg, 0)
cl = make_gpu(cfg, w, B)
got = gpu_scores(cl, batch)
cl.stream_status()
np.save({out!r}, got)
"""


def _run(case, persist, tmp_path):
    out = str(tmp_path / f"{case}_{persist}.npy")
    code = _CODE.format(root=ROOT, tests=os.path.join(ROOT, "tests"), case=case, out=out)
    env = dict(os.environ, CLIMBER_ATTN_PERSIST=str(persist))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("case", ["small", "medium", "medium_bidir", "medium_empty", "large"])
def test_persistent_attention_matches_one_tile_kernel(case, tmp_path):
    a = _run(case, 1, tmp_path)
    b = _run(case, 0, tmp_path)
    assert np.all(np.isfinite(a)) and a.shape == b.shape
    ab = np.abs(a.astype(np.float64) - b.astype(np.float64))
    rel = ab / np.maximum(np.abs(b.astype(np.float64)), 1.0)
    assert ab.max() <= 2e-2 and rel.max() <= 2e-2, (case, float(ab.max()), float(rel.max()))


def test_attention_deterministic_across_launches():
    """Identical launches give identical scores (SURVEY §8(b) determinism):
    a `large` wave scored repeatedly on one handle and re-encoded, bit for
    bit (the persistent history kernel in the encode, SUMI in the score)."""
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import synth
    from helpers import make_gpu, to_dev
    cfg = synth.preset("large", L=2)
    B = 16
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 8, B=B)
    cl = make_gpu(cfg, w, B, kv_users=2 * B)
    item, action, scenario, ts, cand = to_dev(batch)
    hs = cl.encode_users(batch.ev_offsets, item, action, scenario, ts, batch.r)
    ref = cl.score_batched(hs, batch.cand_offsets, cand).clone()
    for _ in range(4):
        got = cl.score_batched(hs, batch.cand_offsets, cand)
        assert torch.equal(got, ref), float((got - ref).abs().max())
    h2 = cl.encode_users(batch.ev_offsets, item, action, scenario, ts, batch.r)
    got = cl.score_batched(h2, batch.cand_offsets, cand)
    cl.stream_status()
    assert torch.equal(got, ref), float((got - ref).abs().max())
    cl.release(h2)
    cl.release(hs)
