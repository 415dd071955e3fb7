"""Kernel-level mask evidence ("full-visible masks between each
candidate item and the entire history, and also employ diagonal masks for
inter-item isolation"; G1 causal / bidirectional history, G14 self, G15).

`climber_debug_attn_probe` runs the PRODUCTION attention kernels (tcgen05
d_h 32 / 64, mma.sync, fp32 SIMT: whichever the encode / score launch for the
config) on q = k = 0 and one-hot V, so each output channel says whether the
kernel read one particular key.  The mask recovered that way is compared bit
for bit with the oracle's per-pair rule `canonical_mask` (itself pinned by
brute force and closed forms in test_oracle_pins.py).  The candidate-to-
candidate block is checked on its diagonal (the self term); the SUMI kernels
have no operand through which a candidate could read another candidate's K/V.
"""
import numpy as np
import pytest

import oracle as O
import synth
from helpers import make_gpu, to_dev

pytestmark = pytest.mark.gpu


def _bf16(x):
    return float(synth.round_bf16(np.array([x], np.float32))[0])


def kernel_mask(cl, cfg, handle, k, v, M, layer=0):
    """[(n_k + M)]^2 canonical-layout mask of block k recovered from the kernels."""
    nk, dh, H = cfg.n_k, cfg.d_h, cfg.h
    T = nk + M
    first = nk - v
    mask = np.zeros((T, T), np.uint8)
    per = H * (dh - 1)
    for off in range(0, nk, per):
        oh = cl.debug_attn_probe(handle, 0, layer, k, M, off)   # the kernels are layer-agnostic
        os_ = cl.debug_attn_probe(handle, 1, layer, k, M, off)
        for hh in range(H):
            for c in range(dh - 1):
                j = off + hh * (dh - 1) + c
                if j >= nk:
                    break
                col = hh * dh + c
                att_h = oh[:, col] != 0            # history rows (internal slot order)
                att_c = os_[:, col] != 0           # candidate rows
                if j >= v:                         # a pad key must never be read
                    assert not att_h.any() and not att_c.any(), ("pad key attended", k, j, v)
                    continue
                rows = np.nonzero(att_h)[0]
                assert np.all(rows < v), ("pad history row attends", k, rows[rows >= v])
                mask[first + rows, first + j] = 1
                mask[nk + np.nonzero(att_c)[0], first + j] = 1
        selfc = os_[:, [hh * dh + dh - 1 for hh in range(H)]] != 0
        assert np.all(selfc == selfc[:, :1]), "self term differs between heads"
        mask[nk + np.arange(M), nk + np.arange(M)] = selfc[:, 0]
        # weights are uniform over the visible set: every non-zero output of a
        # row is bf16/fp32(1 / |set|) (an extra hidden key would lower them)
        for o in (oh, os_):
            nzr = [np.unique(r[r != 0]) for r in o]
            assert all(len(u) <= 1 for u in nzr), "non-uniform weights on q = k = 0"
    return mask, (oh, os_)


def _check_user(cl, cfg, handle, vlen, M):
    for k in range(cfg.N_b):
        v = int(vlen[k])
        got, (oh, os_) = kernel_mask(cl, cfg, handle, k, v, M)
        ref = O.canonical_mask(v, cfg.n_k, M, cfg.hist_causal)
        assert np.array_equal(got, ref), (cfg.name, k, v, np.argwhere(got != ref)[:8])
        # value check on the last probe: 1/|set| within the output precision
        first = cfg.n_k - v
        cnt_c = ref[cfg.n_k:, :].sum(1)
        dh = cfg.d_h
        selfv = os_[:, dh - 1]
        exp = np.array([_bf16(1.0 / c) if cfg.dtype == "bf16" else 1.0 / c for c in cnt_c])
        np.testing.assert_allclose(selfv, exp, rtol=2 ** -7 if cfg.dtype == "bf16" else 1e-5)
        if v > 0:
            cnt_h = ref[first:cfg.n_k, :].sum(1)
            assert np.all(cnt_h >= 1)


CASES = [
    # name, cfg, B, M, user recipe
    ("tiny_fp32_causal", synth.preset("tiny", L=2), 1, 16),
    ("tiny_fp32_bidir", synth.preset("tiny", L=2, hist_causal=0), 1, 16),
    ("small_bf16", synth.preset("small", B=2), 2, 128),                     # mma.sync history, tcgen05 SUMI d_h 32
    ("medium_bf16_causal", synth.preset("medium", B=2), 2, 300),            # tcgen05 d_h 32, ragged v
    ("medium_bf16_bidir", synth.preset("medium", B=2, hist_causal=0), 2, 300),
    ("large_bf16", synth.preset("large", B=1, L=2, n_s=8192), 1, 1000),     # tcgen05 d_h 64, 8 query tiles, tail 104
]


@pytest.mark.parametrize("name,cfg,B,M", CASES, ids=[c[0] for c in CASES])
def test_kernel_masks_bit_exact(name, cfg, B, M):
    cfg = cfg.replace(M=M)
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 4, B=B, M=M)
    cl = make_gpu(cfg, w, B)
    item, action, scenario, ts, cand = to_dev(batch)
    hs = cl.encode_users(batch.ev_offsets, item, action, scenario, ts, batch.r)
    for b in range(B):
        _, vlen = cl.debug_extract(hs[b])
        _check_user(cl, cfg, hs[b], vlen, M)
    cl.release(hs)
    cl.close()


@pytest.mark.parametrize("causal", [1, 0])
def test_kernel_masks_empty_and_partial_blocks_M1(causal):
    """tcgen05 kernels (medium, d_h 32) on a user whose blocks are empty (v_k = 0),
    short (v_k < 128: one partial query tile) and full, with M = 1 and M = 129
    (one candidate past a tile edge)."""
    cfg = synth.preset("medium", hist_causal=causal)
    w = synth.make_weights(cfg, 0)
    rng = np.random.default_rng(8)
    # actions only 'play_full' and 'like': the {share, comment} and {click}
    # blocks stay empty; 'like' is rare -> a short block
    u = synth.make_user(cfg, rng, n_s=1500, M=129, action_probs=(0.93, 0.0, 0.0, 0.07, 0.0, 0.0))
    cl = make_gpu(cfg, w, 1)
    item, action, scenario, ts, cand = to_dev(u)
    hs = cl.encode_users(u.ev_offsets, item, action, scenario, ts, u.r)
    _, vlen = cl.debug_extract(hs[0])
    assert 0 in vlen and any(0 < v < 128 for v in vlen) and cfg.n_k in vlen, vlen
    for M in (1, 129):
        _check_user(cl, cfg, hs[0], vlen, M)
    cl.release(hs)
    cl.close()
