"""Pins of the oracle's bit-wise gating fusion (BGF, Eq. 4) and
of the scenario indexing of its temperatures.  CPU only.

P:L244: "f_gate represents a squeeze-and-excitation module"; "the
temperature coefficient is solely determined by the recommendation scenario".
Reading G17: f_gate = FC(N_b d -> N_b d / 4) + b, ReLU, FC(-> N_b d) + b,
sigmoid, on vec(G) in block-major order; G16: one fusion ATL with full
visibility among the N_b tokens, temperature tau_f[r][head].

None of these tests re-types the oracle's formula:
  * the fusion ATL + SE + head are rebuilt from torch library modules
    (F.rms_norm, F.scaled_dot_product_attention, nn.Linear, nn.ReLU,
    nn.Sigmoid) on tensors assembled block by block with torch.cat;
  * saturated gates give closed forms (sigma(+40) = 1, sigma(-40) ~ 0, ReLU of
    an all-negative pre-activation = 0) that select single blocks of vec(G);
  * scenario locality: editing another scenario's table leaves scores
    bit-identical, editing the request's scenario changes them.
A dropped ReLU, sigma(-z), swapped SE layers, tau_f[0] in place of tau_f[r],
or a permuted block order in vec(G) fails at least one test here.
"""
import numpy as np
import pytest
import torch
import torch.nn as nn
import torch.nn.functional as Fnn

import oracle as O
import synth


def _t(a):
    return torch.tensor(np.asarray(a, np.float64))


def _torch_fusion_atl(E, w, tau_row, d_h, eps):
    """One pre-norm Transformer layer over the N_b tokens of each candidate
    with full attention (G16); per-head tau applied by scaling the queries so
    SDPA's fixed 1/sqrt(d_h) supplies the rest (G2).  E [M][N_b][d]."""
    X = _t(E)
    Mc, Nb, d = X.shape
    H = d // d_h
    Hn = Fnn.rms_norm(X, (d,), weight=_t(w.f_g1), eps=eps)
    P = Hn @ _t(w.f_w_qkv)
    q, k, v = P[..., :d], P[..., d:2 * d], P[..., 2 * d:]
    heads = lambda z: z.view(Mc, Nb, H, d_h).transpose(1, 2)          # [M][H][N_b][d_h]
    q = heads(q) / _t(tau_row).view(1, H, 1, 1)
    a = Fnn.scaled_dot_product_attention(q, heads(k), heads(v))       # no mask: full visibility
    X = X + a.transpose(1, 2).reshape(Mc, Nb, d) @ _t(w.f_w_o)
    X = X + Fnn.silu(Fnn.rms_norm(X, (d,), weight=_t(w.f_g2), eps=eps) @ _t(w.f_w1)) @ _t(w.f_w2)
    return X


def _torch_se_head(G, w):
    """Squeeze-and-excitation + head from nn modules (G17, G18).  vec(G) is
    assembled explicitly block after block (block-major) with torch.cat."""
    Mc, Nb, d = G.shape
    s = torch.cat([G[:, k, :] for k in range(Nb)], dim=1)             # [M][N_b d]
    fc1 = nn.Linear(Nb * d, w.w_se1.shape[1]).double()
    fc2 = nn.Linear(w.w_se1.shape[1], Nb * d).double()
    head = nn.Linear(Nb * d, 1).double()
    with torch.no_grad():
        fc1.weight.copy_(_t(w.w_se1).T)
        fc1.bias.copy_(_t(w.b_se1))
        fc2.weight.copy_(_t(w.w_se2).T)
        fc2.bias.copy_(_t(w.b_se2))
        head.weight.copy_(_t(w.w_head)[None, :])
        head.bias.copy_(_t(w.b_head))
        gate = nn.Sequential(fc1, nn.ReLU(), fc2, nn.Sigmoid())(s)
        Y = s * gate                                                  # G . sigma(f_gate(G)), Eq. 4
        return Y, head(Y)[:, 0]


def _user(cfg, seed, n_s=150, M=7, r=None):
    u = synth.make_user(cfg, np.random.default_rng(seed), n_s=n_s, M=M, r=r)
    return u


@pytest.mark.parametrize("shape", [dict(N_b=2, d=32, h=2), dict(N_b=4, d=16, h=4)])
def test_bgf_and_head_match_torch_modules(shape):
    """Eq. 4 + head rebuilt from torch modules, at r != 0 with distinct per-
    scenario, per-head tau_f (so tau_f[0] or a head mix-up would differ)."""
    cfg = synth.preset("tiny", L=2, R=4, **shape)
    w = synth.make_weights(cfg, 21)
    # distinct tau_f rows, well apart, so the scenario row matters
    tau_f = np.array([[0.5 + 0.37 * r + 0.11 * h for h in range(cfg.h)] for r in range(cfg.R)], np.float32)
    w = w.scaled(tau_f=synth.round_bf16(tau_f))
    strats = synth.strategies_for(cfg.N_b, cfg.R)
    for r in (1, 3):
        u = _user(cfg, 30 + r, r=r)
        item, action, scenario, ts = u.user_events(0)
        cache = O.encode_user(cfg, w, strats, item, action, scenario, r, ts)
        E = O.block_outputs(cfg, w, cache, u.user_cands(0))
        G = _torch_fusion_atl(E, w, w.tau_f[r], cfg.d_h, cfg.rms_eps)
        Y_ref, s_ref = _torch_se_head(G, w)
        Y = O.bgf(cfg, w, E, r)
        np.testing.assert_allclose(Y.reshape(len(E), -1), Y_ref.numpy(), rtol=0, atol=1e-12)
        np.testing.assert_allclose(O.head(cfg, w, Y), s_ref.numpy(), rtol=0, atol=1e-12)
        # and the whole oracle path agrees with it
        np.testing.assert_allclose(O.sumi_scores(cfg, w, strats, u, 0), s_ref.numpy(), rtol=0, atol=1e-12)
        # the reference really depends on the scenario row: tau_f[0] gives other scores
        G0 = _torch_fusion_atl(E, w, w.tau_f[0], cfg.d_h, cfg.rms_eps)
        assert np.max(np.abs(_torch_se_head(G0, w)[1].numpy() - s_ref.numpy())) > 1e-6


def _identity_fusion(w):
    """f_w_o = 0 and f_w2 = 0: both residual branches of the fusion ATL vanish,
    so G = E exactly (Eq. 4's G(S) = ATL(E(S)) with zero branch outputs)."""
    return w.scaled(f_w_o=np.zeros_like(w.f_w_o), f_w2=np.zeros_like(w.f_w2))


@pytest.mark.parametrize("on_block", [0, 1, 3])
def test_saturated_gate_selects_one_block(on_block):
    """W_se1 = 0 and b_se1 < 0: ReLU(b_se1) = 0, so z = b_se2 whatever W_se2 is
    (a large W_se2 is kept to make a dropped ReLU visible).  b_se2 = +40 on
    block `on_block`'s d entries and -40 elsewhere: sigma = 1 there and
    ~4e-18 elsewhere, so score = b_head + w_head[block] . E[block]."""
    cfg = synth.preset("tiny", L=2, R=4, N_b=4, d=16, h=2)
    w = _identity_fusion(synth.make_weights(cfg, 22))
    d, Nb = cfg.d, cfg.N_b
    rng = np.random.default_rng(5)
    b_se2 = np.full(Nb * d, -40.0, np.float32)
    b_se2[on_block * d:(on_block + 1) * d] = 40.0
    w = w.scaled(w_se1=np.zeros_like(w.w_se1), b_se1=np.full_like(w.b_se1, -1.0),
                 w_se2=synth.round_bf16(rng.standard_normal(w.w_se2.shape).astype(np.float32) * 30),
                 b_se2=b_se2, b_head=np.array([0.25], np.float32))
    strats = synth.strategies_for(Nb, cfg.R)
    u = _user(cfg, 40, r=2)
    item, action, scenario, ts = u.user_events(0)
    cache = O.encode_user(cfg, w, strats, item, action, scenario, 2, ts)
    E = O.block_outputs(cfg, w, cache, u.user_cands(0))
    s = O.score_user(cfg, w, cache, u.user_cands(0))
    wh = np.asarray(w.w_head, np.float64)
    expect = 0.25 + E[:, on_block, :] @ wh[on_block * d:(on_block + 1) * d]
    scale = np.abs(E).max() * np.abs(wh).sum()
    assert np.max(np.abs(s - expect)) < 1e-12 * max(1.0, scale)
    # the other blocks really carry signal: opening all gates changes the score
    w_all = w.scaled(b_se2=np.full(Nb * d, 40.0, np.float32))
    s_all = O.score_user(cfg, w_all, cache, u.user_cands(0))
    expect_all = 0.25 + E.reshape(len(E), -1) @ wh
    assert np.max(np.abs(s_all - expect_all)) < 1e-12 * max(1.0, scale)
    assert np.max(np.abs(s_all - s)) > 1e-3


def test_relu_passes_positive_pre_activation():
    """W_se1 = 0 and b_se1 = c e_j with c > 0 (ReLU is the identity there), so
    z_i = c W_se2[j, i] + b_se2[i].  Row j of W_se2 is chosen so that z = +40
    on block 1 and -40 elsewhere: block 1 alone is selected.
    Together with the previous test (negative pre-activation -> 0) this fixes
    ReLU on both sides of zero."""
    cfg = synth.preset("tiny", L=1, R=2, N_b=2, d=16, h=2)
    w = _identity_fusion(synth.make_weights(cfg, 23))
    d, Nb = cfg.d, cfg.N_b
    Hse = w.w_se1.shape[1]
    c = 2.0
    w_se2 = np.zeros((Hse, Nb * d), np.float32)
    w_se2[3, :] = -40.0 / c
    w_se2[3, d:2 * d] = 40.0 / c
    b_se1 = np.zeros(Hse, np.float32)
    b_se1[3] = c
    w = w.scaled(w_se1=np.zeros_like(w.w_se1), b_se1=b_se1, w_se2=w_se2,
                 b_se2=np.zeros(Nb * d, np.float32), b_head=np.array([0.0], np.float32))
    strats = synth.strategies_for(Nb, cfg.R)
    u = _user(cfg, 41, r=1)
    item, action, scenario, ts = u.user_events(0)
    cache = O.encode_user(cfg, w, strats, item, action, scenario, 1, ts)
    E = O.block_outputs(cfg, w, cache, u.user_cands(0))
    s = O.score_user(cfg, w, cache, u.user_cands(0))
    wh = np.asarray(w.w_head, np.float64)
    expect = E[:, 1, :] @ wh[d:2 * d]
    assert np.max(np.abs(s - expect)) < 1e-12 * max(1.0, np.abs(E).max() * np.abs(wh).sum())


def test_gate_is_half_when_z_is_zero_and_head_reads_block_major():
    """All SE weights and biases 0: sigma(0) = 1/2 exactly, Y = G / 2.  With G = E
    (identity fusion) and w_head = one-hot on element (k, j), the score is
    E[k, j] / 2: the head reads vec(Y) block-major."""
    cfg = synth.preset("tiny", L=2, R=2, N_b=2, d=16, h=2)
    w = _identity_fusion(synth.make_weights(cfg, 24))
    d, Nb = cfg.d, cfg.N_b
    w = w.scaled(w_se1=np.zeros_like(w.w_se1), b_se1=np.zeros_like(w.b_se1),
                 w_se2=np.zeros_like(w.w_se2), b_se2=np.zeros_like(w.b_se2))
    strats = synth.strategies_for(Nb, cfg.R)
    u = _user(cfg, 42, r=0)
    item, action, scenario, ts = u.user_events(0)
    cache = O.encode_user(cfg, w, strats, item, action, scenario, 0, ts)
    E = O.block_outputs(cfg, w, cache, u.user_cands(0))
    for k, j in ((0, 3), (1, 3), (1, 15)):
        wh = np.zeros(Nb * d, np.float32)
        wh[k * d + j] = 1.0
        s = O.score_user(cfg, w.scaled(w_head=wh), cache, u.user_cands(0))
        assert np.array_equal(s, E[:, k, j] / 2)


@pytest.mark.parametrize("table", ["tau_f", "tau"])
def test_temperature_is_indexed_by_the_request_scenario(table):
    """P:L229 / L246: the temperatures depend on the request scenario r.
    Editing every other scenario's entries leaves the scores bit-identical;
    editing scenario r's entries changes them."""
    cfg = synth.preset("tiny", L=2, R=4, h=2)
    w = synth.make_weights(cfg, 25)
    strats = synth.strategies_for(cfg.N_b, cfg.R)
    r = 2
    u = _user(cfg, 43, r=r)
    base = O.sumi_scores(cfg, w, strats, u, 0)
    arr = getattr(w, table).copy()
    others = [x for x in range(cfg.R) if x != r]
    if table == "tau_f":
        arr[others] *= 3.0
    else:
        arr[:, :, others] *= 3.0
    assert np.array_equal(O.sumi_scores(cfg, w.scaled(**{table: arr}), strats, u, 0), base)
    arr2 = getattr(w, table).copy()
    if table == "tau_f":
        arr2[r] *= 3.0
    else:
        arr2[:, :, r] *= 3.0
    assert np.max(np.abs(O.sumi_scores(cfg, w.scaled(**{table: arr2}), strats, u, 0) - base)) > 1e-6


def test_fusion_temperature_scales_the_fusion_logits():
    """(f_W_q head columns -> a f_W_q, tau_f[r][head] -> a tau_f[r][head]) leaves
    the scores unchanged for every a > 0 (the fusion softmax sees
    q.k / (sqrt(d_h) tau_f)), while scaling tau_f alone does not."""
    cfg = synth.preset("tiny", L=1, R=2, h=2)
    w = synth.make_weights(cfg, 26)
    strats = synth.strategies_for(cfg.N_b, cfg.R)
    u = _user(cfg, 44, r=1)
    base = O.sumi_scores(cfg, w, strats, u, 0)
    fq = w.f_w_qkv.astype(np.float64).copy()
    tf = w.tau_f.astype(np.float64).copy()
    dh = cfg.d_h
    a = (4.0, 0.25)
    for hh in range(cfg.h):
        fq[:, hh * dh:(hh + 1) * dh] *= a[hh]
        tf[:, hh] *= a[hh]
    s2 = O.sumi_scores(cfg, w.scaled(f_w_qkv=fq, tau_f=tf), strats, u, 0)
    assert np.max(np.abs(s2 - base)) < 1e-11
    s3 = O.sumi_scores(cfg, w.scaled(tau_f=tf), strats, u, 0)
    assert np.max(np.abs(s3 - base)) > 1e-6
