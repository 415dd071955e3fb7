"""Pins of the fp64 oracle against what the paper and mathematics fix
(SURVEY.md §8(c) "What pins each part").  CPU only.

Each test names the passage it follows.  None of them re-types the oracle's
formula: they use hand-derived closed forms (tests/golden), brute force,
invariants, special cases that reduce to a library routine (torch SDPA), or
exact equivalences between independently structured code paths.
"""
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as Fnn

import oracle as O
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.txt")


def _golden():
    rows = {}
    for line in open(GOLD):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        name, tau, a, b = line.split()
        rows.setdefault(name, []).append((float(tau), float(a), float(b)))
    return rows


# ---------------------------------------------------------------------------
# worked examples W1-W3 (closed forms; Eq. 3 with G2/G14)
# ---------------------------------------------------------------------------
def test_w1_candidate_attention_closed_form():
    K = np.array([[1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])   # k1, k2, k_self
    V = np.array([[1.0, 0.0], [0.0, 1.0], [0.0, 0.0]])   # v1, v2, v_self
    q = np.array([[2.0, 0.0]])
    for tau, o0, o1 in _golden()["W1"]:
        o = O.attention(q, K, V, [tau], 2)[0]
        assert abs(o[0] - o0) < 1e-14 and abs(o[1] - o1) < 1e-14


def test_w3_causal_history_row():
    K = np.array([[1.0, 0.0], [0.0, 1.0]])
    V = np.array([[1.0, 0.0], [0.0, 1.0]])
    Q = np.array([[5.0, -3.0], [0.0, 2.0]])
    mask = np.tril(np.ones((2, 2), bool))
    (tau, p1, p2), = _golden()["W3"]
    o = O.attention(Q, K, V, [tau], 2, mask)
    assert abs(o[1, 0] - p1) < 1e-14 and abs(o[1, 1] - p2) < 1e-14
    assert np.array_equal(o[0], V[0])   # row 1 sees only itself


def test_w2_rmsnorm():
    (_, a, b), = _golden()["W2"]
    y = O.rmsnorm(np.array([3.0, 4.0]), np.ones(2), 0.0)
    assert abs(y[0] - a) < 1e-15 and abs(y[1] - b) < 1e-15


# ---------------------------------------------------------------------------
# softmax with temperature (Eq. 3)
# ---------------------------------------------------------------------------
def _entropy(p):
    p = p[p > 0]
    return -np.sum(p * np.log(p))


def test_softmax_invariants():
    rng = np.random.default_rng(0)
    for _ in range(100):
        z = rng.standard_normal(7) * 3
        for tau in (0.5, 1.0, 2.0, 4.0):
            p = O.softmax_tau(z, tau)
            assert abs(p.sum() - 1) < 1e-12
            assert np.allclose(O.softmax_tau(z + 11.5, tau), p, atol=1e-14, rtol=0)
        ents = [_entropy(O.softmax_tau(z, t)) for t in (0.5, 1.0, 2.0, 4.0)]
        assert all(a < b for a, b in zip(ents, ents[1:]))
        assert np.allclose(O.softmax_tau(z, 1e9), np.full(7, 1 / 7), atol=1e-8)
        p0 = O.softmax_tau(z, 1e-6)
        assert p0[np.argmax(z)] > 1 - 1e-9
    assert np.array_equal(O.softmax_tau(np.zeros(2), 1.0), np.array([0.5, 0.5]))


# ---------------------------------------------------------------------------
# extraction (Eq. 2; G11)
# ---------------------------------------------------------------------------
def _bf_extract(action, scenario, strat, n_k):
    amask, smask = strat
    matches = [i for i in range(len(action))
               if (amask >> int(action[i])) & 1 and (smask >> int(scenario[i])) & 1]
    return matches[-n_k:] if n_k > 0 else []


def test_extract_brute_force_and_invariants():
    rng = np.random.default_rng(1)
    for trial in range(60):
        n_s = int(rng.integers(0, 300))
        R = int(rng.integers(1, 5))
        action = rng.integers(0, 6, n_s).astype(np.uint8)
        scenario = rng.integers(0, R, n_s).astype(np.uint8)
        n_k = int(rng.integers(1, 40))
        strats = [(int(rng.integers(0, 64)), int(rng.integers(0, 1 << R))) for _ in range(4)]
        idx, vlen = O.extract(action, scenario, strats, n_k)
        for k, st in enumerate(strats):
            ref = _bf_extract(action, scenario, st, n_k)
            assert vlen[k] == len(ref)
            assert list(idx[k, n_k - vlen[k]:]) == ref
            assert np.all(idx[k, :n_k - vlen[k]] == -1)
            # order preservation: strictly increasing event indices (subsequence of S)
            assert all(a < b for a, b in zip(ref, ref[1:]))
            # monotonicity under filter enlargement
            big = (st[0] | (1 << int(rng.integers(0, 6))), st[1])
            _, vb = O.extract(action, scenario, [big], n_k)
            assert vb[0] >= vlen[k]
            # idempotence: extracting from the extracted sequence gives it back
            sub = np.array(ref, dtype=np.int64)
            idx2, v2 = O.extract(action[sub], scenario[sub], [st], n_k)
            assert v2[0] == len(ref) and list(sub[idx2[0, n_k - v2[0]:]]) == ref


def test_extract_special_cases():
    rng = np.random.default_rng(2)
    n_s = 50
    action = rng.integers(0, 6, n_s).astype(np.uint8)
    scenario = rng.integers(0, 2, n_s).astype(np.uint8)
    # identity: all actions/scenarios, budget >= n_s
    idx, v = O.extract(action, scenario, [(63, 3)], 64)
    assert v[0] == n_s and list(idx[0, 64 - n_s:]) == list(range(n_s))
    # empty match -> v = 0, all pad
    a2 = np.zeros(n_s, np.uint8)
    idx, v = O.extract(a2, scenario, [(1 << synth.A_LIKE, 3)], 8)
    assert v[0] == 0 and np.all(idx == -1)
    # disjoint filters share no events
    idx, v = O.extract(action, scenario, [(0b000011, 3), (0b111100, 3)], 64)
    s0 = set(idx[0][idx[0] >= 0])
    s1 = set(idx[1][idx[1] >= 0])
    assert not (s0 & s1) and len(s0) + len(s1) == n_s


# ---------------------------------------------------------------------------
# SUMI masks
# ---------------------------------------------------------------------------
def test_mask_closed_forms():
    m = O.canonical_mask(2, 2, 1)
    # candidate row attends to {h1, h2, self}
    assert list(m[2]) == [1, 1, 1]
    for v, n_k, M in [(0, 4, 3), (3, 5, 4), (5, 5, 1), (7, 8, 6)]:
        for causal in (1, 0):
            mk = O.canonical_mask(v, n_k, M, causal)
            hist_pairs = v * (v + 1) // 2 if causal else v * v
            assert int(mk.sum()) == hist_pairs + M * (v + 1)
            assert np.array_equal(mk[n_k:, n_k:], np.eye(M, dtype=np.uint8))
            assert mk[:n_k, n_k:].sum() == 0                      # history never sees items
            assert mk[:n_k - v].sum() == 0 and mk[:, :n_k - v].sum() == 0   # pads


# ---------------------------------------------------------------------------
# reduction to a standard pre-norm causal Transformer (north star; S:L541 #4)
# using library routines only: F.rms_norm, F.scaled_dot_product_attention, F.silu
# ---------------------------------------------------------------------------
def _torch_block(X, w, k, tau_rows, d_h, eps, causal=True):
    """Standard pre-norm Transformer on X [T][d]; tau applied by scaling each
    head's queries (so per-head tau is checked against SDPA's fixed 1/sqrt(d_h))."""
    X = torch.tensor(X, dtype=torch.float64)
    T, d = X.shape
    H = d // d_h
    L = w.w_qkv.shape[1]
    for l in range(L):
        t = lambda a: torch.tensor(np.asarray(a, np.float64))
        g1, wqkv, wo, g2, w1, w2 = (t(getattr(w, n)[k, l]) for n in ("g1", "w_qkv", "w_o", "g2", "w1", "w2"))
        Hn = Fnn.rms_norm(X, (d,), weight=g1, eps=eps)
        P = Hn @ wqkv
        q, kk, v = P[:, :d], P[:, d:2 * d], P[:, 2 * d:]
        q = q.view(T, H, d_h).transpose(0, 1) / t(tau_rows[l]).view(H, 1, 1)
        kk = kk.view(T, H, d_h).transpose(0, 1)
        v = v.view(T, H, d_h).transpose(0, 1)
        if causal:
            a = Fnn.scaled_dot_product_attention(q[None], kk[None], v[None], is_causal=True)[0]
        else:
            msk = torch.ones(T, T, dtype=torch.bool)
            msk[:T - 1, T - 1] = False
            a = Fnn.scaled_dot_product_attention(q[None], kk[None], v[None], attn_mask=msk)[0]
        X = X + a.transpose(0, 1).reshape(T, d) @ wo
        X = X + Fnn.silu(Fnn.rms_norm(X, (d,), weight=g2, eps=eps) @ w1) @ w2
    return X.numpy()


@pytest.mark.parametrize("causal", [1, 0])
@pytest.mark.parametrize("unit_tau", [True, False])
def test_reduces_to_standard_transformer(causal, unit_tau):
    cfg = synth.preset("tiny", N_b=1, n_k=64, L=2, hist_causal=causal)
    w = synth.make_weights(cfg, 5)
    if unit_tau:
        w = w.scaled(tau=np.ones_like(w.tau))
    strats = synth.strategies_for(1, cfg.R)
    rng = np.random.default_rng(3)
    u = synth.make_user(cfg, rng, n_s=40, M=5)
    item, action, scenario, _ = u.user_events(0)
    r = int(u.r[0])
    cache = O.encode_user(cfg, w, strats, item, action, scenario, r)
    assert cache.vlen[0] == 40                               # identity extraction
    E = O.block_outputs(cfg, w, cache, u.user_cands(0))
    for m, c in enumerate(u.user_cands(0)):
        X = np.vstack([np.asarray(w.emb_item[item], np.float64) + w.emb_act[action] + w.emb_scn[scenario],
                       np.asarray(w.emb_item[c], np.float64) + w.emb_scn[r]])
        ref = _torch_block(X, w, 0, w.tau[:, 0, r, :], cfg.d_h, cfg.rms_eps, causal=bool(causal))
        np.testing.assert_allclose(E[m, 0], ref[-1], rtol=0, atol=1e-11)


# ---------------------------------------------------------------------------
# SUMI with cache == brute force, each item appended alone (north star; S:L538 #1)
# ---------------------------------------------------------------------------
def test_sumi_equals_brute_force_many_triples():
    rng = np.random.default_rng(11)
    n_trip = 0
    shapes = [dict(N_b=2, n_k=8, L=2, d=16, h=2), dict(N_b=1, n_k=12, L=1, d=16, h=4),
              dict(N_b=4, n_k=6, L=3, d=8, h=2), dict(N_b=2, n_k=16, L=2, d=32, h=2)]
    for si, sh in enumerate(shapes):
        for causal in (1, 0):
            cfg = synth.preset("tiny", V=200, M=4, hist_causal=causal, **sh)
            w = synth.make_weights(cfg, 100 + si)
            strats = synth.strategies_for(cfg.N_b, cfg.R) if cfg.N_b in (1, 2, 4) else None
            for t in range(26):
                n_s = int(rng.integers(0, 40))       # includes v_k = 0 cases
                probs = synth.ACTION_PROBS if t % 3 else (0.0, 0.5, 0.0, 0.0, 0.5, 0.0)
                u = synth.make_user(cfg, rng, n_s=n_s, M=int(rng.integers(1, 5)), action_probs=probs)
                item, action, scenario, _ = u.user_events(0)
                r = int(u.r[0])
                s = O.sumi_scores(cfg, w, strats, u, 0)
                bf = O.brute_force_scores(cfg, w, strats, item, action, scenario, r, u.user_cands(0))
                assert np.max(np.abs(s - bf) / np.maximum(np.abs(bf), 1)) < 1e-12
                n_trip += 1
    assert n_trip >= 200


# ---------------------------------------------------------------------------
# candidate isolation ("diagonal masks"; S:L539 #2)
# ---------------------------------------------------------------------------
def test_candidate_isolation():
    cfg = synth.preset("tiny", L=2)
    w = synth.make_weights(cfg, 7)
    strats = synth.strategies_for(cfg.N_b, cfg.R)
    rng = np.random.default_rng(4)
    u = synth.make_user(cfg, rng, n_s=200, M=12)
    item, action, scenario, _ = u.user_events(0)
    cache = O.encode_user(cfg, w, strats, item, action, scenario, int(u.r[0]))
    cands = u.user_cands(0)
    base = O.score_user(cfg, w, cache, cands)
    for _ in range(20):
        perm = rng.permutation(len(cands))
        assert np.max(np.abs(O.score_user(cfg, w, cache, cands[perm]) - base[perm])) < 1e-12
        keep = np.sort(rng.choice(len(cands), size=5, replace=False))
        extra = rng.integers(0, cfg.V, 3).astype(np.int32)
        s2 = O.score_user(cfg, w, cache, np.concatenate([cands[keep], extra]))
        assert np.max(np.abs(s2[:5] - base[keep])) < 1e-12
    dup = O.score_user(cfg, w, cache, np.array([cands[0], cands[0]]))
    assert dup[0] == dup[1]


# ---------------------------------------------------------------------------
# zero-weights closed form: E_k = c0, G = E, sigma(0) = 1/2
# ---------------------------------------------------------------------------
def test_zero_weights_closed_form():
    cfg = synth.preset("tiny", L=2)
    w = synth.zero_weights_like(synth.make_weights(cfg, 9))
    w = w.scaled(b_head=np.array([0.375], np.float32))
    strats = synth.strategies_for(cfg.N_b, cfg.R)
    u = synth.make_user(cfg, np.random.default_rng(5), n_s=100, M=6)
    s = O.sumi_scores(cfg, w, strats, u, 0)
    r = int(u.r[0])
    for m, c in enumerate(u.user_cands(0)):
        c0 = np.asarray(w.emb_item[c], np.float64) + w.emb_scn[r]
        expect = 0.375 + 0.5 * sum(float(np.dot(w.w_head[k * cfg.d:(k + 1) * cfg.d], c0))
                                   for k in range(cfg.N_b))
        assert abs(s[m] - expect) < 1e-12


def test_empty_history_attends_self_only():
    rng = np.random.default_rng(6)
    q, ks, vs = rng.standard_normal((3, 1, 4))
    o = O.attention(q, ks, vs, [0.7, 1.3], 2)     # v_k = 0: only the self key
    assert np.array_equal(o, vs)


def test_single_block_fusion_is_value():
    """N_b = 1: the fusion ATL's 1x1 softmax is 1."""
    rng = np.random.default_rng(8)
    Q, K, V = rng.standard_normal((3, 1, 8))
    assert np.allclose(O.attention(Q, K, V, [0.3, 5.0], 4), V, atol=1e-15)


# ---------------------------------------------------------------------------
# exact invariants pinning per-head tau indexing
# ---------------------------------------------------------------------------
def _scores(cfg, w, strats, u):
    return O.sumi_scores(cfg, w, strats, u, 0)


def test_tau_query_rescaling_and_head_permutation():
    cfg = synth.preset("tiny", L=2, h=4)
    w = synth.make_weights(cfg, 12)
    strats = synth.strategies_for(cfg.N_b, cfg.R)
    u = synth.make_user(cfg, np.random.default_rng(9), n_s=120, M=5)
    base = _scores(cfg, w, strats, u)
    d, dh, H = cfg.d, cfg.d_h, cfg.h
    # (W_q head h -> a_h W_q, tau[..., h] -> a_h tau): unchanged
    a = np.array([2.0, 0.5, 4.0, 0.25])
    wq = w.w_qkv.copy()
    tau = w.tau.copy()
    for hh in range(H):
        wq[..., :, hh * dh:(hh + 1) * dh] *= a[hh]
        tau[..., hh] *= a[hh]
    s2 = _scores(cfg, w.scaled(w_qkv=wq, tau=tau), strats, u)
    assert np.max(np.abs(s2 - base)) < 1e-11
    # a changed tau for one head must change the scores (tau is actually used per head)
    tau3 = w.tau.copy()
    tau3[..., 1] *= 3.0
    assert np.max(np.abs(_scores(cfg, w.scaled(tau=tau3), strats, u) - base)) > 1e-6
    # head permutation: columns of Q,K,V, rows of W_o, and tau's head index
    perm = np.array([2, 0, 3, 1])
    cols = np.concatenate([np.arange(p * dh, (p + 1) * dh) for p in perm])
    wqkv = w.w_qkv.copy()
    for part in range(3):
        wqkv[..., part * d:(part + 1) * d] = w.w_qkv[..., part * d + cols]
    wo = w.w_o[..., cols, :]
    fq = w.f_w_qkv.copy()
    for part in range(3):
        fq[:, part * d:(part + 1) * d] = w.f_w_qkv[:, part * d + cols]
    w4 = w.scaled(w_qkv=wqkv, w_o=wo, tau=w.tau[..., perm], f_w_qkv=fq,
                  f_w_o=w.f_w_o[cols, :], tau_f=w.tau_f[:, perm])
    assert np.max(np.abs(_scores(cfg, w4, strats, u) - base)) < 1e-11


def test_flop_counter_vs_table4_shape():
    """The per-layer FLOP increment is linear in L (P:L410-417 shows a constant
    3.25e8 per extra layer at s=800): flops(L+1) - flops(L) is constant."""
    vals = []
    for L in (2, 3, 4, 5):
        cfg = synth.preset("large", L=L)
        vals.append(O.flops_user(cfg, [cfg.n_k] * cfg.N_b, 1000)["total"])
    inc = np.diff(vals)
    assert np.all(inc == inc[0])


# ---------------------------------------------------------------------------
# relative attention bias f_b^{p,t}(a_k, r) (Eq. 3; NEXT-1,
# readings G6b-G6e in DESIGN.md)
# ---------------------------------------------------------------------------
def test_bucket_functions_vs_boundary_tables():
    # positions: 16 exact buckets, then each octave [2^e, 2^(e+1)) cut into 4
    # equal-width parts (bucket = 16 + 4 (e - 4) + part), capped at 63 (S:L285 T5 style)
    ref = {}
    for a in range(0, 20000):
        if a < 16:
            ref[a] = a
        else:
            e = 4
            while 2 ** (e + 1) <= a:
                e += 1
            part = (a - 2 ** e) // (2 ** e // 4)
            ref[a] = min(16 + 4 * (e - 4) + part, 63)
    for a, b in ref.items():
        assert O.bucket_pos(a) == b, a
        if a > 0:
            assert O.bucket_pos(-a) == b + 64
    assert O.bucket_pos(16) == 16 and O.bucket_pos(20) == 17 and O.bucket_pos(31) == 19
    assert O.bucket_pos(32) == 20 and O.bucket_pos(1023) == 39 and O.bucket_pos(1 << 20) == 63
    # time deltas in seconds: {0, <1 min, <1 h, <1 d, <1 w, <30 d, >= 30 d}
    table = [(0, 0), (1, 1), (59, 1), (60, 2), (3599, 2), (3600, 3), (86399, 3), (86400, 4),
             (7 * 86400 - 1, 4), (7 * 86400, 5), (30 * 86400 - 1, 5), (30 * 86400, 6), (10 ** 9, 6)]
    for dt, b in table:
        assert O.bucket_time(dt) == b, dt
        if dt > 0:
            assert O.bucket_time(-dt) == b + 7


def _bias_user(cfg, seed, n_s=120, M=6):
    u = synth.make_user(cfg, np.random.default_rng(seed), n_s=n_s, M=M)
    return u


def test_constant_bias_is_a_softmax_shift():
    # a bias that is the same for every (query, key) pair of a row cannot change
    # the softmax (it is added inside R before the normalisation, Eq. 3)
    cfg = synth.preset("tiny", L=2, rel_bias=1)
    w = synth.make_weights(cfg, 3)
    strats = synth.strategies_for(cfg.N_b, cfg.R)
    u = _bias_user(cfg, 21)
    w0 = w.scaled(b_pos=None, b_time=None)
    wc = w.scaled(b_pos=np.full_like(w.b_pos, 1.75), b_time=np.full_like(w.b_time, -0.5))
    s0, sc, sb = (O.sumi_scores(cfg, ww, strats, u, 0) for ww in (w0, wc, w))
    assert np.max(np.abs(sc - s0)) < 1e-12
    assert np.max(np.abs(sb - s0)) > 1e-3        # the drawn tables do matter


def test_bias_enters_before_the_temperature():
    # (W_q, f_b, tau) -> alpha (W_q, f_b, tau) leaves (q.k + f_b) / (sqrt(d_h) tau)
    # unchanged; scaling the bias less than tau does not (pins R = QK^T + f_b, then / f_tc)
    cfg = synth.preset("tiny", L=2, rel_bias=1)
    w = synth.make_weights(cfg, 4)
    strats = synth.strategies_for(cfg.N_b, cfg.R)
    u = _bias_user(cfg, 22)
    base = O.sumi_scores(cfg, w, strats, u, 0)
    a = 2.5
    wq = w.w_qkv.copy()
    wq[..., :cfg.d] *= a
    w_all = w.scaled(w_qkv=wq, b_pos=w.b_pos * a, b_time=w.b_time * a, tau=w.tau * a)
    assert np.max(np.abs(O.sumi_scores(cfg, w_all, strats, u, 0) - base)) < 1e-10
    w_nob = w.scaled(w_qkv=wq, tau=w.tau * a)
    assert np.max(np.abs(O.sumi_scores(cfg, w_nob, strats, u, 0) - base)) > 1e-4


@pytest.mark.parametrize("causal", [1, 0])
def test_bias_reduces_to_sdpa_float_mask(causal):
    # N_b = 1: the block stack equals a pre-norm Transformer whose attention is
    # torch SDPA with an additive float mask f_b / (sqrt(d_h) tau) (library routine)
    cfg = synth.preset("tiny", N_b=1, n_k=64, L=2, hist_causal=causal, rel_bias=1)
    w = synth.make_weights(cfg, 6)
    strats = synth.strategies_for(1, cfg.R)
    u = _bias_user(cfg, 23, n_s=40, M=3)
    item, action, scenario, ts = u.user_events(0)
    r = int(u.r[0])
    cache = O.encode_user(cfg, w, strats, item, action, scenario, r, ts)
    E = O.block_outputs(cfg, w, cache, u.user_cands(0))
    d, dh, H = cfg.d, cfg.d_h, cfg.h
    for m, c in enumerate(u.user_cands(0)):
        X = torch.tensor(np.vstack([np.asarray(w.emb_item[item], np.float64) + w.emb_act[action] + w.emb_scn[scenario],
                                    np.asarray(w.emb_item[c], np.float64) + w.emb_scn[r]]))
        T = X.shape[0]
        times = np.concatenate([ts, [ts[-1]]])          # the item sits at the request time
        for l in range(cfg.L):
            t = lambda a_: torch.tensor(np.asarray(a_, np.float64))
            g1, wqkv, wo, g2, w1, w2 = (t(getattr(w, n)[0, l]) for n in ("g1", "w_qkv", "w_o", "g2", "w1", "w2"))
            P = Fnn.rms_norm(X, (d,), weight=g1, eps=cfg.rms_eps) @ wqkv
            q, kk, v = (P[:, i * d:(i + 1) * d].view(T, H, dh).transpose(0, 1) for i in range(3))
            tau = t(w.tau[l, 0, r])
            q = q / tau.view(H, 1, 1)
            mask = torch.zeros(H, T, T, dtype=torch.float64)
            for i in range(T):
                for j in range(T):
                    allowed = (j <= i) if causal else (j < T - 1 or i == T - 1)
                    if not allowed:
                        mask[:, i, j] = -math.inf
                        continue
                    bp, bt = O.bucket_pos(i - j), O.bucket_time(int(times[i]) - int(times[j]))
                    for hh in range(H):
                        mask[hh, i, j] = float(w.b_pos[l, 0, r, hh, bp] + w.b_time[l, 0, r, hh, bt]) / (
                            math.sqrt(dh) * float(tau[hh]))
            a_ = Fnn.scaled_dot_product_attention(q[None], kk[None], v[None], attn_mask=mask[None])[0]
            X = X + a_.transpose(0, 1).reshape(T, d) @ wo
            X = X + Fnn.silu(Fnn.rms_norm(X, (d,), weight=g2, eps=cfg.rms_eps) @ w1) @ w2
        np.testing.assert_allclose(E[m, 0], X[-1].numpy(), rtol=0, atol=1e-10)


def test_one_hot_position_bias_closed_forms():
    # a dominant bias on one position bucket makes every row attend to exactly
    # one key: bucket 0 -> itself (A = I), bucket 1 -> the previous token
    # (offset i - j = +1, pins the sign of the position offset)
    rng = np.random.default_rng(9)
    T, H, dh = 7, 2, 4
    Q, K, V = rng.standard_normal((3, T, H * dh))
    pos = np.arange(T)
    t0 = np.zeros(T, np.int64)
    for bucket, shift in ((0, 0), (1, 1)):
        bp = np.zeros((H, O.NB_POS))
        bp[:, bucket] = 1e4
        bias = O.rel_bias(bp, np.zeros((H, O.NB_TIME)), pos, t0, pos, t0)
        out = O.attention(Q, K, V, [0.8, 1.7], dh, None, bias)
        np.testing.assert_allclose(out[shift:], V[:T - shift], rtol=0, atol=1e-12)


def test_one_hot_time_bias_picks_the_event_within_the_hour():
    # the candidate (at the request time t_req = last event) attends only to the
    # history event whose age t_req - t_j falls in [1 min, 1 h) when that bucket
    # dominates: pins t_req - t_j (not t_j - t_req) and the bucket edges
    H, dh = 2, 4
    t_hist = np.array([0, 100_000, 196_400, 199_000, 199_990], np.int64)   # ages 2e5, 1e5, 3600, 1000, 10
    t_req = 200_000
    v = len(t_hist)
    rng = np.random.default_rng(10)
    q, ks, vs = rng.standard_normal((3, 1, H * dh))
    Kh, Vh = rng.standard_normal((2, v, H * dh))
    bt = np.zeros((H, O.NB_TIME))
    bt[:, 2] = 1e4                                    # bucket 2 = [60 s, 1 h)
    bias = O.rel_bias(np.zeros((H, O.NB_POS)), bt, [v], [t_req], np.arange(v + 1),
                      np.concatenate([t_hist, [t_req]]))
    out = O.attention(q, np.vstack([Kh, ks]), np.vstack([Vh, vs]), [1.0, 0.6], dh, None, bias)
    np.testing.assert_allclose(out[0], Vh[3], rtol=0, atol=1e-12)        # age 1000 s only


def test_sumi_equals_brute_force_with_bias():
    rng = np.random.default_rng(12)
    n_trip = 0
    for si, sh in enumerate([dict(N_b=2, n_k=8, L=2, d=16, h=2), dict(N_b=1, n_k=12, L=2, d=16, h=4)]):
        for causal in (1, 0):
            cfg = synth.preset("tiny", V=200, M=4, hist_causal=causal, rel_bias=1, **sh)
            w = synth.make_weights(cfg, 200 + si)
            strats = synth.strategies_for(cfg.N_b, cfg.R)
            for t in range(12):
                n_s = int(rng.integers(0, 40))       # includes v_k = 0 cases
                u = synth.make_user(cfg, rng, n_s=n_s, M=int(rng.integers(1, 5)))
                item, action, scenario, ts = u.user_events(0)
                s = O.sumi_scores(cfg, w, strats, u, 0)
                bf = O.brute_force_scores(cfg, w, strats, item, action, scenario, int(u.r[0]),
                                          u.user_cands(0), ts)
                assert np.max(np.abs(s - bf) / np.maximum(np.abs(bf), 1)) < 1e-12
                n_trip += 1
    assert n_trip >= 48
