"""Plain, slow, fp64 reference of the SUMI hot path.  TEST INFRASTRUCTURE ONLY
(see ``oracle/__init__.py``).

Step order follows SURVEY.md §8(c) "The algorithm, step by step":
  extract (Eq. 2) -> embed -> per block k, per layer l: ATL (Eq. 3) over the
  history rows (K/V cached) and over the candidate rows (SUMI masks, §3.2)
  -> BGF (Eq. 4) -> head.
A separate brute-force path (``brute_force_scores``) runs the plain causal
stack over [S_k ; item] for every item alone, with no cache.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np

f64 = np.float64


# ---------------------------------------------------------------------------
# a1: Multi-scale sequence extraction  (Eq. 1-2; G11, G12)
# ---------------------------------------------------------------------------
def extract(action: np.ndarray, scenario: np.ndarray, strategies: Sequence[tuple],
            n_k: int) -> Tuple[np.ndarray, np.ndarray]:
    """S_k = MSE(S, a_k) for every strategy k.

    Scan the chronological events from newest to oldest, keep those whose
    action is in the strategy's action set and whose scenario is in its
    scenario set, stop after n_k, then restore chronological order (G11:
    "the most recent n_k matches, order kept").  Canonical layout (G12):
    left-padded to n_k with -1.

    Returns idx int32 [N_b][n_k] (event indices into the user's events) and
    vlen int32 [N_b].
    """
    n_s = len(action)
    N_b = len(strategies)
    idx = np.full((N_b, n_k), -1, np.int32)
    vlen = np.zeros(N_b, np.int32)
    for k, (amask, smask) in enumerate(strategies):
        kept: List[int] = []
        i = n_s - 1
        while i >= 0 and len(kept) < n_k:
            if (amask >> int(action[i])) & 1 and (smask >> int(scenario[i])) & 1:
                kept.append(i)
            i -= 1
        kept.reverse()
        v = len(kept)
        vlen[k] = v
        idx[k, n_k - v:] = kept
    return idx, vlen


# ---------------------------------------------------------------------------
# SUMI masks ("full-visible masks between each candidate item and the
# entire history ... diagonal masks for inter-item isolation"; S:L311-318;
# G1 causal history, G14 the candidate sees itself)
# ---------------------------------------------------------------------------
def canonical_mask(v: int, n_k: int, M: int, hist_causal: int = 1) -> np.ndarray:
    """Dense boolean mask [(n_k+M)][(n_k+M)] for one block, uint8, true = attend.

    Rows/cols 0..n_k-1 are history slots, left-padded (slot i valid iff
    i >= n_k - v); rows/cols n_k..n_k+M-1 are the M candidates.
    """
    T = n_k + M
    mask = np.zeros((T, T), np.uint8)
    first = n_k - v
    for i in range(T):
        for j in range(T):
            i_hist, j_hist = i < n_k, j < n_k
            if i_hist and i < first:
                continue                       # pad row
            if j_hist and j < first:
                continue                       # pad column
            if i_hist and j_hist:
                ok = (j <= i) if hist_causal else True
            elif i_hist and not j_hist:
                ok = False                     # history never sees candidates
            elif not i_hist and j_hist:
                ok = True                      # candidate -> entire history
            else:
                ok = (i == j)                  # diagonal isolation
            mask[i, j] = 1 if ok else 0
    return mask


# ---------------------------------------------------------------------------
# elementary operations (Eq. 3 and readings G2, G7, G8)
# ---------------------------------------------------------------------------
def rmsnorm(x: np.ndarray, g: np.ndarray, eps: float) -> np.ndarray:
    """Pre-norm (G7): x / sqrt(mean(x^2) + eps) * g, over the last axis."""
    x = np.asarray(x, f64)
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * np.asarray(g, f64)


def silu(x: np.ndarray) -> np.ndarray:
    """f_FFN activation (G8)."""
    return x / (1.0 + np.exp(-x))


def sigmoid(x: np.ndarray) -> np.ndarray:
    return 1.0 / (1.0 + np.exp(-x))


def softmax_tau(z: np.ndarray, tau: float, mask: np.ndarray = None) -> np.ndarray:
    """Softmax(z / tau) over the last axis, masked entries get weight 0.

    Eq. 3: A = Softmax(R / f_tc(a_k, r)).  Every row used on this path has at
    least one unmasked entry (G15).
    """
    z = np.asarray(z, f64) / tau
    if mask is not None:
        z = np.where(mask, z, -np.inf)
    zmax = np.max(z, axis=-1, keepdims=True)
    e = np.exp(z - zmax)
    if mask is not None:
        e = np.where(mask, e, 0.0)
    return e / np.sum(e, axis=-1, keepdims=True)


def attention(Q, K, V, tau_heads, d_h, mask=None, bias=None):
    """Multi-head attention of Eq. 3: per head h,
    R_h = Q_h K_h^T + f_b[h]  (f_b = 0 unless ``bias`` [H][T][S] is given, G6),
    A_h = Softmax(R_h / (sqrt(d_h) * tau[h]))  (G2, G3: Eq. 3 divides R, bias
    included, by f_tc), O_h = A_h V_h.
    Q [T][d], K,V [S][d], mask [T][S] bool or None.  Heads are contiguous d_h
    column groups."""
    T = Q.shape[0]
    H = len(tau_heads)
    out = np.zeros((T, H * d_h), f64)
    if T == 0:                       # empty history (v_k = 0): nothing to attend from
        return out
    for hh in range(H):
        sl = slice(hh * d_h, (hh + 1) * d_h)
        R = Q[:, sl] @ K[:, sl].T
        if bias is not None:
            R = R + bias[hh]
        A = softmax_tau(R / math.sqrt(d_h), float(tau_heads[hh]), mask)
        out[:, sl] = A @ V[:, sl]
    return out


# ---------------------------------------------------------------------------
# relative attention bias f_b^{p,t}(a_k, r) of Eq. 3 (
# SURVEY §8(f) NEXT-1; readings G6b-G6e in DESIGN.md): a per-(layer, block,
# scenario, head) table over bucketed position offsets plus one over bucketed
# time deltas ("bias[head][i][j] = b_pos[..][bucket_p(i-j)] +
# b_time[..][bucket_t(t_i - t_j)]").
# ---------------------------------------------------------------------------
NB_POS = 128                                       # 64 offset buckets per sign
NB_TIME = 14                                       # 7 time buckets per sign
TIME_EDGES = (60, 3600, 86400, 604800, 2592000)    # 1 min, 1 h, 1 d, 1 w, 30 d


def bucket_pos(delta: int) -> int:
    """T5-style log buckets, integer-exact (G6c): |delta| < 16 gets
    its own bucket; above, 4 buckets per octave, 16 + 4 (e - 4) + the two bits
    after the leading one, e = floor(log2 |delta|), capped at 63; negative
    offsets (bidirectional history only) use buckets 64..127."""
    a = abs(int(delta))
    if a < 16:
        b = a
    else:
        e = a.bit_length() - 1
        b = min(16 + 4 * (e - 4) + ((a >> (e - 2)) & 3), 63)
    return b + (64 if delta < 0 else 0)


def bucket_time(dt: int) -> int:
    """Time-delta buckets in seconds {0, <1m, <1h, <1d, <1w, <30d, >=30d}
    (S:L285); negative deltas use buckets 7..13."""
    a = abs(int(dt))
    b = 0 if a == 0 else 1 + sum(1 for edge in TIME_EDGES if a >= edge)
    return b + (7 if dt < 0 else 0)


def rel_bias(b_pos_heads, b_time_heads, pos_q, t_q, pos_k, t_k) -> np.ndarray:
    """f_b [H][T][S] for query positions/times (pos_q, t_q) and key positions/
    times (pos_k, t_k); b_*_heads [H][NB]."""
    dp = np.subtract.outer(np.asarray(pos_q, np.int64), np.asarray(pos_k, np.int64))
    dt = np.subtract.outer(np.asarray(t_q, np.int64), np.asarray(t_k, np.int64))
    # the scalar bucket functions, evaluated once per distinct offset
    up, ip = np.unique(dp, return_inverse=True)
    ut, it = np.unique(dt, return_inverse=True)
    bp = np.array([bucket_pos(x) for x in up], np.int64)[ip].reshape(dp.shape)
    bt = np.array([bucket_time(x) for x in ut], np.int64)[it].reshape(dt.shape)
    H = len(b_pos_heads)
    out = np.zeros((H,) + dp.shape, f64)
    for hh in range(H):
        out[hh] = np.asarray(b_pos_heads[hh], f64)[bp] + np.asarray(b_time_heads[hh], f64)[bt]
    return out


@dataclass
class LayerW:
    g1: np.ndarray
    w_qkv: np.ndarray
    w_o: np.ndarray
    g2: np.ndarray
    w1: np.ndarray
    w2: np.ndarray


def block_layer(w, k: int, l: int) -> LayerW:
    return LayerW(*(np.asarray(getattr(w, n)[k, l], f64) for n in ("g1", "w_qkv", "w_o", "g2", "w1", "w2")))


def fusion_layer(w) -> LayerW:
    return LayerW(*(np.asarray(getattr(w, n), f64) for n in ("f_g1", "f_w_qkv", "f_w_o", "f_g2", "f_w1", "f_w2")))


def qkv(X, lw: LayerW, eps):
    d = X.shape[-1]
    P = rmsnorm(X, lw.g1, eps) @ lw.w_qkv       # f_QKV(X) (Eq. 3) after pre-norm (G7)
    return P[..., :d], P[..., d:2 * d], P[..., 2 * d:]


def ffn_residual(X, lw: LayerW, eps):
    """X + f_FFN(RMSNorm(X)) with f_FFN = W2 . SiLU(W1 .) (G7, G8)."""
    return X + silu(rmsnorm(X, lw.g2, eps) @ lw.w1) @ lw.w2


def atl_layer(X, lw: LayerW, tau_heads, d_h, mask, eps, bias=None):
    """One ATL (Eq. 3) over a whole sequence with an explicit mask
    (and relative bias [H][T][T] when given).  Returns (X_next, K, V)."""
    Q, K, V = qkv(X, lw, eps)
    X = X + attention(Q, K, V, tau_heads, d_h, mask, bias) @ lw.w_o
    return ffn_residual(X, lw, eps), K, V


def _bias_tables(w, l, k, r):
    """The (layer, block, scenario) slices of the bias tables, or None (f_b = 0)."""
    if getattr(w, "b_pos", None) is None:
        return None
    return np.asarray(w.b_pos[l, k, r], f64), np.asarray(w.b_time[l, k, r], f64)


# ---------------------------------------------------------------------------
# a2 embedding ("embedding lookup"; G10)
# ---------------------------------------------------------------------------
def embed_history(w, item, action, scenario, idx_k):
    sel = idx_k[idx_k >= 0]
    return (np.asarray(w.emb_item[item[sel]], f64) + np.asarray(w.emb_act[action[sel]], f64)
            + np.asarray(w.emb_scn[scenario[sel]], f64))


def embed_candidates(w, cands, r):
    return np.asarray(w.emb_item[cands], f64) + np.asarray(w.emb_scn[r], f64)[None, :]


# ---------------------------------------------------------------------------
# a3: encode the user once, cache per-layer K/V ("first generates
# multi-layered key-value (KV) cache vectors from user features")
# ---------------------------------------------------------------------------
@dataclass
class Cache:
    idx: np.ndarray          # [N_b][n_k] canonical
    vlen: np.ndarray         # [N_b]
    K: list                  # K[k][l] -> [v_k][d] fp64
    V: list
    r: int
    t_hist: list = None      # [N_b] -> int64 [v_k] event times of S_k (relative bias)
    t_req: int = 0           # request time (G6e: the last event's timestamp)


def request_time(ts) -> int:
    """G6e: the events passed to encode end at the request, so the request
    (= candidate) time is the last event's timestamp; 0 for an empty sequence."""
    return int(ts[-1]) if ts is not None and len(ts) > 0 else 0


def encode_user(cfg, w, strategies, item, action, scenario, r: int, ts=None) -> Cache:
    idx, vlen = extract(action, scenario, strategies, cfg.n_k)
    Ks, Vs, Ts = [], [], []
    for k in range(cfg.N_b):
        X = embed_history(w, item, action, scenario, idx[k])
        v = X.shape[0]
        if cfg.hist_causal:
            mask = np.tril(np.ones((v, v), bool))       # G1: causal history
        else:
            mask = np.ones((v, v), bool)
        sel = idx[k][idx[k] >= 0]
        t_k = np.asarray(ts, np.int64)[sel] if ts is not None else np.zeros(v, np.int64)
        pos = np.arange(v)                              # G6d: position = index within S_k
        Kk, Vk = [], []
        for l in range(cfg.L):
            lw = block_layer(w, k, l)
            tb = _bias_tables(w, l, k, r)
            bias = rel_bias(tb[0], tb[1], pos, t_k, pos, t_k) if tb is not None else None
            X, K, V = atl_layer(X, lw, w.tau[l, k, r], cfg.d_h, mask, cfg.rms_eps, bias)
            Kk.append(K)
            Vk.append(V)
        Ks.append(Kk)
        Vs.append(Vk)
        Ts.append(t_k)
    return Cache(idx, vlen, Ks, Vs, r, Ts, request_time(ts))


# ---------------------------------------------------------------------------
# a4: score M candidates against the cache
# ---------------------------------------------------------------------------
def candidate_layer(C, lw: LayerW, tau_heads, d_h, K_hist, V_hist, eps, tables=None, t_hist=None, t_req=0):
    """Each candidate row attends to the cached history K/V of this layer and
    to itself only (full-visible to history, diagonal among candidates).  With
    bias tables, a candidate sits at position v_k and time t_req (G6d, G6e)."""
    Q, Ks, Vs = qkv(C, lw, eps)
    Mc = C.shape[0]
    v = K_hist.shape[0]
    bias = None
    if tables is not None:
        pos_k = np.arange(v + 1)                        # history 0..v-1, self at v
        t_k = np.concatenate([np.asarray(t_hist, np.int64), [t_req]])
        bias = rel_bias(tables[0], tables[1], [v], [t_req], pos_k, t_k)
    O = np.zeros_like(Q)
    for m in range(Mc):
        Kc = np.vstack([K_hist, Ks[m:m + 1]])
        Vc = np.vstack([V_hist, Vs[m:m + 1]])
        O[m] = attention(Q[m:m + 1], Kc, Vc, tau_heads, d_h, None, bias)[0]
    C = C + O @ lw.w_o
    return ffn_residual(C, lw, eps)


def block_outputs(cfg, w, cache: Cache, cands) -> np.ndarray:
    """E(S_k) for every candidate: [M][N_b][d] (G13: candidate row after the
    last layer, no final norm)."""
    c0 = embed_candidates(w, cands, cache.r)
    E = np.zeros((len(cands), cfg.N_b, cfg.d), f64)
    for k in range(cfg.N_b):
        C = c0.copy()
        for l in range(cfg.L):
            C = candidate_layer(C, block_layer(w, k, l), w.tau[l, k, cache.r], cfg.d_h,
                                cache.K[k][l], cache.V[k][l], cfg.rms_eps,
                                _bias_tables(w, l, k, cache.r),
                                cache.t_hist[k] if cache.t_hist is not None else None, cache.t_req)
        E[:, k, :] = C
    return E


# ---------------------------------------------------------------------------
# a5/a6: bit-wise gating fusion (Eq. 4) and the head (G18)
# ---------------------------------------------------------------------------
def bgf(cfg, w, E: np.ndarray, r: int) -> np.ndarray:
    """Y(S) = G(S) . sigma(f_gate(G(S))),  G(S) = ATL(E(S)).
    Fusion ATL: no relative bias, temperature from the scenario only,
    full visibility among the N_b tokens (G16).  f_gate = squeeze-and-excitation
    FC(N_b d -> N_b d/4)+b, ReLU, FC(-> N_b d)+b (G17).  E [M][N_b][d]."""
    lw = fusion_layer(w)
    Mc = E.shape[0]
    G = np.zeros_like(E)
    for m in range(Mc):
        G[m], _, _ = atl_layer(E[m], lw, w.tau_f[r], cfg.d_h, None, cfg.rms_eps)
    s = G.reshape(Mc, cfg.N_b * cfg.d)                           # vec(G), block-major
    z = np.maximum(s @ np.asarray(w.w_se1, f64) + np.asarray(w.b_se1, f64), 0.0)
    z = z @ np.asarray(w.w_se2, f64) + np.asarray(w.b_se2, f64)
    return (s * sigmoid(z)).reshape(Mc, cfg.N_b, cfg.d)


def head(cfg, w, Y: np.ndarray) -> np.ndarray:
    """score = w_head . vec(Y) + b_head, a logit (G18)."""
    return Y.reshape(Y.shape[0], -1) @ np.asarray(w.w_head, f64) + float(w.b_head[0])


def score_user(cfg, w, cache: Cache, cands) -> np.ndarray:
    E = block_outputs(cfg, w, cache, np.asarray(cands))
    return head(cfg, w, bgf(cfg, w, E, cache.r))


def sumi_scores(cfg, w, strategies, batch, b: int) -> np.ndarray:
    item, action, scenario, ts = batch.user_events(b)
    cache = encode_user(cfg, w, strategies, item, action, scenario, int(batch.r[b]), ts)
    return score_user(cfg, w, cache, batch.user_cands(b))


# ---------------------------------------------------------------------------
# brute force: every item appended alone to [S_k], no cache
# ---------------------------------------------------------------------------
def brute_force_scores(cfg, w, strategies, item, action, scenario, r: int, cands, ts=None) -> np.ndarray:
    idx, _ = extract(action, scenario, strategies, cfg.n_k)
    t_req = request_time(ts)
    out = np.zeros(len(cands), f64)
    for m, c in enumerate(cands):
        E = np.zeros((1, cfg.N_b, cfg.d), f64)
        for k in range(cfg.N_b):
            X = np.vstack([embed_history(w, item, action, scenario, idx[k]),
                           embed_candidates(w, np.array([c]), r)])
            T = X.shape[0]
            if cfg.hist_causal:
                mask = np.tril(np.ones((T, T), bool))        # plain causal, j <= i
            else:                                             # prefix-LM
                mask = np.ones((T, T), bool)
                mask[:T - 1, T - 1] = False
            sel = idx[k][idx[k] >= 0]                         # the sequence [S_k ; item]:
            pos = np.arange(T)                                # positions 0..T-1
            t_seq = np.concatenate([np.asarray(ts, np.int64)[sel] if ts is not None else np.zeros(T - 1, np.int64),
                                    [t_req]])                 # item at the request time
            for l in range(cfg.L):
                tb = _bias_tables(w, l, k, r)
                bias = rel_bias(tb[0], tb[1], pos, t_seq, pos, t_seq) if tb is not None else None
                X, _, _ = atl_layer(X, block_layer(w, k, l), w.tau[l, k, r], cfg.d_h, mask, cfg.rms_eps, bias)
            E[0, k] = X[-1]
        out[m] = head(cfg, w, bgf(cfg, w, E, r))[0]
    return out


# ---------------------------------------------------------------------------
# algorithmic FLOP count (SURVEY §8(d) "Roofline"; the bench's achieved TFLOP/s)
# ---------------------------------------------------------------------------
def flops_user(cfg, vlen: Sequence[int], M: int) -> dict:
    """Multiply-adds x2 that SUMI itself must compute for one request: encode
    (all layers' history QKV/attention/O/FFN, last layer K/V only) plus every
    candidate through N_b x L layers, BGF and the head.  Causal history
    attention counts v(v+1)/2 score pairs."""
    d, F, L, dh, H = cfg.d, cfg.F, cfg.L, cfg.d_h, cfg.h
    enc = att_h = cand = att_c = 0
    for v in vlen:
        v = int(v)
        pairs = v * (v + 1) // 2 if cfg.hist_causal else v * v
        enc += (L - 1) * (2 * v * d * 3 * d + 2 * v * d * d + 2 * 2 * v * d * F) + 2 * v * d * 2 * d
        att_h += (L - 1) * 2 * 2 * pairs * d
        cand += L * M * (2 * d * 3 * d + 2 * d * d + 2 * 2 * d * F)
        att_c += L * M * 2 * 2 * (v + 1) * d
    Nb = cfg.N_b
    fus = M * Nb * (2 * d * 3 * d + 2 * d * d + 2 * 2 * d * F) + M * 2 * 2 * Nb * Nb * d
    se = M * (2 * cfg.D_se * cfg.H_se * 2) + M * 2 * cfg.D_se
    return {"encode_gemm": enc, "encode_attn": att_h, "cand_gemm": cand, "cand_attn": att_c,
            "fusion": fus, "se_head": se,
            "total": enc + att_h + cand + att_c + fus + se}
