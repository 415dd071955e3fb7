"""Seeded synthetic inputs for the Climber SUMI hot path.

This module is the ONLY code shared by the fp64 oracle (``oracle/``) and the
CUDA path (``paper_2502_09888_b200``).  It draws random numbers and lays them
out; it holds none of the method's arithmetic (no extraction, no attention, no
norms, no fusion).  The recipe follows SURVEY.md §8(d) "Synthetic inputs" and is
restated in DESIGN.md §3:

* events: actions i.i.d. {play_full .40, skip .25, click .15, like .12,
  share .04, comment .04}; scenarios uniform over R; items Zipf(s=1.1) over V
  (music-catalogue popularity skew, "> 6M items"); timestamps
  t0 ~ U[0, 1e8], integer gaps ~ Exp(mean 600 s) (chronological, ties allowed).
* strategies (Eq. 2: one filter a_k per block): see
  ``strategies_for``.
* weights: N(0, sigma^2) per SURVEY §8(d), every value rounded to bf16 (RNE) so
  that the oracle consumes exactly the values the GPU holds.
* candidates: M Zipf items per user, request scenario r ~ U{0..R-1}.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

# Action vocabulary (Event.action).  Order fixes the ids.
ACTIONS = ("play_full", "skip", "click", "like", "share", "comment")
A_PLAY, A_SKIP, A_CLICK, A_LIKE, A_SHARE, A_COMMENT = range(6)
ACTION_PROBS = (0.40, 0.25, 0.15, 0.12, 0.04, 0.04)
N_ACTIONS = 6


@dataclass
class Config:
    """Model + workload shape (SURVEY §8 "Concrete config shapes")."""
    name: str
    B: int            # users per batch
    N_b: int          # blocks (strategies)
    n_k: int          # per-block budget (n = N_b * n_k)
    M: int            # candidates per user
    L: int            # layers per block
    d: int            # width
    h: int            # heads
    n_s: int          # events per user (lower bound when n_s_max is set)
    n_s_max: int = 0  # >0: n_s ~ U[n_s, n_s_max] per user (medium)
    V: int = 1 << 20  # item vocabulary
    R: int = 4        # scenarios
    dtype: str = "bf16"   # "bf16" or "fp32" (verification build)
    hist_causal: int = 1
    ffn_mult: int = 4
    se_reduction: int = 4
    rms_eps: float = 1e-6
    zipf_s: float = 1.1
    rel_bias: int = 0     # 1: Eq. 3's relative bias f_b^{p,t}(a_k, r)

    @property
    def d_h(self) -> int:
        return self.d // self.h

    @property
    def n(self) -> int:
        return self.N_b * self.n_k

    @property
    def F(self) -> int:
        return self.ffn_mult * self.d

    @property
    def D_se(self) -> int:
        return self.N_b * self.d

    @property
    def H_se(self) -> int:
        return (self.N_b * self.d) // self.se_reduction

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


PRESETS: Dict[str, Config] = {
    # BASELINE.json configs[0..4]; SURVEY §8 table (readings G23-G26)
    "tiny": Config("tiny", B=1, N_b=2, n_k=32, M=16, L=1, d=32, h=2, n_s=256,
                   V=1000, R=2, dtype="fp32"),
    "small": Config("small", B=32, N_b=4, n_k=64, M=128, L=2, d=128, h=4, n_s=2048),
    "medium": Config("medium", B=256, N_b=4, n_k=256, M=512, L=4, d=256, h=8,
                     n_s=1024, n_s_max=4096),
    "large": Config("large", B=1024, N_b=8, n_k=512, M=1000, L=8, d=512, h=8, n_s=8192),
    # sweep centre point; the axes are varied by bench/test code
    "sweep": Config("sweep", B=256, N_b=8, n_k=256, M=1000, L=8, d=512, h=8, n_s=6144),
}


def preset(name: str, **kw) -> Config:
    return PRESETS[name].replace(**kw) if kw else PRESETS[name]


# ---------------------------------------------------------------------------
# strategies (a_k of Eq. 2).  A strategy is (action bitmask, scenario bitmask).
# ---------------------------------------------------------------------------
def strategies_for(N_b: int, R: int) -> List[tuple]:
    """SURVEY §8(d) "Strategies"."""
    allR = (1 << R) - 1
    A = lambda *xs: sum(1 << x for x in xs)
    if N_b == 1:
        return [(A(*range(N_ACTIONS)), allR)]
    if N_b == 2:
        return [(A(A_PLAY, A_LIKE), allR), (A(A_SHARE, A_COMMENT, A_CLICK), allR)]
    base4 = [(A(A_PLAY), allR), (A(A_LIKE), allR), (A(A_SHARE, A_COMMENT), allR),
             (A(A_CLICK), allR)]
    if N_b == 4:
        return base4
    if N_b == 8:
        return base4 + [(A(A_PLAY), 1 << (r % R)) for r in range(4)]
    raise ValueError(f"no strategy recipe for N_b={N_b}")


# ---------------------------------------------------------------------------
# bf16 rounding (RNE) of synthetic weights
# ---------------------------------------------------------------------------
def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 (ties to even); returns fp32."""
    x = np.array(x, dtype=np.float32, copy=True, order="C")
    u = x.view(np.uint32)          # finite values: u + 0x8000 cannot overflow 32 bits
    lsb = (u >> 16) & 1
    lsb += 0x7FFF
    u += lsb
    u &= 0xFFFF0000
    return x


def _normal(rng, shape, std) -> np.ndarray:
    return round_bf16(rng.standard_normal(shape, dtype=np.float32) * np.float32(std))


@dataclass
class Weights:
    """All parameters, fp32 arrays holding bf16-exact values, [in][out] layout.

    Naming follows PAPER.md Eq. 3-4 and SURVEY §8(b) ``climber_weights``.
    """
    emb_item: np.ndarray   # [V][d]
    emb_act: np.ndarray    # [6][d]
    emb_scn: np.ndarray    # [R][d]
    g1: np.ndarray         # [N_b][L][d]
    w_qkv: np.ndarray      # [N_b][L][d][3d]  (columns: Q | K | V, head-major)
    w_o: np.ndarray        # [N_b][L][d][d]
    g2: np.ndarray         # [N_b][L][d]
    w1: np.ndarray         # [N_b][L][d][F]
    w2: np.ndarray         # [N_b][L][F][d]
    tau: np.ndarray        # [L][N_b][R][h]   f_tc(a_k, r) per head
    f_g1: np.ndarray       # fusion ATL, [d]
    f_w_qkv: np.ndarray    # [d][3d]
    f_w_o: np.ndarray      # [d][d]
    f_g2: np.ndarray       # [d]
    f_w1: np.ndarray       # [d][F]
    f_w2: np.ndarray       # [F][d]
    tau_f: np.ndarray      # [R][h]
    w_se1: np.ndarray      # [N_b d][N_b d / 4]
    b_se1: np.ndarray      # [N_b d / 4]
    w_se2: np.ndarray      # [N_b d / 4][N_b d]
    b_se2: np.ndarray      # [N_b d]
    w_head: np.ndarray     # [N_b d]
    b_head: np.ndarray     # [1]
    # relative attention bias tables (Eq. 3 f_b^{p,t}(a_k, r)), only when cfg.rel_bias:
    b_pos: Optional[np.ndarray] = None   # [L][N_b][R][h][NB_POS]  position-offset buckets
    b_time: Optional[np.ndarray] = None  # [L][N_b][R][h][NB_TIME] time-delta buckets

    def scaled(self, **repl) -> "Weights":
        return dataclasses.replace(self, **repl)


# Shapes of the bias tables (interface sizes): 64 position
# buckets per offset sign, 7 time-delta buckets per sign.
NB_POS = 128
NB_TIME = 14


def make_weights(cfg: Config, seed: int = 0) -> Weights:
    w = _make_weights(cfg, seed)
    if cfg.rel_bias:
        # a separate stream, so the other parameters do not depend on rel_bias;
        # std 0.5 sqrt(d_h): comparable to the raw q.k scores the bias is added to
        rng = np.random.default_rng(np.random.PCG64([seed, 7]))
        sd = 0.5 * cfg.d_h ** 0.5
        w.b_pos = _normal(rng, (cfg.L, cfg.N_b, cfg.R, cfg.h, NB_POS), sd)
        w.b_time = _normal(rng, (cfg.L, cfg.N_b, cfg.R, cfg.h, NB_TIME), sd)
    return w


def _make_weights(cfg: Config, seed: int) -> Weights:
    rng = np.random.default_rng(np.random.PCG64(seed))
    d, L, N_b, F, R, h = cfg.d, cfg.L, cfg.N_b, cfg.F, cfg.R, cfg.h
    Dse, Hse = cfg.D_se, cfg.H_se
    tau_draw = lambda shape: round_bf16(np.exp(rng.uniform(np.log(0.5), np.log(2.0), shape)).astype(np.float32))
    gain = lambda shape: round_bf16((1.0 + 0.1 * rng.standard_normal(shape)).astype(np.float32))
    return Weights(
        emb_item=_normal(rng, (cfg.V, d), 1.0),
        emb_act=_normal(rng, (N_ACTIONS, d), 1.0),
        emb_scn=_normal(rng, (R, d), 1.0),
        g1=gain((N_b, L, d)),
        w_qkv=_normal(rng, (N_b, L, d, 3 * d), (1.0 / d) ** 0.5),
        w_o=_normal(rng, (N_b, L, d, d), (1.0 / (2 * L * d)) ** 0.5),
        g2=gain((N_b, L, d)),
        w1=_normal(rng, (N_b, L, d, F), (1.0 / d) ** 0.5),
        w2=_normal(rng, (N_b, L, F, d), (1.0 / (8 * L * d)) ** 0.5),
        tau=tau_draw((L, N_b, R, h)),
        f_g1=gain((d,)),
        f_w_qkv=_normal(rng, (d, 3 * d), (1.0 / d) ** 0.5),
        f_w_o=_normal(rng, (d, d), (1.0 / (2 * d)) ** 0.5),
        f_g2=gain((d,)),
        f_w1=_normal(rng, (d, F), (1.0 / d) ** 0.5),
        f_w2=_normal(rng, (F, d), (1.0 / (8 * d)) ** 0.5),
        tau_f=tau_draw((R, h)),
        w_se1=_normal(rng, (Dse, Hse), (1.0 / Dse) ** 0.5),
        b_se1=_normal(rng, (Hse,), 0.1),
        w_se2=_normal(rng, (Hse, Dse), (4.0 / Dse) ** 0.5),
        b_se2=_normal(rng, (Dse,), 0.1),
        w_head=_normal(rng, (Dse,), (1.0 / Dse) ** 0.5),
        b_head=np.zeros((1,), np.float32),
    )


def zero_weights_like(w: Weights, keep=("emb_item", "emb_act", "emb_scn", "w_head", "b_head",
                                         "tau", "tau_f", "g1", "g2", "f_g1", "f_g2")) -> Weights:
    """Every listed-not-kept parameter set to 0 (zero-weights closed form)."""
    repl = {}
    for f in dataclasses.fields(w):
        if f.name not in keep and getattr(w, f.name) is not None:
            repl[f.name] = np.zeros_like(getattr(w, f.name))
    return w.scaled(**repl)


# ---------------------------------------------------------------------------
# events, candidates
# ---------------------------------------------------------------------------
@dataclass
class Batch:
    """One batch of B requests, events as SoA (SURVEY §8(b) climber_events)."""
    ev_offsets: np.ndarray  # int64 [B+1]
    item: np.ndarray        # int32 [total events]
    action: np.ndarray      # uint8
    scenario: np.ndarray    # uint8
    ts: np.ndarray          # int64, non-decreasing within a user
    r: np.ndarray           # int32 [B] request scenario
    cand_offsets: np.ndarray  # int64 [B+1]
    cand: np.ndarray        # int32 [total candidates]

    @property
    def B(self) -> int:
        return len(self.r)

    def user_events(self, b: int):
        s, e = int(self.ev_offsets[b]), int(self.ev_offsets[b + 1])
        return self.item[s:e], self.action[s:e], self.scenario[s:e], self.ts[s:e]

    def user_cands(self, b: int) -> np.ndarray:
        return self.cand[int(self.cand_offsets[b]):int(self.cand_offsets[b + 1])]

    def subset(self, users) -> "Batch":
        users = list(users)
        ev = [self.user_events(b) for b in users]
        cands = [self.user_cands(b) for b in users]
        off = np.zeros(len(users) + 1, np.int64)
        off[1:] = np.cumsum([len(e[0]) for e in ev])
        coff = np.zeros(len(users) + 1, np.int64)
        coff[1:] = np.cumsum([len(c) for c in cands])
        cat = lambda i, dt: (np.concatenate([e[i] for e in ev]).astype(dt) if users else np.zeros(0, dt))
        return Batch(off, cat(0, np.int32), cat(1, np.uint8), cat(2, np.uint8), cat(3, np.int64),
                     self.r[users].copy(),
                     coff, (np.concatenate(cands).astype(np.int32) if users else np.zeros(0, np.int32)))


def _zipf_sampler(V: int, s: float):
    p = 1.0 / np.arange(1, V + 1, dtype=np.float64) ** s
    cdf = np.cumsum(p)
    cdf /= cdf[-1]

    def draw(rng, n):
        return np.minimum(np.searchsorted(cdf, rng.random(n)), V - 1).astype(np.int32)
    return draw


_ZIPF_CACHE: Dict[tuple, object] = {}


def zipf_draw(rng, V, s, n):
    key = (V, s)
    if key not in _ZIPF_CACHE:
        _ZIPF_CACHE[key] = _zipf_sampler(V, s)
    return _ZIPF_CACHE[key](rng, n)


def make_batch(cfg: Config, seed: int = 1, B: Optional[int] = None, M: Optional[int] = None,
               n_s: Optional[int] = None) -> Batch:
    rng = np.random.default_rng(np.random.PCG64(seed))
    B = cfg.B if B is None else B
    M = cfg.M if M is None else M
    if n_s is not None:
        lens = np.full(B, n_s, np.int64)
    elif cfg.n_s_max > 0:
        lens = rng.integers(cfg.n_s, cfg.n_s_max + 1, size=B).astype(np.int64)
    else:
        lens = np.full(B, cfg.n_s, np.int64)
    off = np.zeros(B + 1, np.int64)
    off[1:] = np.cumsum(lens)
    tot = int(off[-1])
    item = zipf_draw(rng, cfg.V, cfg.zipf_s, tot)
    action = rng.choice(N_ACTIONS, size=tot, p=ACTION_PROBS).astype(np.uint8)
    scenario = rng.integers(0, cfg.R, size=tot).astype(np.uint8)
    gaps = np.floor(rng.exponential(600.0, size=tot)).astype(np.int64)
    ts = np.empty(tot, np.int64)
    for b in range(B):
        s, e = off[b], off[b + 1]
        if e > s:
            t0 = int(rng.integers(0, 10 ** 8))
            g = gaps[s:e].copy()
            g[0] = 0
            ts[s:e] = t0 + np.cumsum(g)
    r = rng.integers(0, cfg.R, size=B).astype(np.int32)
    coff = np.arange(B + 1, dtype=np.int64) * M
    cand = zipf_draw(rng, cfg.V, cfg.zipf_s, B * M)
    return Batch(off, item, action, scenario, ts, r, coff, cand)


def make_user(cfg: Config, rng, n_s: int, M: int, r: Optional[int] = None,
              action_probs=ACTION_PROBS) -> Batch:
    """A single-request batch with explicit sizes (test helper)."""
    item = zipf_draw(rng, cfg.V, cfg.zipf_s, n_s)
    action = rng.choice(N_ACTIONS, size=n_s, p=action_probs).astype(np.uint8)
    scenario = rng.integers(0, cfg.R, size=n_s).astype(np.uint8)
    ts = np.cumsum(np.floor(rng.exponential(600.0, size=n_s)).astype(np.int64))
    rr = int(rng.integers(0, cfg.R)) if r is None else r
    cand = zipf_draw(rng, cfg.V, cfg.zipf_s, M)
    return Batch(np.array([0, n_s], np.int64), item, action, scenario, ts,
                 np.array([rr], np.int32), np.array([0, M], np.int64), cand)
