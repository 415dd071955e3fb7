"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle on the same
seeded synthetic inputs (north star tolerances; masks/indices bit-exact)."""
import numpy as np
import pytest

import oracle as O
import synth
from helpers import gpu_scores, make_gpu, oracle_scores, parity_err, to_dev, tolerance

pytestmark = pytest.mark.gpu


def _check_cfg(cfg, B, users, seed_w=0, seed_b=1, **kw):
    w = synth.make_weights(cfg, seed_w)
    batch = synth.make_batch(cfg, seed_b, B=B)
    cl = make_gpu(cfg, w, B, **kw)
    got = gpu_scores(cl, batch)
    cl.stream_status()
    ref = oracle_scores(cfg, w, batch, users)
    tol = tolerance(cfg)
    worst = (0.0, 0.0)
    for b, r in ref.items():
        s0, s1 = int(batch.cand_offsets[b]), int(batch.cand_offsets[b + 1])
        ab, rel = parity_err(got[s0:s1], r)
        worst = (max(worst[0], ab), max(worst[1], rel))
    assert np.all(np.isfinite(got))
    assert worst[0] <= tol and worst[1] <= tol, (cfg.name, worst)
    return worst


def test_tiny_fp32():
    _check_cfg(synth.preset("tiny"), B=1, users=[0])


@pytest.mark.parametrize("causal", [1, 0])
def test_tiny_l2_fp32(causal):
    cfg = synth.preset("tiny", L=2, B=3, hist_causal=causal)
    _check_cfg(cfg, B=3, users=[0, 1, 2])


def test_tiny_bf16():
    cfg = synth.preset("tiny", L=2, dtype="bf16")
    _check_cfg(cfg, B=2, users=[0, 1])


def test_small_fp32_verification_build():
    cfg = synth.preset("small", dtype="fp32")
    _check_cfg(cfg, B=4, users=[0, 1, 2, 3])


def test_small_bf16():
    _check_cfg(synth.preset("small"), B=32, users=[0, 7, 31])


def test_medium_bf16_ragged():
    _check_cfg(synth.preset("medium"), B=8, users=[0, 3, 7])


def test_large_bf16():
    cfg = synth.preset("large")
    _check_cfg(cfg, B=2, users=[0, 1], max_wave_pairs=2000)


@pytest.mark.parametrize("name", ["large", "medium"])
def test_single_request_bf16(name):
    # latency mode (B = 1): small launches
    _check_cfg(synth.preset(name), B=1, users=[0])


def test_single_request_small_gemm_tiles():
    # the 128 x 128 single-CTA GEMM tiles on every small launch (knobs read once
    # per process): their RESID_NORM epilogue must write the same per-128-column
    # norm partials as the 256-wide pair tiles
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path[:0] = [%r, %r]; import synth, test_gpu_parity as t; "
            "t._check_cfg(synth.preset('medium'), B=1, users=[0]); t._check_cfg(synth.preset('large'), B=1, users=[0])"
            % (root, os.path.join(root, "tests")))
    env = dict(os.environ, CLIMBER_GEMM_SMALL_WAVES="4", CLIMBER_GEMM_SMALL_GFLOP="1e9")
    subprocess.run([sys.executable, "-c", code], env=env, check=True, cwd=root, timeout=600)


def test_sweep_corner_bf16():
    cfg = synth.preset("sweep", L=2, n_k=64, M=100, n_s=1536)
    _check_cfg(cfg, B=2, users=[0, 1])


# ---------------------------------------------------------------------------
# integer parity: extraction indices and canonical masks bit-exact
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["tiny", "small", "medium"])
def test_extract_and_mask_bit_exact(name):
    cfg = synth.preset(name)
    if name == "tiny":
        cfg = cfg.replace(hist_causal=0)
    w = synth.make_weights(cfg, 0)
    B = 3
    batch = synth.make_batch(cfg, 2, B=B)
    cl = make_gpu(cfg, w, B)
    item, action, scenario, ts, cand = to_dev(batch)
    hs = cl.encode_users(batch.ev_offsets, item, action, scenario, ts, batch.r)
    strats = synth.strategies_for(cfg.N_b, cfg.R)
    for b in range(B):
        _, a, sc, _ = batch.user_events(b)
        idx, vlen = cl.debug_extract(hs[b])
        ridx, rvlen = O.extract(a, sc, strats, cfg.n_k)
        assert np.array_equal(idx, ridx) and np.array_equal(vlen, rvlen)
        M = 5
        mask = cl.debug_mask(hs[b], M)
        for k in range(cfg.N_b):
            assert np.array_equal(mask[k], O.canonical_mask(int(rvlen[k]), cfg.n_k, M, cfg.hist_causal))
    cl.release(hs)


def test_kv_cache_matches_oracle():
    cfg = synth.preset("tiny", L=2)
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 1, B=1)
    cl = make_gpu(cfg, w, 1)
    item, action, scenario, ts, cand = to_dev(batch)
    hs = cl.encode_users(batch.ev_offsets, item, action, scenario, ts, batch.r)
    it, a, sc, _ = batch.user_events(0)
    cache = O.encode_user(cfg, w, synth.strategies_for(cfg.N_b, cfg.R), it, a, sc, int(batch.r[0]))
    for k in range(cfg.N_b):
        for l in range(cfg.L):
            v = int(cache.vlen[k])
            K, V = cl.debug_kv(hs[0], l, k, v)
            np.testing.assert_allclose(K, cache.K[k][l], atol=1e-4, rtol=1e-4)
            np.testing.assert_allclose(V, cache.V[k][l], atol=1e-4, rtol=1e-4)
    cl.release(hs)


# ---------------------------------------------------------------------------
# invariants on the GPU: permutation (bitwise), determinism, reuse, isolation
# ---------------------------------------------------------------------------
def test_permutation_determinism_and_cache_reuse_bitwise():
    import torch
    cfg = synth.preset("small")
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 3, B=4)
    cl = make_gpu(cfg, w, 4, kv_users=8)
    s1, hs, (item, action, scenario, ts, cand) = gpu_scores(cl, batch, release=False)
    s2 = cl.score_batched(hs, batch.cand_offsets, cand).cpu().numpy()
    assert np.array_equal(s1, s2)                     # reuse + run-to-run determinism
    M = cfg.M
    rng = np.random.default_rng(0)
    perm = np.concatenate([b * M + rng.permutation(M) for b in range(4)])
    s3 = cl.score_batched(hs, batch.cand_offsets, cand[torch.from_numpy(perm).cuda()]).cpu().numpy()
    assert np.array_equal(s3, s1[perm])               # permuting candidates permutes scores bitwise
    # a bystander's score does not depend on the other candidates (isolation)
    sub = cand.view(4, M)[:, :7].contiguous().view(-1)
    off = np.arange(5, dtype=np.int64) * 7
    s4 = cl.score_batched(hs, off, sub).cpu().numpy().reshape(4, 7)
    assert np.array_equal(s4, s1.reshape(4, M)[:, :7])
    # re-encoding the same user gives bit-identical scores
    s5 = gpu_scores(cl, batch)
    assert np.array_equal(s5, s1)
    cl.release(hs)


def test_empty_history_and_single_candidate():
    cfg = synth.preset("tiny", L=2)
    w = synth.make_weights(cfg, 0)
    rng = np.random.default_rng(1)
    u = synth.make_user(cfg, rng, n_s=0, M=1)
    cl = make_gpu(cfg, w, 1)
    got = gpu_scores(cl, u)
    ref = oracle_scores(cfg, w, u)[0]
    assert parity_err(got, ref)[0] < 1e-4


def test_device_errors_and_stale_handles():
    import torch
    from paper_2502_09888_b200 import ClimberError
    cfg = synth.preset("tiny")
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 1, B=1)
    cl = make_gpu(cfg, w, 1)
    item, action, scenario, ts, cand = to_dev(batch)
    bad_cand = cand.clone()
    bad_cand[3] = cfg.V + 5
    hs = cl.encode_users(batch.ev_offsets, item, action, scenario, ts, batch.r)
    s = cl.score_batched(hs, batch.cand_offsets, bad_cand).cpu().numpy()
    with pytest.raises(ClimberError) as ei:
        cl.stream_status()
    assert ei.value.name == "E_OUT_OF_RANGE"
    assert np.isnan(s[3]) and np.all(np.isfinite(np.delete(s, 3)))   # only that candidate
    cl.release(hs)
    with pytest.raises(ClimberError) as ei:
        cl.release(hs)
    assert ei.value.name == "E_STALE"
    with pytest.raises(ClimberError) as ei:
        cl.score_batched(hs, batch.cand_offsets, cand)
    assert ei.value.name == "E_STALE"
    ts_bad = ts.clone()
    ts_bad[10] = ts_bad[9] - 1
    hs = cl.encode_users(batch.ev_offsets, item, action, scenario, ts_bad, batch.r)
    with pytest.raises(ClimberError) as ei:
        cl.stream_status()
    assert ei.value.name == "E_UNSORTED"
    cl.release(hs)
    with pytest.raises(ClimberError) as ei:
        cl.score_batched(hs, np.array([0, cfg.M + 1]), cand)
    assert ei.value.name in ("E_INVALID_ARG", "E_STALE")


def test_rank_host_end_to_end():
    cfg = synth.preset("small")
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 1, B=4)
    cl = make_gpu(cfg, w, 4)
    s_host = cl.rank_host(batch.ev_offsets, batch.item, batch.action, batch.scenario, batch.ts, batch.r,
                          batch.cand_offsets, batch.cand)
    s_dev = gpu_scores(cl, batch)
    assert np.array_equal(s_host, s_dev)


def _one_user(batch, b):
    """Host arrays of user b alone (offsets rebased to 0)."""
    e0, e1 = int(batch.ev_offsets[b]), int(batch.ev_offsets[b + 1])
    c0, c1 = int(batch.cand_offsets[b]), int(batch.cand_offsets[b + 1])
    return (np.array([0, e1 - e0], np.int64), batch.item[e0:e1], batch.action[e0:e1], batch.scenario[e0:e1],
            batch.ts[e0:e1], batch.r[b:b + 1], np.array([0, c1 - c0], np.int64), batch.cand[c0:c1])


@pytest.mark.parametrize("name", ["small", "medium"])
def test_latency_mode_cuda_graph(name):
    # rank_host with B = 1 replays one captured CUDA graph per (events, candidates)
    # shape; the scores must equal the eager encode + score path bit for bit,
    # across replays, shape changes and handle slots
    cfg = synth.preset(name)
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 3, B=4)
    cl = make_gpu(cfg, w, 4)
    eager = gpu_scores(cl, batch)
    n_before = cl.launch_count
    for rep in range(2):
        for b in (0, 1, 1, 2, 0, 3):
            got = cl.rank_host(*_one_user(batch, b))
            c0, c1 = int(batch.cand_offsets[b]), int(batch.cand_offsets[b + 1])
            assert np.array_equal(got, eager[c0:c1]), (name, rep, b)
    assert cl.launch_count > n_before  # replays are counted as kernel launches
    cl.stream_status()
    ref = oracle_scores(cfg, w, batch, [1])[1]
    c0, c1 = int(batch.cand_offsets[1]), int(batch.cand_offsets[2])
    ab, rel = parity_err(cl.rank_host(*_one_user(batch, 1)), ref)
    assert ab <= tolerance(cfg) and rel <= tolerance(cfg)


# ---------------------------------------------------------------------------
# Eq. 3 relative attention bias f_b^{p,t}(a_k, r)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("causal", [1, 0])
def test_rel_bias_fp32_tiny(causal):
    cfg = synth.preset("tiny", L=2, B=3, hist_causal=causal, rel_bias=1)
    _check_cfg(cfg, B=3, users=[0, 1, 2])


@pytest.mark.parametrize("name,users", [("medium", [0, 3]), ("large", [0])])
def test_rel_bias_bf16(name, users):
    cfg = synth.preset(name, rel_bias=1)
    _check_cfg(cfg, B=4, users=users, max_wave_pairs=4 * cfg.M)
    # the bias is live on this path: the same inputs without it score differently
    batch = synth.make_batch(cfg, 1, B=2)
    w = synth.make_weights(cfg, 0)
    with_b = gpu_scores(make_gpu(cfg, w, 2), batch)
    cfg0 = cfg.replace(rel_bias=0)
    without = gpu_scores(make_gpu(cfg0, w, 2), batch)
    assert np.max(np.abs(with_b - without)) > 0.03   # above the 2e-2 parity bound: a dropped bias fails parity


def test_rel_bias_bf16_latency_mode_and_config_errors():
    from paper_2502_09888_b200 import ClimberError
    cfg = synth.preset("medium", rel_bias=1)
    _check_cfg(cfg, B=1, users=[0])           # single request: small-launch GEMM tiles
    # n_k = 64 (one half-empty 128-row history tile) is covered by the tcgen05 kernel
    _check_cfg(synth.preset("small", rel_bias=1), B=2, users=[0, 1])
    bad = synth.preset("tiny", rel_bias=1, dtype="bf16")   # d_h = 16: no tcgen05 attention
    with pytest.raises(ClimberError) as ei:
        make_gpu(bad, synth.make_weights(bad, 0), 1)
    assert ei.value.name == "E_CONFIG"


# ---------------------------------------------------------------------------
# SUMI forward of compressed training records (NEXT-3)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["small", "medium"])
def test_forward_sumi_record_equals_susi_records(name):
    # one "single user, multiple items" record scores every item exactly as the
    # "single user, single item" records of the same pairs do (bitwise), and as
    # the cached serving path
    import torch
    cfg = synth.preset(name)
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 4, B=2, M=24)
    cl = make_gpu(cfg, w, 24, M_max=24)
    item, action, scenario, ts, cand = to_dev(batch)
    sumi = cl.forward(batch.ev_offsets, item, action, scenario, ts, batch.r, batch.cand_offsets, cand)
    serve = gpu_scores(cl, batch)
    assert np.array_equal(sumi.cpu().numpy(), serve)
    for b in range(batch.B):
        u = batch.subset([b] * 24)                       # 24 records of user b, one item each
        c0 = int(batch.cand_offsets[b])
        items = torch.from_numpy(batch.cand[c0:c0 + 24].copy()).cuda()
        dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        susi = cl.forward(u.ev_offsets, dv(u.item), dv(u.action), dv(u.scenario), dv(u.ts), u.r,
                          np.arange(25, dtype=np.int64), items)
        assert torch.equal(susi, sumi[c0:c0 + 24])
    cl.stream_status()


def test_sync_check_reports_non_finite_scores():
    # CLIMBER_SYNC_CHECK=1 (read at create): a score that is not finite fails
    # the score call with E_NUMERIC.  An item embedding near the fp32 maximum
    # overflows its candidate rows' projections (inf * 0 = NaN after the norm).
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r"""
import sys, numpy as np; sys.path[:0] = [%r, %r]
import synth
from helpers import make_gpu, gpu_scores
from paper_2502_09888_b200 import ClimberError
cfg = synth.preset("small"); w = synth.make_weights(cfg, 0); batch = synth.make_batch(cfg, 1, B=2)
ok = gpu_scores(make_gpu(cfg, w, 2), batch)
assert np.all(np.isfinite(ok))
emb = w.emb_item.copy(); emb[int(batch.cand[5])] = 3e38
cl = make_gpu(cfg, w.scaled(emb_item=emb), 2)
try:
    gpu_scores(cl, batch)
    print("no error")
except ClimberError as e:
    print(e.name)
""" % (root, os.path.join(root, "tests"))
    env = dict(os.environ, CLIMBER_SYNC_CHECK="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.strip().endswith("E_NUMERIC"), (out.stdout, out.stderr[-2000:])


def test_large_in_bench_launch_configuration_sampled():
    # BASELINE configs[3] in the launch configuration bench.py times (waves of
    # 64 users, up to 65536 pairs per wave, 1000 candidates per user): 128 users
    # = two encode waves and two score waves; sampled users vs the oracle
    cfg = synth.preset("large")
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 1, B=128)
    from paper_2502_09888_b200 import Climber, ModelConfig
    cl = Climber(ModelConfig.from_any(cfg), w, synth.strategies_for(cfg.N_b, cfg.R), max_users=128,
                 max_wave_users=64, max_wave_pairs=65536, kv_users=128)
    got = gpu_scores(cl, batch)
    cl.stream_status()
    assert np.all(np.isfinite(got))
    ref = oracle_scores(cfg, w, batch, [0, 77, 127])
    for b, r in ref.items():
        ab, rel = parity_err(got[batch.cand_offsets[b]:batch.cand_offsets[b + 1]], r)
        assert ab <= tolerance(cfg) and rel <= tolerance(cfg), (b, ab, rel)


def test_sweep_deep_and_long_corners_bf16():
    # BASELINE configs[4] axis ends: 16 layers, and n = 8192 (n_k = 1024)
    for kw in (dict(L=16, n_k=128, M=64, n_s=3 * 128 * 8), dict(L=2, n_k=1024, M=64, n_s=3 * 1024 * 8)):
        _check_cfg(synth.preset("sweep", **kw), B=1, users=[0])
