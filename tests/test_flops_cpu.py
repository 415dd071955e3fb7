"""The bench's per-class algorithmic FLOP count on actual v_{b,k}
(paper_2502_09888_b200/flops.py) sums to the oracle's independently written
flops_user, for ragged lengths, empty blocks and both mask modes."""
import numpy as np

import oracle as O
import synth
from paper_2502_09888_b200.flops import class_flops


def test_class_flops_sum_to_oracle_count():
    rng = np.random.default_rng(0)
    for causal in (1, 0):
        for name in ("small", "medium", "large"):
            cfg = synth.preset(name, hist_causal=causal)
            vlens = [rng.integers(0, cfg.n_k + 1, cfg.N_b) for _ in range(5)]
            vlens[1][:] = 0
            cands = [int(rng.integers(1, cfg.M + 1)) for _ in range(5)]
            f = class_flops(cfg.d, cfg.L, cfg.N_b, cfg.ffn_mult, cfg.se_reduction, cfg.hist_causal, vlens, cands)
            ref = sum(O.flops_user(cfg, vl, M)["total"] for vl, M in zip(vlens, cands))
            assert abs(sum(f.values()) - ref) <= 1e-9 * ref, (name, causal)
            # attention parts separately
            ref_h = sum(O.flops_user(cfg, vl, M)["encode_attn"] for vl, M in zip(vlens, cands))
            ref_c = sum(O.flops_user(cfg, vl, M)["cand_attn"] for vl, M in zip(vlens, cands))
            assert f["attn_hist"] == ref_h and f["attn_sumi"] == ref_c
