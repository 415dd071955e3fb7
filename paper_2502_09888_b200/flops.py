"""Algorithmic FLOP count of the SUMI path on the ACTUAL subsequence lengths
v_{b,k}, per kernel class of the bench's breakdown ("the
harness counts FLOPs from the actual v_{b,k}").  Measurement bookkeeping for
bench.py, not part of the compute path: padded rows and masked keys that the
kernels execute are not counted.  Conventions of SURVEY §8(c) G7-G19: encode
runs layers 0..L-2 in full and only the K/V projection at layer L-1; causal
history attention counts v (v + 1) / 2 score pairs (bidirectional v^2);
a candidate attends to v keys plus itself; 2 FLOP per multiply-add."""
from typing import Dict, Iterable, Sequence

CLASSES = ("gemm_qkv", "gemm_o", "gemm_ffn_up", "gemm_ffn_down", "gemm_se", "attn_hist", "attn_sumi",
           "attn_fusion", "head")


def class_flops(d: int, L: int, N_b: int, ffn_mult: int, se_reduction: int, hist_causal: int,
                vlens: Iterable[Sequence[int]], cands: Iterable[int]) -> Dict[str, float]:
    """vlens: per user, its N_b valid lengths; cands: per user, its candidate count."""
    F = ffn_mult * d
    Dse = N_b * d
    Hse = Dse // se_reduction
    f = dict.fromkeys(CLASSES, 0.0)
    for vl, M in zip(vlens, cands):
        for v in vl:
            v = int(v)
            pairs = v * (v + 1) // 2 if hist_causal else v * v
            # encode: layers 0 .. L-2 in full, layer L-1 K / V only
            f["gemm_qkv"] += (L - 1) * 2.0 * v * d * 3 * d + 2.0 * v * d * 2 * d
            f["gemm_o"] += (L - 1) * 2.0 * v * d * d
            f["gemm_ffn_up"] += (L - 1) * 2.0 * v * d * F
            f["gemm_ffn_down"] += (L - 1) * 2.0 * v * F * d
            f["attn_hist"] += (L - 1) * 4.0 * pairs * d
            # the candidates through every layer of this block
            f["gemm_qkv"] += L * M * 2.0 * d * 3 * d
            f["gemm_o"] += L * M * 2.0 * d * d
            f["gemm_ffn_up"] += L * M * 2.0 * d * F
            f["gemm_ffn_down"] += L * M * 2.0 * F * d
            f["attn_sumi"] += L * M * 4.0 * (v + 1) * d
        # BGF: the fusion ATL over the N_b tokens of every candidate, SE gate, head
        f["gemm_qkv"] += M * N_b * 2.0 * d * 3 * d
        f["gemm_o"] += M * N_b * 2.0 * d * d
        f["gemm_ffn_up"] += M * N_b * 2.0 * d * F
        f["gemm_ffn_down"] += M * N_b * 2.0 * F * d
        f["attn_fusion"] += M * 4.0 * N_b * N_b * d
        f["gemm_se"] += M * 2.0 * Dse * Hse * 2
        f["head"] += M * 2.0 * Dse
    return f
