"""One small encode + score per config through the C ABI, for compute-sanitizer
(tools/sanitize.sh).  Checks the scores against the fp64 oracle so a run that
passes the sanitizer also computed the right thing."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import synth  # noqa: E402
from helpers import gpu_scores, make_gpu, oracle_scores, parity_err, tolerance  # noqa: E402

CASES = {
    "tiny": (synth.preset("tiny", L=2), 1),
    "small": (synth.preset("small", B=2), 2),                      # tcgen05 GEMMs + SUMI d_h 32
    "medium": (synth.preset("medium", M=160, n_s=1024, n_s_max=1400), 1),  # tcgen05 history + SUMI, ragged
    "large": (synth.preset("large", M=130, L=2, n_s=2048), 1),     # d_h 64 kernels, 2 query tiles
}

for name in sys.argv[1:] or list(CASES):
    cfg, B = CASES[name]
    w = synth.make_weights(cfg, 0)
    batch = synth.make_batch(cfg, 1, B=B)
    cl = make_gpu(cfg, w, B)
    got = gpu_scores(cl, batch)
    cl.stream_status()
    ref = oracle_scores(cfg, w, batch, [0])[0]
    ab, rel = parity_err(got[:len(ref)], ref)
    assert ab <= tolerance(cfg) and rel <= tolerance(cfg), (name, ab, rel)
    print(f"{name}: ok (max abs {ab:.2e})", flush=True)
    cl.close()
