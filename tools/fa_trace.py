"""clock64 timeline of one attention launch of the two-tile kernel
(CLIMBER_FA_TRACE=n selects the n-th SUMI launch of the process): encode +
score one wave of users of a preset, eagerly (no CUDA graph)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import synth  # noqa: E402
from paper_2502_09888_b200 import Climber, ModelConfig  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "large"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
cfg = synth.preset(name, L=2, rel_bias=int(sys.argv[3]) if len(sys.argv) > 3 else 0)
w = synth.make_weights(cfg, 0)
b = synth.make_batch(cfg, 1, B=B)
cl = Climber(ModelConfig.from_any(cfg), w, synth.strategies_for(cfg.N_b, cfg.R), max_users=B, kv_users=B)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
ev = [dev(a) for a in (b.item, b.action, b.scenario, b.ts)]
hs = cl.encode_users(b.ev_offsets, *ev, b.r)
cl.score_batched(hs, b.cand_offsets, dev(b.cand))
torch.cuda.synchronize()
