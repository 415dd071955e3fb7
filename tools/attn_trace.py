"""clock64 timeline of one SUMI attention launch (CLIMBER_ATTN_TRACE=n must be
set in the environment): encode + score a few users of a preset."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2502_09888_b200 import Climber, ModelConfig
name = sys.argv[1] if len(sys.argv) > 1 else "large"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cfg = synth.preset(name)
w = synth.make_weights(cfg, 0)
b = synth.make_batch(cfg, 1, B=B)
cl = Climber(ModelConfig.from_any(cfg), w, synth.strategies_for(cfg.N_b, cfg.R), max_users=B, kv_users=B)
for _ in range(2):
    cl.rank_host(b.ev_offsets, b.item, b.action, b.scenario, b.ts, b.r, b.cand_offsets, b.cand)
torch.cuda.synchronize()
