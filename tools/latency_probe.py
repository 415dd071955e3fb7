"""Where does one request's latency go?  Host wall time vs summed device time
of the library's kernels (CUDA events per launch) for B=1 requests."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2502_09888_b200 import Climber, ModelConfig
name = sys.argv[1] if len(sys.argv) > 1 else "large"
cfg = synth.preset(name)
w = synth.make_weights(cfg, 0)
batch = synth.make_batch(cfg, 1, B=8)
cl = Climber(ModelConfig.from_any(cfg), w, synth.strategies_for(cfg.N_b, cfg.R), max_users=8, kv_users=8)
reqs = [batch.subset([b]) for b in range(8)]
def one(u):
    return cl.rank_host(u.ev_offsets, u.item, u.action, u.scenario, u.ts, u.r, u.cand_offsets, u.cand)
for u in reqs[:3]: one(u)
torch.cuda.synchronize()
cl.profile(True)
n0 = cl.launch_count
t0 = time.perf_counter()
for u in reqs: one(u)
wall = (time.perf_counter() - t0) / len(reqs) * 1e3
cl.profile(False)
prof = cl.profile_read()
dev = sum(v["ms"] for v in prof.values()) / len(reqs)
print(json.dumps({"config": name, "wall_ms_per_request": wall, "device_ms_per_request": dev,
                  "launches_per_request": (cl.launch_count - n0) / len(reqs),
                  "by_class_ms": {k: round(v["ms"] / len(reqs), 3) for k, v in prof.items() if v["launches"]}}))
