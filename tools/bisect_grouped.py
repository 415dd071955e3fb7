import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, synth
from helpers import gpu_scores, make_gpu
cfg = synth.preset("small")
w = synth.make_weights(cfg, 0)
batch = synth.make_batch(cfg, 1, B=4)
os.environ["CLIMBER_GROUPED"] = "0"
cl = make_gpu(cfg, w, 4)
ref = gpu_scores(cl, batch)
os.environ["CLIMBER_GROUPED"] = "1"
for mask in (0, 1, 2, 4, 8, 16, 31):
    os.environ["CLIMBER_GROUPED_MASK"] = str(mask)
    got = gpu_scores(cl, batch)
    print(mask, float(np.abs(got - ref).max()))
