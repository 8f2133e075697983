"""Eager (non-graph) trainer steps for ncu: every kernel is a separate launch.
usage: python tools/profile_step.py [workload] [warmup] [steps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_15022_b200 import holo, synthetic as S

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 1
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
wl = S.workload(name)
cfg = wl["cfg"]; c, h, w, n = cfg["channels"], cfg["height"], cfg["width"], cfg["count"]
g32 = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in wl["gaussians"].items()}
tr = holo.Trainer(holo.GaussianSet(n, c, **g32), w, h, holo.RealField(c, h, w, wl["target"].astype(np.float32)),
                  wl["masks"], wl["distances"], holo.PropagationSpec(tuple(wl["wavelengths"])),
                  total_steps=warm + steps + 1)
for _ in range(warm + steps):
    tr.step(sync_loss=False)
print("loss", tr.last_loss())
