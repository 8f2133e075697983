"""R virtual row-slab ranks on one GPU (parallel.LocalSlabGroup, peer-put),
one profiled step for ncu --profile-from-start off.
usage: python tools/slab_profile.py [workload] [R] [warmup]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_15022_b200 import holo, parallel as P, synthetic as S

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 8
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 3
wl = S.workload(name)
cfg = wl["cfg"]
C_, h, w, n, L = cfg["channels"], cfg["height"], cfg["width"], cfg["count"], cfg["planes"]
g32 = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in wl["gaussians"].items()}


def mk(r):
    t = holo.Trainer(holo.GaussianSet(n, C_, **g32), w, h,
                     holo.RealField(C_, h, w, wl["target"].astype(np.float32).astype(np.float64)),
                     wl["masks"], wl["distances"], holo.PropagationSpec(tuple(wl["wavelengths"])),
                     total_steps=warm + 10)
    t.set_row_slab(r, R)
    return t


grp = P.LocalSlabGroup([mk(r) for r in range(R)], C_, h, w, L, put=True)
for _ in range(warm):
    grp.step(with_loss=False)
torch.cuda.synchronize()
torch.cuda.profiler.start()
grp.step(with_loss=False)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("loss", grp.step())
