"""Runs one cfg step stage by stage through the standalone C-ABI entry points
and reports non-finite values / magnitudes per stage (debug helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_15022_b200 import holo, synthetic as S

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
wl = S.workload(name)
cfg = wl["cfg"]; c, h, w, n, L = cfg["channels"], cfg["height"], cfg["width"], cfg["count"], cfg["planes"]
g32 = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in wl["gaussians"].items()}
gs = holo.GaussianSet(n, c, **g32)
p = gs.to_device()
spec = holo.PropagationSpec(tuple(wl["wavelengths"]))
def rep(tag, t):
    t = t.float()
    bad = (~torch.isfinite(t)).sum().item()
    print(f"{tag:12s} nonfinite={bad} absmax={t.abs().max().item():.4e} norm={t.norm().item():.4e}", flush=True)
f = holo.rasterize_forward_device(p, n, c, w, h); rep("raster", f)
U = holo.propagate_multi_device(f, spec, wl["distances"]); rep("U", U)
I = (U[..., 0] ** 2 + U[..., 1] ** 2).contiguous(); rep("I", I)
tgt = torch.from_numpy(wl["target"].astype(np.float32)).cuda()
m = torch.from_numpy(wl["masks"]).cuda()
for kind in ("recon", "ssim", "training"):
    v, g = holo.loss_device(kind, I, tgt, m); print(kind, v); rep("g_" + kind, g)
v, g = holo.loss_device("training", I, tgt, m)
if (~torch.isfinite(g)).any():
    idx = (~torch.isfinite(g)).nonzero()[:5]; print("bad idx", idx.tolist())
dU = torch.stack([2 * U[..., 0] * g, 2 * U[..., 1] * g], -1).contiguous(); rep("dU", dU)
back = holo.propagate_multi_backward_device(dU, spec, wl["distances"]); rep("back", back)
gr = holo.rasterize_backward_device(p, n, c, back); rep("grads", gr)
if (~torch.isfinite(gr)).any():
    idx = (~torch.isfinite(gr)).nonzero()[:10].flatten().tolist(); print("bad grad idx", idx, "N", n)
