"""Trains cfg N steps with per-step loss sync; on a non-finite gradient dumps
the offending Gaussians and re-runs the stages standalone (debug helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_15022_b200 import holo, synthetic as S

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
graph = len(sys.argv) > 3 and sys.argv[3] == "graph"
wl = S.workload(name)
cfg = wl["cfg"]; c, h, w, n, L = cfg["channels"], cfg["height"], cfg["width"], cfg["count"], cfg["planes"]
g32 = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in wl["gaussians"].items()}
gs = holo.GaussianSet(n, c, **g32)
tr = holo.Trainer(gs, w, h, holo.RealField(c, h, w, wl["target"].astype(np.float32)), wl["masks"],
                  wl["distances"], holo.PropagationSpec(tuple(wl["wavelengths"])), total_steps=steps + 5)
tr.use_graph(graph)
prev = tr.params().copy()
for s in range(steps):
    try:
        loss = tr.step()
    except holo.HoloError as e:
        print("step", s, "error:", e)
        gr = tr.grads_tensor().cpu().numpy()
        bad = np.nonzero(~np.isfinite(gr))[0]
        print("bad grad idx", bad[:20], "count", bad.size)
        g = holo.GaussianSet.from_flat(prev.astype(np.float64), n, c)
        ids = sorted(set(int(i // 2) for i in bad[bad < 2 * n]))[:5]
        for i in ids:
            print("gaussian", i, {k: getattr(g, k)[[2*i, 2*i+1]] if k in ("pre_position", "pre_scale") else getattr(g, k)[i*c:(i+1)*c] if k in ("amplitude", "phase") else getattr(g, k)[i] for k in holo.GROUPS})
        break
    if s % 25 == 0 or s < 3:
        print("step", s, "loss", loss, flush=True)
    prev = tr.params().copy()
