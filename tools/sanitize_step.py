"""One trainer step (and one 1080p propagation) for compute-sanitizer runs on
the compile-time planned kernels.  usage: python tools/sanitize_step.py {cfg1|runhost|prop1080}"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_15022_b200 import holo, synthetic as S  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
if what == "cfg1":
    wl = S.workload("cfg1")
    cfg = wl["cfg"]
    c, h, w, n = cfg["channels"], cfg["height"], cfg["width"], cfg["count"]
    g = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in wl["gaussians"].items()}
    tr = holo.Trainer(holo.GaussianSet(n, c, **g), w, h, holo.RealField(c, h, w, wl["target"].astype(np.float32)),
                      wl["masks"], wl["distances"], holo.PropagationSpec(tuple(wl["wavelengths"])), 5)
    print("loss", tr.step())
elif what == "runhost":  # the per-tile backward (default) + the pipelined host loop at cfg1
    wl = S.workload("cfg1")
    cfg = wl["cfg"]
    c, h, w, n = cfg["channels"], cfg["height"], cfg["width"], cfg["count"]
    g = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in wl["gaussians"].items()}
    tr = holo.Trainer(holo.GaussianSet(n, c, **g), w, h, holo.RealField(c, h, w, wl["target"].astype(np.float32)),
                      wl["masks"], wl["distances"], holo.PropagationSpec(tuple(wl["wavelengths"])), 10)
    host = torch.from_numpy(tr.params().copy()).pin_memory()
    print("losses", tr.run_host(host, 3))
else:
    f = torch.randn((3, 1080, 1920, 2), device="cuda")
    out = holo.propagate_multi_device(f, holo.PropagationSpec(), [3e-3])
    back = holo.propagate_multi_backward_device(out, holo.PropagationSpec(), [3e-3])
    torch.cuda.synchronize()
    print("ok", float(back.abs().sum()))
