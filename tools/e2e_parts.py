"""Diagnostic: cfg2 step_host with upload only / download only / both, and the
pipelined run_host, wall-clock per step (where the e2e time goes)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_15022_b200 import holo, synthetic as S

wl = S.workload("cfg2")
cfg = wl["cfg"]
c, h, w, n = cfg["channels"], cfg["height"], cfg["width"], cfg["count"]
g32 = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in wl["gaussians"].items()}
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    tr = holo.Trainer(holo.GaussianSet(n, c, **g32), w, h, holo.RealField(c, h, w, wl["target"].astype(np.float32)),
                      wl["masks"], wl["distances"], holo.PropagationSpec(tuple(wl["wavelengths"])), total_steps=2000)
    tr.use_graph(True)
    host = torch.empty(tr.param_count, dtype=torch.float32, pin_memory=True)
    host.copy_(torch.from_numpy(tr.params()))
    K = 50

    def timed(f):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(K):
            f()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / K * 1e3

    out = {
        "device_step_sync": timed(lambda: tr.step(sync_loss=True)),
        "upload_only": timed(lambda: tr.step_host(host, None)),
        "download_only": timed(lambda: tr.step_host(None, host)),
        "both": timed(lambda: tr.step_host(host, host)),
    }
    tr.run_host(host, 3)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr.run_host(host, K)
    torch.cuda.synchronize()
    out["run_host"] = (time.perf_counter() - t0) / K * 1e3
print({k: round(v, 3) for k, v in out.items()}, "ms per step")
