"""Times hs_trainer_step_host (graph and eager) against set_params + step + get_params at cfg2."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_15022_b200 import holo, synthetic as S
wl = S.workload("cfg2")
cfg = wl["cfg"]; c, h, w, n = cfg["channels"], cfg["height"], cfg["width"], cfg["count"]
g32 = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in wl["gaussians"].items()}
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    tr = holo.Trainer(holo.GaussianSet(n, c, **g32), w, h, holo.RealField(c, h, w, wl["target"].astype(np.float32)),
                      wl["masks"], wl["distances"], holo.PropagationSpec(tuple(wl["wavelengths"])), total_steps=1000)
    host = torch.from_numpy(tr.params()).pin_memory()
    lib = holo._lib.load()
    for graph in (True, False):
        tr.use_graph(graph)
        for _ in range(3):
            tr.step_host(host, host)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(30):
            tr.step_host(host, host)
        t1 = time.perf_counter()
        print(f"step_host graph={graph}: {(t1 - t0) / 30 * 1e3:.3f} ms")
    tr.use_graph(True)
    hp = holo.C.c_void_p(host.data_ptr())
    t0 = time.perf_counter()
    for _ in range(30):
        holo.check(lib.hs_trainer_set_params(tr.h, hp, 0)); tr.step(sync_loss=True); holo.check(lib.hs_trainer_get_params(tr.h, hp, 0))
    t1 = time.perf_counter()
    print(f"set+step+get graph: {(t1 - t0) / 30 * 1e3:.3f} ms")
    t0 = time.perf_counter()
    for _ in range(30):
        tr.step(sync_loss=True)
    t1 = time.perf_counter()
    print(f"device step + loss sync: {(t1 - t0) / 30 * 1e3:.3f} ms")
