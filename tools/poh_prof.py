"""Wall time of the device-resident random-POH loop (hs_convert_random_poh_field) at the
cfg5 grid for two step counts: the difference is the per-step cost.  usage: python tools/poh_prof.py [steps]"""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch, ctypes as C
from paper_2511_15022_b200 import holo, _lib, synthetic as S
wl = S.workload("cfg5", 0); cfg = wl["cfg"]; c, h, w, L = cfg["channels"], cfg["height"], cfg["width"], cfg["planes"]
spec = holo.PropagationSpec(tuple(wl["wavelengths"]))
field = torch.randn((c, h, w, 2), device="cuda")
lib = _lib.load()
def run(steps):
    phase = torch.from_numpy(holo.random_phase(1, c * h * w).astype(np.float32)).cuda()
    d = (C.c_double * L)(*wl["distances"])
    tgt = np.ascontiguousarray(wl["target"], dtype=np.float32); msk = np.ascontiguousarray(wl["masks"], dtype=np.uint8)
    pc = holo.hs_poh_config(c, h, w, L, C.cast(d, C.POINTER(C.c_double)), spec.c_struct(), tgt.ctypes.data_as(C.POINTER(C.c_float)),
                            msk.ctypes.data_as(C.POINTER(C.c_uint8)), steps, 0.1, 0.01, 2.5e-3)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    holo.check(lib.hs_convert_random_poh_field(holo.ctx_handle(), C.byref(pc), holo._ptr(field), holo._ptr(phase), None))
    torch.cuda.synchronize(); return time.perf_counter() - t0
run(5)
for s in (int(sys.argv[1]) if len(sys.argv) > 1 else 20, 100):
    print(s, "steps", round(run(s) * 1e3, 2), "ms")
