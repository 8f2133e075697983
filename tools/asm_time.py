"""Time the 1080p RGB single-plane ASM forward (rows, columns, rows) through
propagate_device with CUDA events; results are not checked (A/B of kernel
variants that may be numerically wrong).  usage: python tools/asm_time.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2511_15022_b200 import holo

c, h, w = 3, 1080, 1920
f = torch.randn(c, h, w, 2, device="cuda", dtype=torch.float32)
spec = holo.PropagationSpec((639e-9, 532e-9, 473e-9))
for _ in range(3):
    holo.propagate_device(f, spec, 2e-3, 0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    holo.propagate_device(f, spec, 2e-3, 0)
e1.record()
torch.cuda.synchronize()
print(f"asm forward 1080p x3: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
