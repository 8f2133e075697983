"""PCIe copy probe: 9.6 MB (cfg2 parameters) H2D alone, D2H alone, both at once
on two streams, and chunked; pinned host memory, CUDA events.  One JSON line."""
import json
import torch

n = 2_400_000  # floats = 9.6 MB
h1 = torch.empty(n, dtype=torch.float32, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


def chunked(k):
    def f():
        for i in range(k):
            a, b = n * i // k, n * (i + 1) // k
            d1[a:b].copy_(h1[a:b], non_blocking=True)
    return f


out = {"bytes": 4 * n,
       "h2d_us": timed(lambda: d1.copy_(h1, non_blocking=True)),
       "d2h_us": timed(lambda: h2.copy_(d2, non_blocking=True)),
       "h2d_and_d2h_concurrent_us": timed(both),
       "h2d_4_chunks_us": timed(chunked(4)),
       "h2d_16_chunks_us": timed(chunked(16))}
out["h2d_GBps"] = out["bytes"] / out["h2d_us"] / 1e3
out["d2h_GBps"] = out["bytes"] / out["d2h_us"] / 1e3
print(json.dumps(out))
