"""Measured tensor-core verdict for the column pass (north_star: tensor cores
only if a DFT-as-GEMM stage beats the bandwidth-bound FFT).

The cfg2 column pass transforms 3 x 3840 columns of length 2160 (forward FFT of
the 1080 live rows, x H, inverse FFT keeping 1080 rows).  As GEMMs on the
tensor cores, a length-2160 DFT is two Cooley-Tukey stages 2160 = N1 x N2 with
a twiddle multiply between them; a complex GEMM is one real GEMM on the
[[Ar, -Ai], [Ai, Ar]] block matrix.  This probe times, with cuBLAS (tcgen05 on
B200) and CUDA events, ONLY the GEMMs of the four stages of one column pass
(forward + inverse DFT, first forward stage pruned to the live rows, last
inverse stage to the kept rows) -- twiddles, the transfer multiply, layout
transposes and HBM staging excluded, so it is a lower bound for any
tensor-core column pass -- in each precision, and the rel-L2 error of a full
2160-point DFT against numpy's fp64 FFT in that precision:
  bf16 x1, bf16 x3 (hi/lo split, 3 products), tf32 x1, tf32 x3, fp32 (CUDA cores).
Prints one JSON line.  usage: python tools/tc_dft_probe.py [N1 N2]
"""
import json
import sys

import numpy as np
import torch

N = 2160
COLS = 3 * 3840


def dft_mat(n, sign=-1):
    k = np.arange(n)
    return np.exp(sign * 2j * np.pi * np.outer(k, k) / n)


def real_block(a):
    """complex (m x k) -> real (2m x 2k) [[Re, -Im], [Im, Re]]."""
    return np.block([[a.real, -a.imag], [a.imag, a.real]])


def to_tf32(x):
    """Round fp32 to tf32 (10 explicit mantissa bits), kept in an fp32 container."""
    xi = x.view(torch.int32)
    return ((xi + 0x1000) & ~0x1FFF).view(torch.float32)


def split(x, dt):
    hi = x.to(dt)
    lo = (x - hi.float()).to(dt)
    return hi, lo


def mm32(a, b):
    """bf16 operands, fp32 accumulation AND fp32 output (a bf16-rounded output
    would cap every split scheme at bf16 precision)."""
    return torch.mm(a, b, out_dtype=torch.float32)


def mm(a, b, mode):
    """a @ b (fp32 in/out) in a precision mode."""
    if mode == "fp32":
        torch.backends.cuda.matmul.allow_tf32 = False
        return a @ b
    if mode == "tf32x1":
        torch.backends.cuda.matmul.allow_tf32 = True
        return a @ b
    if mode == "tf32x3":
        torch.backends.cuda.matmul.allow_tf32 = True
        a_hi, b_hi = to_tf32(a), to_tf32(b)
        a_lo, b_lo = a - a_hi, b - b_hi
        return a_hi @ b_hi + a_hi @ b_lo + a_lo @ b_hi
    if mode == "bf16x1":
        return mm32(a.to(torch.bfloat16), b.to(torch.bfloat16))
    if mode == "bf16x3":
        ah, al = split(a, torch.bfloat16)
        bh, bl = split(b, torch.bfloat16)
        return mm32(ah, bh) + mm32(ah, bl) + mm32(al, bh)
    raise ValueError(mode)


def gemm_inputs(mode, a, b):
    """Pre-converted operands so the timed region holds only GEMMs."""
    if mode in ("fp32", "tf32x1"):
        return [(a, b)]
    if mode == "bf16x1":
        return [(a.to(torch.bfloat16), b.to(torch.bfloat16))]
    if mode == "bf16x3":
        ah, al = split(a, torch.bfloat16)
        bh, bl = split(b, torch.bfloat16)
        return [(ah, bh), (ah, bl), (al, bh)]
    if mode == "tf32x3":
        ah, bh = to_tf32(a), to_tf32(b)
        return [(ah, bh), (ah, b - bh), (a - ah, bh)]
    raise ValueError(mode)


def two_stage_dft(x, n1, n2, mode):
    """Length-N DFT of the columns of x (N x M complex128 numpy) with two GEMM
    stages in `mode`; returns complex128 numpy."""
    m = x.shape[1]
    dev = "cuda"
    A1 = torch.tensor(real_block(dft_mat(n1)), dtype=torch.float32, device=dev)
    A2 = torch.tensor(real_block(dft_mat(n2)), dtype=torch.float32, device=dev)
    # n = n2_count * n1 + n2 ;  x1[n1, (n2, col)]
    xr = x.reshape(n1, n2 * m)
    X = torch.tensor(np.concatenate([xr.real, xr.imag]), dtype=torch.float32, device=dev)
    Y = mm(A1, X, mode)  # (2 n1) x (n2 m): y[k1, n2, col]
    yr = (Y[:n1].double() + 1j * Y[n1:].double()).cpu().numpy().reshape(n1, n2, m)
    k1 = np.arange(n1)[:, None, None]
    nn2 = np.arange(n2)[None, :, None]
    yr = yr * np.exp(-2j * np.pi * k1 * nn2 / (n1 * n2))
    z = np.transpose(yr, (1, 0, 2)).reshape(n2, n1 * m)  # [n2, (k1, col)]
    Z = torch.tensor(np.concatenate([z.real, z.imag]), dtype=torch.float32, device=dev)
    W = mm(A2, Z, mode)  # (2 n2) x (n1 m): out[k2, k1, col], k = k1 + n1 k2
    w = (W[:n2].double() + 1j * W[n2:].double()).cpu().numpy().reshape(n2, n1, m)
    return w.reshape(n1 * n2, m)


def time_pass(n1, n2, mode, iters=20):
    """GEMM time of one cfg2 column pass: 4 stages over COLS columns; the first
    forward stage sees only the live half of the rows (K pruned by 2), the last
    inverse stage produces only the kept half of the outputs (M pruned by 2)."""
    dev = "cuda"
    shapes = [  # (M, K, Ncols) of the real block GEMMs
        (2 * n1, n1, n2 * COLS),       # fwd stage A, K = 2 n1 / 2 (live rows)
        (2 * n2, 2 * n2, n1 * COLS),   # fwd stage B
        (2 * n1, 2 * n1, n2 * COLS),   # inv stage A
        (n2, 2 * n2, n1 * COLS),       # inv stage B, only the kept half of the outputs
    ]
    ops = []
    for (M, K, Nc) in shapes:
        a = torch.randn(M, K, device=dev)
        b = torch.randn(K, Nc, device=dev)
        ops.append(gemm_inputs(mode, a, b))
    torch.backends.cuda.matmul.allow_tf32 = mode.startswith("tf32")

    def run():
        for pairs in ops:
            for a, b in pairs:
                if a.dtype == torch.bfloat16:
                    mm32(a, b)
                else:
                    torch.mm(a, b)

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        run()
    e1.record()
    e1.synchronize()
    flops = sum(2.0 * M * K * Nc for (M, K, Nc) in shapes) * len(ops[0])
    ms = e0.elapsed_time(e1) / iters
    return ms, flops / (ms * 1e-3) / 1e12


def main():
    n1, n2 = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (48, 45)
    assert n1 * n2 == N
    rng = np.random.default_rng(0)
    x = rng.standard_normal((N, 64)) + 1j * rng.standard_normal((N, 64))
    x[N // 4 + N // 2:] = 0
    x[:N // 4] = 0  # centred live half, like the padded column
    ref = np.fft.fft(x, axis=0)
    out = {"probe": "DFT-as-GEMM column pass (cfg2: 3 x 3840 columns of 2160)", "n1": n1, "n2": n2,
           "gpu": torch.cuda.get_device_name(), "modes": {}}
    for mode in ("bf16x1", "bf16x3", "tf32x1", "tf32x3", "fp32"):
        y = two_stage_dft(x, n1, n2, mode)
        err = float(np.linalg.norm(y - ref) / np.linalg.norm(ref))
        ms, tflops = time_pass(n1, n2, mode)
        out["modes"][mode] = {"dft_rel_l2": err, "gemm_ms_per_column_pass": ms, "achieved_tflops": tflops,
                              "meets_1e-4_after_4_stages": bool(err * 2 < 1e-4)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
