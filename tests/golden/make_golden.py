"""Generates tests/golden/golden.npz from the reference itself (oracle/_ref =
the reference sources compiled by oracle/Makefile).  Run in the build
container (where /root/reference exists):  python tests/golden/make_golden.py

Every fixture stores its inputs and the reference's outputs, so the CPU tests
(oracle restatement) and the GPU tests (CUDA path) can check against the
reference without the reference being present.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def rounded(s):
    return ref.GaussianSet(s.count, s.channels, *[f32(a) for a in s.arrays()])


def main():
    out = {}
    # tile index + forward + backward on random_set fixtures (test_util.hpp:16-37)
    for i, (seed, n, c, w, h) in enumerate([(1, 9, 1, 26, 20), (4, 9, 3, 53, 41), (21, 12, 1, 55, 37),
                                            (12, 10, 2, 48, 36)]):
        s = rounded(ref.random_set(seed, n, c, w, h))
        out[f"r{i}_meta"] = np.array([n, c, w, h])
        out[f"r{i}_params"] = s.flat()
        ti = ref.build_tile_index(s, w, h)
        out[f"r{i}_tiles"], out[f"r{i}_ids"], out[f"r{i}_ranges"] = ti["tiles"], ti["ids"], ti["ranges"]
        re, im = ref.rasterize_forward(s, w, h)
        out[f"r{i}_fwd"] = np.stack([re, im])
        gre = f32(ref.random_real(seed + 40, c, h, w, -1.0, 1.0))
        gim = f32(ref.random_real(seed + 41, c, h, w, -1.0, 1.0))
        out[f"r{i}_gfield"] = np.stack([gre, gim])
        out[f"r{i}_bwd"] = ref.rasterize_backward(s, gre, gim).flat()
    # propagation (test_propagation.cpp fixtures)
    for i, (c, h, w, pad, ap, d) in enumerate([(1, 24, 32, 2, 0.0, 3e-3), (1, 9, 15, 1, 0.0, 1e-3),
                                               (1, 16, 16, 2, 6.5, 2e-3), (3, 16, 24, 2, 0.0, 5e-3)]):
        wl = {1: (532e-9,), 3: (639e-9, 532e-9, 473e-9)}[c]
        spec = ref.PropagationSpec(wl, 3.74e-6, pad, ap)
        re, im = ref.random_field(100 + i, c, h, w)
        re, im = f32(re), f32(im)
        out[f"p{i}_meta"] = np.array([c, h, w, pad, ap, d])
        out[f"p{i}_in"] = np.stack([re, im])
        out[f"p{i}_out"] = np.stack(ref.propagate(re, im, spec, d))
        out[f"p{i}_back"] = np.stack(ref.propagate(re, im, spec, d, mode=2))
    c, h, w = 3, 20, 28
    spec = ref.PropagationSpec()
    dist = [1e-3, 3e-3, 5e-3]
    re, im = ref.random_field(15, c, h, w)
    out["pm_in"] = np.stack([f32(re), f32(im)])
    ore, oim = ref.propagate_multi(f32(re), f32(im), spec, dist)
    out["pm_out"] = np.stack([ore, oim])
    gre = np.stack([f32(ref.random_field(30 + l, c, h, w)[0]) for l in range(3)])
    gim = np.stack([f32(ref.random_field(40 + l, c, h, w)[1]) for l in range(3)])
    out["pmb_in"] = np.stack([gre, gim])
    out["pmb_out"] = np.stack(ref.propagate_multi_backward(gre, gim, spec, dist))
    # loss (test_loss.cpp fixtures)
    for i, (c, h, w, L) in enumerate([(1, 16, 16, 2), (3, 32, 48, 2)]):
        img = f32(ref.random_real(7 + c, c, h, w, 0.0, 1.0))
        depth = ref.random_real(1007 + c, 1, h, w, 0.0, 1.0)[0]
        recon = f32(np.stack([ref.random_real(50 + l, c, h, w, 0.0, 1.0) for l in range(L)]))
        out[f"l{i}_target"], out[f"l{i}_depth"], out[f"l{i}_recon"] = img, depth, recon
        out[f"l{i}_masks"] = ref.build_masks(depth, L, True)
        for kind in ("training", "recon", "ssim", "mse"):
            v, g = ref.loss(kind, recon, img, depth)
            out[f"l{i}_{kind}_value"] = np.array([v])
            out[f"l{i}_{kind}_grad"] = g
    # full step (pipeline.cpp:253-297) on a small scene
    n, c, w, h, L = 120, 3, 48, 32, 2
    s = rounded(ref.init_gaussians(n, c, w, h, 42))
    target = f32(ref.synthetic_image(42, c, h, w))
    depth = ref.synthetic_depth(43, h, w)
    tr = ref.Trainer(s, w, h, target, depth, L, 3e-3, 2e-3, ref.PropagationSpec(), 8)
    loss, g = tr.step(want_grads=True)
    out["step_meta"] = np.array([n, c, w, h, L])
    out["step_params"] = s.flat()
    out["step_target"], out["step_depth"] = target, depth
    out["step_loss"] = np.array([loss])
    out["step_grads"] = g.flat()
    out["step_after"] = tr.params().flat()
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
