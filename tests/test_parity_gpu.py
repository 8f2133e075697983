"""GPU parity: the B200 kernels (through the C ABI) against the reference
library compiled from its own sources (oracle/_ref), on identical fp32-valued
inputs.  Bars (BASELINE.json north_star): tile binning and sort order
bit-exact; propagated field rel-L2 <= 1e-4; parameter gradients rel-L2 <= 1e-3.
"""
import numpy as np
import pytest

from paper_2511_15022_b200 import synthetic as S

pytestmark = pytest.mark.gpu

RASTER_TOL = 1e-4
FIELD_TOL = 1e-4
GRAD_TOL = 1e-3


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def f32(d):
    return {k: np.asarray(v, dtype=np.float32).astype(np.float64) for k, v in d.items()}


def sets(holo, ref, groups, n, c):
    hs = holo.GaussianSet(n, c, **groups)
    rs = ref.GaussianSet(n, c, *[np.ascontiguousarray(groups[k]) for k in ref.GROUPS])
    return hs, rs


CASES = [  # (seed, n, c, w, h)
    (1, 9, 1, 26, 20), (2, 9, 3, 35, 27), (3, 9, 1, 44, 34), (4, 9, 3, 53, 41),
    (11, 14, 3, 70, 50), (21, 12, 1, 55, 37), (31, 300, 2, 128, 96), (5, 2000, 3, 256, 160),
]


@pytest.mark.parametrize("seed,n,c,w,h", CASES)
def test_tile_index_bit_exact_random_set(holo, ref, seed, n, c, w, h):
    g = f32(S.random_set(seed, n, c))
    hs, rs = sets(holo, ref, g, n, c)
    a = holo.build_tile_index(hs, w, h)
    b = ref.build_tile_index(rs, w, h)
    assert (a.tiles_x, a.tiles_y) == (b["tiles_x"], b["tiles_y"])
    assert np.array_equal(a.pairs[:, 0], b["tiles"])
    assert np.array_equal(a.pairs[:, 1], b["ids"])
    assert np.array_equal(a.ranges, b["ranges"])


@pytest.mark.parametrize("n,c,w,h,seed", [(10_000, 1, 256, 256, 42), (3413, 1, 256, 160, 42),
                                          (50_000, 3, 960, 540, 42)])
def test_tile_index_bit_exact_init(holo, ref, n, c, w, h, seed):
    g = f32(S.init_gaussians(n, c, w, h, seed))
    hs, rs = sets(holo, ref, g, n, c)
    a = holo.build_tile_index(hs, w, h)
    b = ref.build_tile_index(rs, w, h)
    assert a.pairs.shape[0] == b["tiles"].shape[0]
    assert np.array_equal(a.pairs[:, 0], b["tiles"])
    assert np.array_equal(a.pairs[:, 1], b["ids"])
    assert np.array_equal(a.ranges, b["ranges"])


@pytest.mark.parametrize("seed,n,c,w,h", CASES)
def test_rasterize_forward(holo, ref, seed, n, c, w, h):
    g = f32(S.random_set(seed, n, c))
    hs, rs = sets(holo, ref, g, n, c)
    a = holo.rasterize_forward(hs, w, h)
    re, im = ref.rasterize_forward(rs, w, h)
    err = rel_l2(np.stack([a.real, a.imag]), np.stack([re, im]))
    assert err <= RASTER_TOL, err
    assert np.max(np.abs(a.real - re)) < 1e-5


def test_rasterize_forward_init_cfg1(holo, ref):
    n, c, w, h = 10_000, 1, 256, 256
    g = f32(S.init_gaussians(n, c, w, h, 42))
    hs, rs = sets(holo, ref, g, n, c)
    a = holo.rasterize_forward(hs, w, h)
    re, im = ref.rasterize_forward(rs, w, h)
    assert rel_l2(np.stack([a.real, a.imag]), np.stack([re, im])) <= RASTER_TOL


def test_empty_set_rasterizes_to_zeros(holo):
    f = holo.rasterize_forward(holo.GaussianSet(0, 2), 20, 10)
    assert not f.real.any() and not f.imag.any()


def test_high_opacity_tails(holo, ref):
    # test_rasterizer.cpp:76-92
    g = dict(pre_position=np.zeros(2), pre_scale=np.log([2.0, 2.0]), rotation=np.zeros(1),
             amplitude=np.ones(1), phase=np.zeros(1), pre_opacity=np.array([5.0]))
    g = f32(g)
    hs, rs = sets(holo, ref, g, 1, 1)
    a = holo.rasterize_forward(hs, 64, 64)
    re, im = ref.rasterize_forward(rs, 64, 64)
    assert np.max(np.abs(a.real - re)) <= 1e-6
    assert abs(a.real[0, 32, 39]) > 0.0


@pytest.mark.parametrize("tile", [False, True])
@pytest.mark.parametrize("seed,n,c,w,h", CASES)
def test_rasterize_backward(holo, ref, seed, n, c, w, h, tile):
    """Both backward forms (the deterministic gather and the per-tile backward
    with atomics) on canvases that are not whole tiles (partial edge cells)."""
    g = f32(S.random_set(seed, n, c))
    hs, rs = sets(holo, ref, g, n, c)
    wre = S.random_real(seed + 40, c, h, w, -1.0, 1.0).astype(np.float32).astype(np.float64)
    wim = S.random_real(seed + 41, c, h, w, -1.0, 1.0).astype(np.float32).astype(np.float64)
    holo.set_backward_deterministic(not tile)
    try:
        a = holo.rasterize_backward(hs, holo.RealField(c, h, w, wre), holo.RealField(c, h, w, wim))
    finally:
        holo.set_backward_deterministic(True)
    b = ref.rasterize_backward(rs, wre, wim)
    for k in ref.GROUPS:
        err = rel_l2(getattr(a, k), getattr(b, k))
        assert err <= GRAD_TOL, (k, err)


@pytest.mark.parametrize("tile", [False, True])
def test_saturation_gates(holo, tile):
    # test_rasterizer.cpp:225-244 (both backward forms: saturated pixels take the
    # per-tile backward's exact pass)
    holo.set_backward_deterministic(not tile)
    try:
        _saturation_gates(holo)
    finally:
        holo.set_backward_deterministic(True)


def _saturation_gates(holo):
    g = dict(pre_position=np.zeros(2), pre_scale=np.log([10.0, 10.0]), rotation=np.zeros(1),
             amplitude=np.ones(1), phase=np.array([0.3]), pre_opacity=np.array([8.0]))
    hs = holo.GaussianSet(1, 1, **f32(g))
    wre = np.zeros((1, 31, 31))
    wre[0, 15, 15] = 1.0
    gr = holo.rasterize_backward(hs, holo.RealField(1, 31, 31, wre), holo.RealField(1, 31, 31))
    assert gr.pre_opacity[0] == 0.0
    assert gr.pre_scale[0] == 0.0 and gr.pre_scale[1] == 0.0
    assert gr.pre_position[0] == 0.0
    assert gr.amplitude[0] != 0.0


def _knife_edge_set(c):
    """A Gaussian whose cutoff ellipse passes exactly through pixel centres:
    centre (32, 32) (pre-position 0 on a 64x64 canvas), Sigma = 2.5 I (scale
    sqrt(2.4) plus the 0.1 covariance epsilon) and alpha = e^5 / 255, so
    mahal = d^2 / 2.5 = 10 = 2 ln(255 alpha) for the pixels at distance 5
    ((3, 4), (5, 0), ...): the fp32 fast paths see them inside the error band
    and the fp64 decision of rasterizer.cpp:164-169 / :220-228 settles them.
    A second, high-opacity Gaussian (alpha ~ 0.9997, saturating near its centre)
    shares the tile, so a warp holds both the saturating and the band case.
    (The reference keeps the distance-5 pixels: alpha_eff = 1/255 there, so a
    fast path that dropped or mis-weighted them would miss the 1e-6 bar.)"""
    a = np.exp(5.0) / 255.0
    g = dict(pre_position=np.array([0.0, 0.0, np.arctanh(38 / 32 - 1), np.arctanh(29 / 32 - 1)]),
             pre_scale=np.log(np.array([np.sqrt(2.4) - 0.1] * 2 + [2.0, 1.5])),
             rotation=np.array([0.0, 0.4]),
             amplitude=np.linspace(0.3, 0.9, 2 * c), phase=np.linspace(-1.0, 2.0, 2 * c),
             pre_opacity=np.array([np.log(a / (1 - a)), 8.0]))
    return g


@pytest.mark.parametrize("c", [1, 3])
@pytest.mark.parametrize("tile", [False, True])
def test_band_pixels_decided_exactly(holo, ref, c, tile):
    g = f32(_knife_edge_set(c))
    # the fp32 mahalanobis distance of the distance-5 pixels lies inside the
    # band around the cutoff, i.e. the exact passes are exercised
    s2 = (np.float32(np.exp(np.float32(g["pre_scale"][0]))) + np.float32(0.1)) ** 2 + np.float32(0.1)
    m = np.float32(25.0) / np.float32(s2)
    assert abs(float(m) - 10.0) < 1e-5
    hs, rs = sets(holo, ref, g, 2, c)
    a = holo.rasterize_forward(hs, 64, 64)
    re, im = ref.rasterize_forward(rs, 64, 64)
    assert np.max(np.abs(a.real - re)) <= 1e-6 and np.max(np.abs(a.imag - im)) <= 1e-6
    wre = S.random_real(7, c, 64, 64, -1.0, 1.0).astype(np.float32).astype(np.float64)
    wim = S.random_real(8, c, 64, 64, -1.0, 1.0).astype(np.float32).astype(np.float64)
    holo.set_backward_deterministic(not tile)
    try:
        gr = holo.rasterize_backward(hs, holo.RealField(c, 64, 64, wre), holo.RealField(c, 64, 64, wim))
    finally:
        holo.set_backward_deterministic(True)
    want = ref.rasterize_backward(rs, wre, wim)
    for k in ref.GROUPS:
        assert rel_l2(getattr(gr, k), getattr(want, k)) <= 1e-5, k


def spec_for(holo, ref, channels, pad=2, aperture=0.0):
    wl = S.WAVELENGTHS[channels]
    return (holo.PropagationSpec(wl, 3.74e-6, pad, aperture), ref.PropagationSpec(wl, 3.74e-6, pad, aperture))


def field32(seed, c, h, w):
    re, im = S.random_field(seed, c, h, w)
    return re.astype(np.float32).astype(np.float64), im.astype(np.float32).astype(np.float64)


@pytest.mark.parametrize("c,h,w,pad,ap,d", [
    (1, 24, 32, 2, 0.0, 1e-3), (1, 24, 32, 2, 0.0, 1e-2), (3, 16, 24, 2, 0.0, 5e-3),
    (1, 16, 16, 2, 6.5, 2e-3), (1, 9, 15, 1, 0.0, 1e-3), (1, 10, 10, 3, 0.0, 2e-3),
    (3, 20, 28, 2, 0.0, 3e-3), (3, 96, 128, 2, 0.0, 3e-3), (1, 160, 256, 2, 0.0, 3e-3),
    (2, 37, 41, 2, 0.0, 4e-3),
])
def test_propagate(holo, ref, c, h, w, pad, ap, d):
    hsp, rsp = spec_for(holo, ref, c, pad, ap)
    re, im = field32(100 + h, c, h, w)
    a = holo.propagate(holo.ComplexField(c, h, w, re, im), hsp, d)
    b = ref.propagate(re, im, rsp, d)
    err = rel_l2(np.stack([a.real, a.imag]), np.stack(b))
    assert err <= FIELD_TOL, err


def test_propagate_backward_and_mask_distance(holo, ref):
    hsp, rsp = spec_for(holo, ref, 1, 1)
    re, im = field32(12, 1, 32, 32)
    u = holo.ComplexField(1, 32, 32, re, im)
    a = holo.propagate_backward(u, hsp, 4e-3)
    b = ref.propagate(re, im, rsp, 4e-3, mode=2)
    assert rel_l2(np.stack([a.real, a.imag]), np.stack(b)) <= FIELD_TOL
    a = holo.propagate_with_mask_distance(u, hsp, 2e-3, 6e-3)
    b = ref.propagate(re, im, rsp, 2e-3, mode=1, mask_distance=6e-3)
    assert rel_l2(np.stack([a.real, a.imag]), np.stack(b)) <= FIELD_TOL


def test_propagate_multi_and_backward(holo, ref):
    c, h, w = 3, 40, 56
    hsp, rsp = spec_for(holo, ref, c, 2)
    dist = [1e-3, 3e-3, 5e-3]
    re, im = field32(15, c, h, w)
    a = holo.propagate_multi(holo.ComplexField(c, h, w, re, im), hsp, dist)
    bre, bim = ref.propagate_multi(re, im, rsp, dist)
    for l in range(3):
        assert rel_l2(np.stack([a[l].real, a[l].imag]), np.stack([bre[l], bim[l]])) <= FIELD_TOL
    gre = np.stack([field32(30 + l, c, h, w)[0] for l in range(3)])
    gim = np.stack([field32(40 + l, c, h, w)[1] for l in range(3)])
    gs = [holo.ComplexField(c, h, w, gre[l], gim[l]) for l in range(3)]
    a = holo.propagate_multi_backward(gs, hsp, dist)
    b = ref.propagate_multi_backward(gre, gim, rsp, dist)
    assert rel_l2(np.stack([a.real, a.imag]), np.stack(b)) <= FIELD_TOL


@pytest.mark.parametrize("c,h,w,L", [(1, 256, 256, 1), (3, 160, 256, 2), (1, 1080, 1920, 2)])
def test_propagate_multi_static_plans(holo, ref, c, h, w, L):
    """The compile-time planned kernels (cfg1, desk, cfg2 grids), single- and multi-plane."""
    hsp, rsp = spec_for(holo, ref, c, 2)
    dist = S.make_depth_planes(L, 3e-3, 2e-3)
    re, im = field32(300 + h, c, h, w)
    a = holo.propagate_multi(holo.ComplexField(c, h, w, re, im), hsp, dist)
    bre, bim = ref.propagate_multi(re, im, rsp, dist)
    for l in range(L):
        assert rel_l2(np.stack([a[l].real, a[l].imag]), np.stack([bre[l], bim[l]])) <= FIELD_TOL
    gre = np.stack([field32(400 + l, c, h, w)[0] for l in range(L)])
    gim = np.stack([field32(500 + l, c, h, w)[1] for l in range(L)])
    b = holo.propagate_multi_backward([holo.ComplexField(c, h, w, gre[l], gim[l]) for l in range(L)], hsp, dist)
    r = ref.propagate_multi_backward(gre, gim, rsp, dist)
    assert rel_l2(np.stack([b.real, b.imag]), np.stack(r)) <= FIELD_TOL


@pytest.mark.parametrize("h,w,pad", [(512, 512, 1), (256, 256, 3)])
def test_static_grid_sizes_with_other_pads(holo, ref, h, w, pad):
    """A padded grid that has a compile-time plan but a pad factor other than 2
    must take the generic kernels (the planned ones prune for offset = P/4)."""
    hsp, rsp = spec_for(holo, ref, 1, pad)
    re, im = field32(91 + pad, 1, h, w)
    a = holo.propagate(holo.ComplexField(1, h, w, re, im), hsp, 3e-3)
    b = ref.propagate(re, im, rsp, 3e-3)
    assert rel_l2(np.stack([a.real, a.imag]), np.stack(b)) <= FIELD_TOL


@pytest.mark.parametrize("pitch,ap,d", [(1.0e-6, 0.0, 1e-3), (3.74e-6, 900.0, 3e-3)])
def test_cfg2_grid_band_limit_and_aperture(holo, ref, pitch, ap, d):
    """The pair-SIMD column kernel of the cfg2 grid on its fallback paths: a fine
    pitch makes q = (2 pi f / k)^2 exceed the series range (and activates the band
    limit), an aperture switches the transfer to the scalar form."""
    c, h, w = 1, 1080, 1920
    hsp = holo.PropagationSpec((532e-9,), pixel_pitch=pitch, pad_factor=2, aperture_radius=ap)
    rsp = ref.PropagationSpec((532e-9,), pixel_pitch=pitch, pad_factor=2, aperture_radius=ap)
    re, im = field32(79, c, h, w)
    a = holo.propagate(holo.ComplexField(c, h, w, re, im), hsp, d)
    b = ref.propagate(re, im, rsp, d)
    assert rel_l2(np.stack([a.real, a.imag]), np.stack(b)) <= FIELD_TOL
    a = holo.propagate_backward(holo.ComplexField(c, h, w, re, im), hsp, d)
    b = ref.propagate(re, im, rsp, d, mode=2)
    assert rel_l2(np.stack([a.real, a.imag]), np.stack(b)) <= FIELD_TOL


def test_propagate_4k_grid(holo, ref):
    """cfg4 padded grid (4320 x 7680, the CC=2 plan) for one channel, fwd and adjoint."""
    c, h, w = 1, 2160, 3840
    hsp, rsp = spec_for(holo, ref, c, 2)
    re, im = field32(78, c, h, w)
    a = holo.propagate(holo.ComplexField(c, h, w, re, im), hsp, 3e-3)
    b = ref.propagate(re, im, rsp, 3e-3)
    assert rel_l2(np.stack([a.real, a.imag]), np.stack(b)) <= FIELD_TOL
    a = holo.propagate_backward(holo.ComplexField(c, h, w, re, im), hsp, 3e-3)
    b = ref.propagate(re, im, rsp, 3e-3, mode=2)
    assert rel_l2(np.stack([a.real, a.imag]), np.stack(b)) <= FIELD_TOL


def test_propagate_cfg2_grid(holo, ref):
    """Full cfg2 padded grid (2160 x 3840) for one channel vs the reference."""
    c, h, w = 1, 1080, 1920
    hsp, rsp = spec_for(holo, ref, c, 2)
    re, im = field32(77, c, h, w)
    a = holo.propagate(holo.ComplexField(c, h, w, re, im), hsp, 3e-3)
    b = ref.propagate(re, im, rsp, 3e-3)
    assert rel_l2(np.stack([a.real, a.imag]), np.stack(b)) <= FIELD_TOL


@pytest.mark.parametrize("kind", ["training", "recon", "ssim", "mse"])
@pytest.mark.parametrize("c,h,w,L", [(1, 16, 16, 2), (3, 32, 48, 2), (3, 64, 80, 3)])
def test_loss(holo, ref, kind, c, h, w, L):
    img = S.random_real(7 + c, c, h, w, 0.0, 1.0).astype(np.float32).astype(np.float64)
    depth = S.random_real(1007 + c, 1, h, w, 0.0, 1.0)[0]
    recon = np.stack([S.random_real(50 + l, c, h, w, 0.0, 1.0) for l in range(L)])
    recon = recon.astype(np.float32).astype(np.float64)
    tgt = holo.make_target_stack(holo.RealField(c, h, w, img), holo.RealField(1, h, w, depth), L, True)
    grads = []
    v = holo._loss(kind, [holo.RealField(c, h, w, recon[l]) for l in range(L)], tgt, grads)
    rv, rg = ref.loss(kind, recon, img, depth)
    assert abs(v - rv) <= 1e-5 * max(1.0, abs(rv)), (v, rv)
    assert rel_l2(np.stack([g.values for g in grads]), rg) <= 1e-4


def test_adan_matches_reference_trajectory(holo, ref):
    # test_optimizer.cpp vector trajectory (fp32 device state)
    a = holo.Adan()
    a.add_group("xy", 2, 0.05)
    r = ref.Adan()
    r.add_group("xy", 2, 0.05)
    x = np.array([0.7, -0.3])
    xr = x.copy()
    for _ in range(4):
        a.step("xy", x, np.array([2.0 * x[0], np.cos(x[1])]))
        r.step("xy", xr, np.array([2.0 * xr[0], np.cos(xr[1])]))
    assert np.max(np.abs(x - xr)) < 1e-6


def test_adan_nonfinite_names_group(holo):
    a = holo.Adan()
    a.add_group("params", 2, 0.1)
    with pytest.raises(holo.HoloNonFinite, match="params"):
        a.step("params", np.zeros(2), np.array([np.nan, 0.0]))
    with pytest.raises(holo.HoloInvalidArgument):
        a.add_group("params", 2, 0.1)


@pytest.mark.parametrize("c,w,h,n,L", [(1, 64, 48, 400, 1), (3, 96, 64, 1500, 2), (3, 256, 160, 3413, 2)])
def test_full_step_matches_reference(holo, ref, c, w, h, n, L):
    g = f32(S.init_gaussians(n, c, w, h, 42))
    hs, rs = sets(holo, ref, g, n, c)
    target = S.synthetic_image(42, c, h, w).astype(np.float32).astype(np.float64)
    depth = S.synthetic_depth(43, h, w)
    masks = S.build_masks(depth, L, True)
    dist = S.make_depth_planes(L, 3e-3, 2e-3)
    wl = S.WAVELENGTHS[c]
    tr = holo.Trainer(hs, w, h, holo.RealField(c, h, w, target), masks, dist,
                      holo.PropagationSpec(wl), total_steps=20)
    rt = ref.Trainer(rs, w, h, target, depth, L, 3e-3, 2e-3, ref.PropagationSpec(wl), 20)
    tr.forward_backward()
    grads = tr.grads_tensor().cpu().numpy().astype(np.float64)
    tr.apply_update()
    loss = tr.last_loss()[0]
    rloss, rgrads = rt.step(want_grads=True)
    assert abs(loss - rloss) / abs(rloss) < 1e-4
    o = 0
    for k in ref.GROUPS:
        rgk = getattr(rgrads, k)
        err = rel_l2(grads[o:o + rgk.size], rgk)
        assert err <= GRAD_TOL, (k, err)
        o += rgk.size
    p0 = hs.flat()
    dp = tr.params().astype(np.float64) - p0
    dr = rt.params().flat() - p0
    assert rel_l2(dp, dr) <= 1e-2  # Adan's first step is ~lr*sign(g): tiny-g signs may flip


def test_trainer_graph_replay_matches_eager(holo):
    c, w, h, n, L = 3, 96, 64, 1500, 1
    g = f32(S.init_gaussians(n, c, w, h, 42))
    hs = holo.GaussianSet(n, c, **g)
    target = holo.RealField(c, h, w, S.synthetic_image(42, c, h, w))
    masks = S.build_masks(S.synthetic_depth(43, h, w), L, True)
    dist = S.make_depth_planes(L, 3e-3, 2e-3)
    a = holo.Trainer(hs, w, h, target, masks, dist, holo.PropagationSpec(), 50)
    b = holo.Trainer(hs, w, h, target, masks, dist, holo.PropagationSpec(), 50)
    for t in (a, b):
        t.set_deterministic(True)  # bit-for-bit needs the gather backward (no atomics)
    b.use_graph(True)
    la = [a.step() for _ in range(5)]
    lb = [b.step() for _ in range(5)]
    assert np.allclose(la, lb, rtol=0, atol=0)
    assert np.array_equal(a.params(), b.params())


def test_profiled_graph_step_matches_and_times_stages(holo):
    """Profiling with graphs on replays a second step graph that also records
    the stage events: the same results as the plain graph, and stage times
    that are positive and add up to the step."""
    c, w, h, n, L = 3, 96, 64, 1500, 2
    g = f32(S.init_gaussians(n, c, w, h, 42))
    target = holo.RealField(c, h, w, S.synthetic_image(42, c, h, w))
    masks = S.build_masks(S.synthetic_depth(43, h, w), L, True)
    dist = S.make_depth_planes(L, 3e-3, 2e-3)
    a, b = (holo.Trainer(holo.GaussianSet(n, c, **g), w, h, target, masks, dist, holo.PropagationSpec(), 50)
            for _ in range(2))
    for t in (a, b):
        t.set_deterministic(True)
        t.use_graph(True)
    b.set_profiling(True)
    for _ in range(3):
        la, lb = a.step(), b.step()
        assert la == lb
        st = b.stage_ms()
        parts = [v for k, v in st.items() if k != "total"]
        assert all(v > 0.0 for v in parts), st
        assert abs(sum(parts) - st["total"]) <= 1e-3 * st["total"] + 1e-3, st
    assert np.array_equal(a.params(), b.params())
    b.set_profiling(False)  # back to the plain step graph
    assert a.step() == b.step()


def test_tile_backward_matches_deterministic_gather(holo, ref):
    """The default per-tile backward (vector atomics into per-Gaussian rows)
    and the deterministic per-Gaussian gather give the same gradients to fp32
    summation-order noise, and both match the reference."""
    c, w, h, n, L = 3, 256, 160, 4000, 2
    g = f32(S.init_gaussians(n, c, w, h, 11))
    img = S.synthetic_image(42, c, h, w)
    depth = S.synthetic_depth(43, h, w)
    masks = S.build_masks(depth, L, True)
    dist = S.make_depth_planes(L, 3e-3, 2e-3)
    mk = lambda: holo.Trainer(holo.GaussianSet(n, c, **g), w, h, holo.RealField(c, h, w, img), masks, dist,
                              holo.PropagationSpec(), 20)
    a, b = mk(), mk()
    b.set_deterministic(True)
    ga, gb = [], []
    for t, out in ((a, ga), (b, gb)):
        t.forward_backward()
        out.append(t.grads_tensor().cpu().numpy().astype(np.float64))
    assert rel_l2(ga[0], gb[0]) < 1e-5, rel_l2(ga[0], gb[0])
    rs = ref.GaussianSet(n, c, *[np.ascontiguousarray(g[k]) for k in ref.GROUPS])
    rt = ref.Trainer(rs, w, h, img.astype(np.float32).astype(np.float64), depth, L, 3e-3, 2e-3,
                     ref.PropagationSpec(), 20)
    _, rgrads = rt.step(want_grads=True)
    want = np.concatenate([getattr(rgrads, k) for k in ref.GROUPS])
    o = 0
    for k, size in zip(ref.GROUPS, (2 * n, 2 * n, n, n * c, n * c, n)):
        assert rel_l2(ga[0][o:o + size], want[o:o + size]) <= 1e-3, k
        o += size


def test_plane_sharded_trainers_sum_to_full_step(holo):
    """Two trainers owning planes [0,2) and [2,4) (hs_trainer_config.plane_begin/end)
    produce gradients and loss partials that sum to the unsharded step's."""
    from paper_2511_15022_b200 import parallel as P
    c, w, h, n, L = 3, 96, 64, 1500, 4
    g = f32(S.init_gaussians(n, c, w, h, 42))
    hs = holo.GaussianSet(n, c, **g)
    target = holo.RealField(c, h, w, S.synthetic_image(42, c, h, w))
    masks = S.build_masks(S.synthetic_depth(43, h, w), L, True)
    dist = S.make_depth_planes(L, 3e-3, 4e-3 / 7)
    spec = holo.PropagationSpec()
    full = holo.Trainer(hs, w, h, target, masks, dist, spec, 10)
    full.set_deterministic(True)
    full.forward_backward()
    gfull = full.grads_tensor().cpu().numpy().astype(np.float64)
    pf = full.loss_partials()
    gs, parts = 0.0, np.zeros(2)
    for r in range(2):
        t = holo.Trainer(hs, w, h, target, masks, dist, spec, 10, plane_range=P.plane_shard(L, r, 2))
        t.set_deterministic(True)
        t.forward_backward()
        gs = gs + t.grads_tensor().cpu().numpy().astype(np.float64)
        parts += np.array(t.loss_partials())
    assert rel_l2(gs, gfull) < 1e-5
    assert parts[0] == pytest.approx(pf[0], rel=1e-6) and parts[1] == pytest.approx(pf[1], rel=1e-6)


def test_channel_sharded_trainers_match_full_step(holo):
    """Wavelength sharding: trainers owning channels [0,2) and [2,3) of a C=3
    scene (hs_trainer_config.channels_total = 3) give geometry gradients that
    sum to the full step's, amplitude/phase gradients equal to its columns, and
    loss partials that sum to its partials."""
    from paper_2511_15022_b200 import parallel as P
    c, w, h, n, L = 3, 96, 64, 1500, 2
    g = f32(S.init_gaussians(n, c, w, h, 42))
    img = S.synthetic_image(42, c, h, w)
    masks = S.build_masks(S.synthetic_depth(43, h, w), L, True)
    dist = S.make_depth_planes(L, 3e-3, 2e-3)
    wl = S.WAVELENGTHS[c]
    full = holo.Trainer(holo.GaussianSet(n, c, **g), w, h, holo.RealField(c, h, w, img), masks, dist,
                        holo.PropagationSpec(wl), 10)
    full.set_deterministic(True)
    full.forward_backward()
    gf = full.grads_tensor().cpu().numpy().astype(np.float64)
    pf = np.array(full.loss_partials())
    geo_sum, parts = 0.0, np.zeros(2)
    for r in range(2):
        b, e = P.channel_shard(c, r, 2)
        cl = e - b
        gs = P.slice_channels(g, n, c, b, e)
        t = holo.Trainer(holo.GaussianSet(n, cl, **gs), w, h, holo.RealField(cl, h, w, img[b:e]), masks, dist,
                         holo.PropagationSpec(wl[b:e]), 10, channels_total=c)
        t.set_deterministic(True)
        t.forward_backward()
        gr = t.grads_tensor().cpu().numpy().astype(np.float64)
        geo = np.concatenate([gr[lo:hi] for lo, hi in P.geometry_ranges(n, cl)])
        geo_sum = geo_sum + geo
        for k, off in (("amplitude", 5 * n), ("phase", 5 * n + n * c)):
            mine = gr[5 * n + (0 if k == "amplitude" else n * cl):][:n * cl].reshape(n, cl)
            ref = gf[off:off + n * c].reshape(n, c)[:, b:e]
            assert rel_l2(mine, ref) < 1e-5, k
        parts += np.array(t.loss_partials())
    geo_full = np.concatenate([gf[lo:hi] for lo, hi in P.geometry_ranges(n, c)])
    assert rel_l2(geo_sum, geo_full) < 1e-5
    assert parts[0] == pytest.approx(pf[0], rel=1e-6) and parts[1] == pytest.approx(pf[1], rel=1e-6)


def test_trainer_step_host_matches_device_step(holo):
    """hs_trainer_step_host (host-resident parameters, one sync) runs the same
    step as set_params + step + get_params."""
    import torch
    c, w, h, n, L = 3, 64, 48, 400, 1
    g = f32(S.init_gaussians(n, c, w, h, 5))
    img = S.synthetic_image(42, c, h, w)
    masks = S.build_masks(S.synthetic_depth(43, h, w), L, True)
    dist = S.make_depth_planes(L, 3e-3, 2e-3)
    mk = lambda: holo.Trainer(holo.GaussianSet(n, c, **g), w, h, holo.RealField(c, h, w, img), masks, dist,
                              holo.PropagationSpec(), 10)
    a, b = mk(), mk()
    for t in (a, b):
        t.set_deterministic(True)
    p0 = a.params()
    host = torch.from_numpy(p0.copy()).pin_memory()
    la = a.step(sync_loss=True)
    pa = a.params()
    lb = b.step_host(host, host)
    assert lb == la
    assert np.array_equal(host.numpy(), pa)


@pytest.mark.parametrize("graphs", [False, True])
def test_trainer_run_host_matches_device_steps(holo, graphs):
    """hs_trainer_run_host (host-resident parameters uploaded and downloaded
    every step, copies pipelined across steps) == the same number of device
    steps, bit for bit, losses included."""
    import torch
    c, w, h, n, L = 3, 64, 48, 400, 1
    g = f32(S.init_gaussians(n, c, w, h, 6))
    img = S.synthetic_image(42, c, h, w)
    masks = S.build_masks(S.synthetic_depth(43, h, w), L, True)
    dist = S.make_depth_planes(L, 3e-3, 2e-3)
    mk = lambda: holo.Trainer(holo.GaussianSet(n, c, **g), w, h, holo.RealField(c, h, w, img), masks, dist,
                              holo.PropagationSpec(), 20)
    a, b = mk(), mk()
    for t in (a, b):
        t.set_deterministic(True)
    b.use_graph(graphs)
    host = torch.from_numpy(b.params().copy()).pin_memory()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        la = [a.step(sync_loss=True) for _ in range(7)]
        lb = list(b.run_host(host, 3)) + list(b.run_host(host, 4))
    assert lb == la
    assert np.array_equal(host.numpy(), a.params())


def test_trainer_run_host_nonfinite_stops_updates(holo):
    """A non-finite gradient in the first step of a run raises naming the
    group (as step_host would), and no later step of the run moves the
    parameters: the host copy equals the initial parameters."""
    import torch
    c, w, h, n, L = 3, 64, 48, 300, 1
    g = f32(S.init_gaussians(n, c, w, h, 3))
    img = S.synthetic_image(42, c, h, w).copy()
    img[1, 10, 10] = np.nan
    masks = S.build_masks(S.synthetic_depth(43, h, w), L, True)
    tr = holo.Trainer(holo.GaussianSet(n, c, **g), w, h, holo.RealField(c, h, w, img), masks,
                      S.make_depth_planes(L, 3e-3, 2e-3), holo.PropagationSpec(), 10)
    tr.use_graph(True)
    p0 = tr.params()
    host = torch.from_numpy(p0.copy()).pin_memory()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        with pytest.raises(holo.HoloNonFinite, match="group position"):
            tr.run_host(host, 5)
    assert np.array_equal(host.numpy(), p0)
    assert np.array_equal(tr.params(), p0)


def test_reserve_pairs_recaptures_the_step_graphs(holo):
    """Growing the tile-pair capacity reallocates the id buffers: the captured
    step graphs (device step and host-resident step) must be re-captured, so
    graph-replayed steps keep matching eager steps bit for bit."""
    import torch
    c, w, h, n, L = 3, 64, 48, 400, 1
    g = f32(S.init_gaussians(n, c, w, h, 9))
    img = S.synthetic_image(42, c, h, w)
    masks = S.build_masks(S.synthetic_depth(43, h, w), L, True)
    dist = S.make_depth_planes(L, 3e-3, 2e-3)
    mk = lambda: holo.Trainer(holo.GaussianSet(n, c, **g), w, h, holo.RealField(c, h, w, img), masks, dist,
                              holo.PropagationSpec(), 10)
    eager, graphed = mk(), mk()
    for t in (eager, graphed):
        t.set_deterministic(True)
    graphed.use_graph(True)
    host = torch.from_numpy(graphed.params().copy()).pin_memory()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        for i in range(4):
            if i == 2:
                graphed.reserve_pairs(1 << 22)
            le = eager.step(sync_loss=True)
            lg = graphed.step_host(host, host)
            assert lg == le, (i, lg, le)
            assert np.array_equal(host.numpy(), eager.params()), i


def test_reserve_pairs_recaptures_the_run_graphs(holo):
    """The same for the pipelined host loop (hs_trainer_run_host): its captured
    first-step and steady-state graphs are dropped with the pair buffers."""
    import torch
    c, w, h, n, L = 3, 64, 48, 400, 1
    g = f32(S.init_gaussians(n, c, w, h, 9))
    img = S.synthetic_image(42, c, h, w)
    masks = S.build_masks(S.synthetic_depth(43, h, w), L, True)
    dist = S.make_depth_planes(L, 3e-3, 2e-3)
    mk = lambda: holo.Trainer(holo.GaussianSet(n, c, **g), w, h, holo.RealField(c, h, w, img), masks, dist,
                              holo.PropagationSpec(), 20)
    eager, graphed = mk(), mk()
    for t in (eager, graphed):
        t.set_deterministic(True)
    graphed.use_graph(True)
    host = torch.from_numpy(graphed.params().copy()).pin_memory()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        want = [eager.step(sync_loss=True) for _ in range(6)]
        got = list(graphed.run_host(host, 3))
        graphed.reserve_pairs(1 << 22)
        got += list(graphed.run_host(host, 3))
    assert got == want
    assert np.array_equal(host.numpy(), eager.params())


def test_trainer_nonfinite_gradient_raises_and_keeps_params(holo):
    """A NaN in the target poisons every gradient: like Adan::step on the first
    group (optimizer.cpp:52-54, groups named as pipeline.cpp:244-249) the step
    raises naming "position", and no group is updated."""
    c, w, h, n, L = 3, 64, 48, 300, 1
    g = f32(S.init_gaussians(n, c, w, h, 3))
    img = S.synthetic_image(42, c, h, w).copy()
    img[1, 10, 10] = np.nan
    masks = S.build_masks(S.synthetic_depth(43, h, w), L, True)
    tr = holo.Trainer(holo.GaussianSet(n, c, **g), w, h, holo.RealField(c, h, w, img), masks,
                      S.make_depth_planes(L, 3e-3, 2e-3), holo.PropagationSpec(), 10)
    p0 = tr.params()
    with pytest.raises(holo.HoloNonFinite, match="group position"):
        tr.step(sync_loss=True)
    assert np.array_equal(tr.params(), p0)
