"""GPU parity at the benchmarked sizes and over trajectories, against the
reference library compiled from its own sources (oracle/_ref):

* cfg2 (1920x1080x3, 200k Gaussians, L=1 -- the configuration bench.py times):
  one full step of pipeline.cpp:253-297 against RefTrainer (loss, per-group
  gradients, updated parameters), the raster field and bit-exact binning; the
  same step decomposed into channel shards and into row slabs (the multi-GPU
  decompositions of SURVEY 8(e)) against the same reference gradients.
* bit-exact build_tile_index (rasterizer.cpp:90-126) on TRAINED parameters
  (200 GPU steps at cfg2 and at cfg4) and on forced fixtures whose densest
  tile holds more than 512 and more than 4096 ids (the segmented sort paths).
* trajectories: a 200-step loss history against RefTrainer, and the
  reference's end-to-end desk regression (acceptance.cpp:303-370, criteria
  6/7: 256x160, two planes, 2000 steps, ratios 2/5/10) against the numbers the
  reference recorded (proj/test_output.txt:25-26) and against RefTrainer.

Bars (BASELINE.json north_star): binning bit-exact; raster / propagated field
rel-L2 <= 1e-4; gradients rel-L2 <= 1e-3.
"""
import os

import numpy as np
import pytest

from paper_2511_15022_b200 import synthetic as S

pytestmark = pytest.mark.gpu

FIELD_TOL = 1e-4
GRAD_TOL = 1e-3


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def f32(d):
    return {k: np.asarray(v, dtype=np.float32).astype(np.float64) for k, v in d.items()}


@pytest.fixture(scope="module", autouse=True)
def _ref_threads(ref):
    ref.set_thread_count(os.cpu_count() or 1)  # results are thread-count independent (rasterizer.hpp:27-29)


def split(ref, flat, n, c):
    out, o = {}, 0
    for k, size in zip(ref.GROUPS, (2 * n, 2 * n, n, n * c, n * c, n)):
        out[k] = np.asarray(flat[o:o + size], dtype=np.float64)
        o += size
    return out


def tile_index_equal(holo, ref, groups, n, c, w, h):
    hs = holo.GaussianSet(n, c, **groups)
    rs = ref.GaussianSet(n, c, *[np.ascontiguousarray(groups[k]) for k in ref.GROUPS])
    a = holo.build_tile_index(hs, w, h)
    b = ref.build_tile_index(rs, w, h)
    assert (a.tiles_x, a.tiles_y) == (b["tiles_x"], b["tiles_y"])
    assert a.pairs.shape[0] == b["tiles"].shape[0], (a.pairs.shape[0], b["tiles"].shape[0])
    cnt = np.diff(b["ranges"].reshape(-1, 2).astype(np.int64), axis=1)
    print(f"PARITY binning bit-exact: {n} Gaussians {w}x{h}, K={a.pairs.shape[0]}, max ids/tile {cnt.max()}")
    assert np.array_equal(a.pairs[:, 0], b["tiles"])
    assert np.array_equal(a.pairs[:, 1], b["ids"])
    assert np.array_equal(a.ranges, b["ranges"])
    return b


def field_ok(a, re, im):
    err = rel_l2(np.stack([a.real, a.imag]), np.stack([re, im]))
    print(f"PARITY raster field rel-L2 {err:.2e}")
    assert err <= FIELD_TOL


class Scene:
    def __init__(self, holo, ref, name, groups=None):
        wl = S.workload(name)
        cfg = wl["cfg"]
        self.w, self.h, self.c, self.n = cfg["width"], cfg["height"], cfg["channels"], cfg["count"]
        self.L, self.dz = cfg["planes"], cfg["dz"]
        self.g = f32(groups if groups is not None else wl["gaussians"])
        self.target = wl["target"].astype(np.float32).astype(np.float64)
        self.depth, self.masks, self.dist = wl["depth"], wl["masks"], wl["distances"]
        self.wl = wl["wavelengths"]
        self.holo, self.ref = holo, ref

    def trainer(self, total=20, groups=None, c_range=None):
        holo = self.holo
        g = self.g if groups is None else groups
        if c_range is None:
            return holo.Trainer(holo.GaussianSet(self.n, self.c, **g), self.w, self.h,
                                holo.RealField(self.c, self.h, self.w, self.target), self.masks, self.dist,
                                holo.PropagationSpec(self.wl), total)
        from paper_2511_15022_b200 import parallel as P
        b, e = c_range
        gs = P.slice_channels(g, self.n, self.c, b, e)
        return holo.Trainer(holo.GaussianSet(self.n, e - b, **gs), self.w, self.h,
                            holo.RealField(e - b, self.h, self.w, self.target[b:e]), self.masks, self.dist,
                            holo.PropagationSpec(self.wl[b:e]), total, channels_total=self.c)

    def ref_trainer(self, total=20, groups=None):
        ref = self.ref
        g = self.g if groups is None else groups
        rs = ref.GaussianSet(self.n, self.c, *[np.ascontiguousarray(g[k]) for k in ref.GROUPS])
        return ref.Trainer(rs, self.w, self.h, self.target, self.depth, self.L, 3e-3, self.dz,
                           ref.PropagationSpec(self.wl), total)


@pytest.fixture(scope="module")
def cfg2(holo, ref):
    sc = Scene(holo, ref, "cfg2")
    rt = sc.ref_trainer()
    rloss, rgrads = rt.step(want_grads=True)
    sc.rloss, sc.rgrads = rloss, np.concatenate([getattr(rgrads, k) for k in ref.GROUPS])
    sc.rparams = rt.params().flat()
    return sc


def check_grads(ref, got, want, n, c, tol=GRAD_TOL):
    o = 0
    errs = {}
    for k, size in zip(ref.GROUPS, (2 * n, 2 * n, n, n * c, n * c, n)):
        errs[k] = err = rel_l2(got[o:o + size], want[o:o + size])
        assert err <= tol, (k, err)
        o += size
    errs["all"] = rel_l2(got, want)
    print("PARITY grads rel-L2", {k: f"{v:.2e}" for k, v in errs.items()})
    assert errs["all"] <= tol


# ---------------------------------------------------------------------------------------------
# cfg2: the benchmarked step against the reference
# ---------------------------------------------------------------------------------------------
def test_cfg2_binning_and_raster_field(cfg2, holo, ref):
    sc = cfg2
    tile_index_equal(holo, ref, sc.g, sc.n, sc.c, sc.w, sc.h)
    rs = ref.GaussianSet(sc.n, sc.c, *[np.ascontiguousarray(sc.g[k]) for k in ref.GROUPS])
    a = holo.rasterize_forward(holo.GaussianSet(sc.n, sc.c, **sc.g), sc.w, sc.h)
    re, im = ref.rasterize_forward(rs, sc.w, sc.h)
    field_ok(a, re, im)


def test_cfg2_full_step_matches_reference(cfg2, holo, ref):
    sc = cfg2
    tr = sc.trainer()
    tr.forward_backward()
    grads = tr.grads_tensor().cpu().numpy().astype(np.float64)
    tr.apply_update()
    loss = tr.last_loss()[0]
    print(f"PARITY cfg2 loss {loss:.9g} ref {sc.rloss:.9g} rel {abs(loss - sc.rloss) / abs(sc.rloss):.2e}")
    assert abs(loss - sc.rloss) / abs(sc.rloss) < 1e-4, (loss, sc.rloss)
    check_grads(ref, grads, sc.rgrads, sc.n, sc.c)
    p0 = np.concatenate([sc.g[k] for k in ref.GROUPS])
    dp = tr.params().astype(np.float64) - p0
    dr = sc.rparams - p0
    # Adan's first update is ~lr * g / (|g| + eps): parameters whose gradient is
    # within fp32 noise of zero may flip sign, so the step is compared in rel-L2.
    print(f"PARITY cfg2 update rel-L2 {rel_l2(dp, dr):.2e}")
    assert rel_l2(dp, dr) <= 1e-2
    # Where the reference gradient stands clear of that noise (above 1e-3 of
    # its group's largest magnitude) the update must agree to fp32 precision:
    # the remaining error is the fp32 rounding of p + delta.
    o, worst = 0, 0.0
    for k, size in zip(ref.GROUPS, (2 * sc.n, 2 * sc.n, sc.n, sc.n * sc.c, sc.n * sc.c, sc.n)):
        gr = sc.rgrads[o:o + size]
        m = np.abs(gr) > 1e-3 * np.abs(gr).max()
        e = rel_l2(dp[o:o + size][m], dr[o:o + size][m])
        worst = max(worst, e)
        print(f"PARITY cfg2 update {k}: {m.mean():.3f} of the entries, rel-L2 {e:.2e}")
        o += size
    assert worst <= 1e-3, worst


def test_cfg2_graph_step_matches_reference(cfg2, holo):
    """The graph-captured step bench.py times (use_graph) gives the same loss."""
    tr = cfg2.trainer()
    tr.use_graph(True)
    loss = tr.step(sync_loss=True)
    assert abs(loss - cfg2.rloss) / abs(cfg2.rloss) < 1e-4


def test_cfg2_channel_shards_match_reference(cfg2, holo, ref):
    """Wavelength sharding over 3 ranks: summed geometry
    gradients and per-rank amplitude/phase columns against the reference step."""
    from paper_2511_15022_b200 import parallel as P
    sc = cfg2
    n, c = sc.n, sc.c
    want = split(ref, sc.rgrads, n, c)
    geo_sum, parts = 0.0, np.zeros(2)
    for r in range(3):
        b, e = P.channel_shard(c, r, 3)
        t = sc.trainer(c_range=(b, e))
        t.forward_backward()
        gr = t.grads_tensor().cpu().numpy().astype(np.float64)
        geo_sum = geo_sum + np.concatenate([gr[lo:hi] for lo, hi in P.geometry_ranges(n, e - b)])
        cl = e - b
        amp = gr[5 * n:5 * n + n * cl].reshape(n, cl)
        ph = gr[5 * n + n * cl:5 * n + 2 * n * cl].reshape(n, cl)
        assert rel_l2(amp, want["amplitude"].reshape(n, c)[:, b:e]) <= GRAD_TOL
        assert rel_l2(ph, want["phase"].reshape(n, c)[:, b:e]) <= GRAD_TOL
        parts += np.array(t.loss_partials())
        del t
    geo_ref = np.concatenate([sc.rgrads[lo:hi] for lo, hi in P.geometry_ranges(n, c)])
    assert rel_l2(geo_sum, geo_ref) <= GRAD_TOL
    loss = P.combine_loss(parts[0], parts[1], c, sc.h, sc.w, sc.L)
    assert abs(loss - sc.rloss) / abs(sc.rloss) < 1e-4


@pytest.mark.parametrize("R", [4])
def test_cfg2_row_slabs_match_reference(cfg2, holo, ref, R):
    """Row slabs (distributed 2D FFT, SURVEY 8(e) cfg4 scheme) at cfg2 over R
    ranks with the peer-put exchange: summed gradients against the reference."""
    from paper_2511_15022_b200 import parallel as P
    sc = cfg2
    trs = []
    for r in range(R):
        t = sc.trainer()
        t.set_row_slab(r, R)
        trs.append(t)
    grp = P.LocalSlabGroup(trs, sc.c, sc.h, sc.w, sc.L, put=True)
    loss = grp.step(with_loss=True)
    got = trs[0].grads_tensor().cpu().numpy().astype(np.float64)
    check_grads(ref, got, sc.rgrads, sc.n, sc.c)
    assert abs(loss - sc.rloss) / abs(sc.rloss) < 1e-4


# ---------------------------------------------------------------------------------------------
# binning on trained parameters and on dense tiles
# ---------------------------------------------------------------------------------------------
def trained(holo, ref, name, steps):
    sc = Scene(holo, ref, name)
    tr = sc.trainer(total=2000)
    tr.use_graph(True)
    for _ in range(steps):
        tr.step(sync_loss=False)
    g = split(ref, tr.params().astype(np.float64), sc.n, sc.c)
    return sc, g


def test_cfg2_trained_binning_raster_and_gradients(holo, ref):
    """After 200 GPU steps at cfg2 the Gaussians have moved, rescaled, rotated
    and changed opacity: the tile lists stay bit-exact, the field and the full
    step's gradients (from the trained state) stay within the bars."""
    sc, g = trained(holo, ref, "cfg2", 200)
    b = tile_index_equal(holo, ref, g, sc.n, sc.c, sc.w, sc.h)
    counts = np.diff(b["ranges"].reshape(-1, 2), axis=1).ravel()
    assert counts.max() > 0
    rs = ref.GaussianSet(sc.n, sc.c, *[np.ascontiguousarray(g[k]) for k in ref.GROUPS])
    a = holo.rasterize_forward(holo.GaussianSet(sc.n, sc.c, **g), sc.w, sc.h)
    re, im = ref.rasterize_forward(rs, sc.w, sc.h)
    field_ok(a, re, im)
    tr = sc.trainer(groups=g)
    tr.forward_backward()
    grads = tr.grads_tensor().cpu().numpy().astype(np.float64)
    loss = tr.last_loss()[0]
    rloss, rg = sc.ref_trainer(groups=g).step(want_grads=True)
    assert abs(loss - rloss) / abs(rloss) < 1e-4
    check_grads(ref, grads, np.concatenate([getattr(rg, k) for k in ref.GROUPS]), sc.n, sc.c)


def test_cfg4_trained_binning(holo, ref):
    """cfg4 (3840x2160x3, 1M Gaussians) after 200 GPU steps: bit-exact tile lists."""
    sc, g = trained(holo, ref, "cfg4", 200)
    tile_index_equal(holo, ref, g, sc.n, sc.c, sc.w, sc.h)


def dense_tile_set(count, c, w, h, seed, cx, cy):
    """`count` small Gaussians centred inside the 16x16 tile at (cx, cy) (ids in
    random spatial order), plus a sparse random background."""
    rng = S.Rng(seed)
    u = rng.uniform(count * (6 + 2 * c)).reshape(count, 6 + 2 * c)
    x = cx * 16 + 16.0 * u[:, 0]
    y = cy * 16 + 16.0 * u[:, 1]
    pos = np.empty(2 * count)
    pos[0::2] = S.unactivate_position(x, w)
    pos[1::2] = S.unactivate_position(y, h)
    sc = np.empty(2 * count)
    sc[0::2] = np.log(0.2 + 0.8 * u[:, 2])
    sc[1::2] = np.log(0.2 + 0.8 * u[:, 3])
    g = dict(pre_position=pos, pre_scale=sc, rotation=-3.2 + 6.4 * u[:, 4], amplitude=(0.05 * u[:, 6::2]).ravel(),
             phase=(-3.2 + 6.4 * u[:, 7::2]).ravel(), pre_opacity=-4.0 + 2.0 * u[:, 5])
    return f32(g)


@pytest.mark.parametrize("count", [700, 5000, 12000])
def test_dense_tile_binning_raster_and_gradients(holo, ref, count):
    """One tile holding > 512 (segment sort) and > 4096 (global sort) ids."""
    c, w, h = 2, 96, 80
    g = dense_tile_set(count, c, w, h, 100 + count, 2, 2)
    b = tile_index_equal(holo, ref, g, count, c, w, h)
    counts = np.diff(b["ranges"].reshape(-1, 2), axis=1).ravel()
    assert counts.max() > (4096 if count > 5000 else 512), counts.max()
    hs = holo.GaussianSet(count, c, **g)
    rs = ref.GaussianSet(count, c, *[np.ascontiguousarray(g[k]) for k in ref.GROUPS])
    a = holo.rasterize_forward(hs, w, h)
    re, im = ref.rasterize_forward(rs, w, h)
    field_ok(a, re, im)
    wre = S.random_real(7, c, h, w, -1.0, 1.0).astype(np.float32).astype(np.float64)
    wim = S.random_real(8, c, h, w, -1.0, 1.0).astype(np.float32).astype(np.float64)
    ga = holo.rasterize_backward(hs, holo.RealField(c, h, w, wre), holo.RealField(c, h, w, wim))
    gb = ref.rasterize_backward(rs, wre, wim)
    for k in ref.GROUPS:
        assert rel_l2(getattr(ga, k), getattr(gb, k)) <= GRAD_TOL, k


# ---------------------------------------------------------------------------------------------
# trajectories
# ---------------------------------------------------------------------------------------------
def desk_trainers(holo, ref, ratio, steps):
    d = S.desk_scene(ratio)
    n, c, w, h = d["count"], d["channels"], d["width"], d["height"]
    g = f32(d["gaussians"])
    target = d["target"].astype(np.float32).astype(np.float64)
    tr = holo.Trainer(holo.GaussianSet(n, c, **g), w, h, holo.RealField(c, h, w, target), d["masks"],
                      d["distances"], holo.PropagationSpec(d["wavelengths"]), steps)
    rs = ref.GaussianSet(n, c, *[np.ascontiguousarray(g[k]) for k in ref.GROUPS])
    rt = ref.Trainer(rs, w, h, target, d["depth"], 2, 3e-3, 2e-3, ref.PropagationSpec(d["wavelengths"]), steps)
    return d, tr, rt, target


def test_loss_history_200_steps_matches_reference(holo, ref):
    """The desk scene (ratio 2) stepped 200 times on both sides with the
    2000-step schedule: every step's loss within 1e-3 relative."""
    d, tr, rt, _ = desk_trainers(holo, ref, 2.0, 2000)
    worst = 0.0
    for s in range(200):
        lg = tr.step(sync_loss=True)
        lr = rt.step()
        worst = max(worst, abs(lg - lr) / abs(lr))
    p = tr.params().astype(np.float64)
    rp = rt.params().flat()
    print(f"PARITY 200-step loss history: worst rel {worst:.2e}, params rel-L2 {rel_l2(p, rp):.2e}")
    assert worst < 1e-3, worst
    assert rel_l2(p, rp) < 1e-2


def metrics(holo, tr, d, target):
    n, c, w, h = d["count"], d["channels"], d["width"], d["height"]
    gs = tr.gaussians()
    field = holo.rasterize_forward(gs, w, h)
    outs = holo.propagate_multi(field, holo.PropagationSpec(d["wavelengths"]), d["distances"])
    recon = [holo.intensity_of(u) for u in outs]
    return holo.compute_metrics(recon, holo.RealField(c, h, w, target))


# proj/test_output.txt:25-26 (acceptance criteria 6 and 7, the reference's recorded run)
DESK_PSNR = {2.0: 32.86, 5.0: 32.17, 10.0: 31.22}
DESK_SSIM_R2 = 0.947


@pytest.mark.parametrize("ratio", [2.0, 5.0, 10.0])
def test_desk_regression_matches_reference_run(holo, ref, ratio):
    """acceptance.cpp:303-370: 2000 steps of the desk scene; mean PSNR (and SSIM
    at ratio 2) of the two reconstructed planes within 0.1 dB (0.005) of the
    reference's recorded values, and PSNR non-increasing in the ratio."""
    # deterministic backward: the 2000-step trajectory is reproducible run to
    # run (the default per-tile backward's atomic order adds fp32 noise that a
    # 2000-step optimisation amplifies; that run is held to a wider band)
    for det, tol in ((True, 0.1), (False, 0.3)):
        d, tr, _, target = desk_trainers(holo, ref, ratio, 2000)
        tr.set_deterministic(det)
        tr.use_graph(True)
        for _ in range(d["steps"]):
            tr.step(sync_loss=False)
        m = metrics(holo, tr, d, target)
        print(f"PARITY desk ratio {ratio} ({'gather' if det else 'tile'} backward): mean PSNR {m.mean_psnr:.4f} dB "
              f"(reference run {DESK_PSNR[ratio]}), mean SSIM {m.mean_ssim:.4f}")
        assert abs(m.mean_psnr - DESK_PSNR[ratio]) <= tol, (ratio, det, m.mean_psnr)
        if ratio == 2.0:
            assert abs(m.mean_ssim - DESK_SSIM_R2) <= 0.005, m.mean_ssim


def _field_with_binning(holo, g, n, c, w, h, tight):
    import ctypes as C
    from paper_2511_15022_b200 import _lib
    holo.check(_lib.load().hs_ctx_set_tight_binning(holo.ctx_handle(), int(tight)))
    try:
        return holo.rasterize_forward(holo.GaussianSet(n, c, **g), w, h)
    finally:
        holo.check(_lib.load().hs_ctx_set_tight_binning(holo.ctx_handle(), 1))


@pytest.mark.parametrize("state", ["init", "trained"])
def test_tight_binning_field_is_bit_identical(holo, ref, state):
    """The trainer bins tightly (only tiles the ellipse can reach): the forward
    field is bit-identical to binning with the reference's box lists, with
    fewer (tile, Gaussian) pairs."""
    if state == "init":
        sc = Scene(holo, ref, "cfg2")
        g = sc.g
    else:
        sc, g = trained(holo, ref, "cfg2", 200)
    a = _field_with_binning(holo, g, sc.n, sc.c, sc.w, sc.h, True)
    b = _field_with_binning(holo, g, sc.n, sc.c, sc.w, sc.h, False)
    assert np.array_equal(a.real, b.real) and np.array_equal(a.imag, b.imag)
    tr = sc.trainer(groups=g)
    tr.forward_backward()
    k_tight = tr.last_loss()[1]
    k_ref = holo.build_tile_index(holo.GaussianSet(sc.n, sc.c, **g), sc.w, sc.h).pairs.shape[0]
    print(f"PARITY tight binning ({state}): field bit-identical, pairs {k_tight} vs reference {k_ref}")
    assert k_tight < k_ref
