"""GPU parity of the phase-only hologram conversion (SURVEY §8(f) rows 1-2,
proj/core/src/convert.cpp) against the reference compiled from its own sources
(oracle/_ref): DPAC encoding, poh_field and the guided random-POH loop."""
import math

import numpy as np
import pytest

from paper_2511_15022_b200 import synthetic as S

pytestmark = pytest.mark.gpu

TAU = 2.0 * math.pi


def phase_err(a, b):
    """RMS of the wrapped angle difference."""
    d = np.remainder(np.asarray(a) - np.asarray(b) + math.pi, TAU) - math.pi
    return float(np.sqrt(np.mean(d * d)))


def field32(seed, c, h, w):
    re = S.random_real(seed, c, h, w, -1.0, 1.0).astype(np.float32).astype(np.float64)
    im = S.random_real(seed + 1, c, h, w, -1.0, 1.0).astype(np.float32).astype(np.float64)
    return re, im


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("c,h,w", [(2, 10, 14), (3, 64, 96)])
def test_dpac_encode(holo, ref, mode, c, h, w):
    re, im = field32(3 + c, c, h, w)
    a = holo.dpac_encode(holo.ComplexField(c, h, w, re, im), mode)
    b = ref.dpac_encode(re, im, mode)
    assert a.format == holo.POH_SMOOTH
    assert np.all(a.phase.values >= 0.0) and np.all(a.phase.values < TAU)
    assert phase_err(a.phase.values, b) < 1e-5


def test_poh_field_unit_magnitude(holo, ref):
    c, h, w = 3, 12, 12
    ph = S.random_real(7, c, h, w, 0.0, TAU).astype(np.float32).astype(np.float64)
    u = holo.poh_field(holo.PhaseOnlyHologram(holo.RealField(c, h, w, ph)))
    re, im = ref.poh_field(ph)
    assert np.max(np.abs(np.hypot(u.real, u.imag) - 1.0)) < 1e-6
    assert np.max(np.abs(u.real - re)) < 1e-6 and np.max(np.abs(u.imag - im)) < 1e-6


@pytest.mark.parametrize("c,h,w,pad,L,steps,lc,lf", [
    (1, 16, 24, 1, 2, 8, 0.0, 0.0),      # test_convert.cpp:121-170 configuration (unguided)
    (1, 16, 16, 1, 2, 40, 0.1, 0.01),    # :172-190 (guided, default lambdas)
    (3, 32, 48, 2, 2, 12, 0.1, 0.01),    # RGB, pad 2 (the cfg5 setting)
])
def test_convert_random_poh_field(holo, ref, c, h, w, pad, L, steps, lc, lf):
    wl = S.WAVELENGTHS[c]
    re, im = field32(13 + c, c, h, w)
    img = S.random_real(11, c, h, w, 0.0, 1.0).astype(np.float32).astype(np.float64)
    depth = S.random_real(110, 1, h, w, 0.0, 1.0)[0]
    dist = S.make_depth_planes(L, 3e-3, 2e-3)
    hspec = holo.PropagationSpec(tuple(wl), pad_factor=pad)
    rspec = ref.PropagationSpec(tuple(wl), pad_factor=pad)
    tgt = holo.make_target_stack(holo.RealField(c, h, w, img), holo.RealField(1, h, w, depth[None]), L, True)
    opt = holo.RandomPohOptions(steps=steps, seed=77, lambda_comp=lc, lambda_field=lf, log_every=4)
    res = holo.convert_random_poh_field(holo.ComplexField(c, h, w, re, im), dist, tgt, hspec, opt)
    rph, rloss = ref.convert_random_poh_field(re, im, img, depth, L, dist, rspec, steps, seed=77, lambda_comp=lc,
                                              lambda_field=lf, log_every=4)
    assert res.poh.format == holo.POH_RANDOM
    assert np.all(res.poh.phase.values >= 0.0) and np.all(res.poh.phase.values < TAU)
    assert len(res.loss_history) == len(rloss)
    np.testing.assert_allclose(res.loss_history, rloss, rtol=2e-4)
    assert phase_err(res.poh.phase.values, rph) < 1e-3
    if lc or lf:
        assert res.loss_history[-1] < res.loss_history[0]


def test_convert_random_poh_rejects_inconsistent_inputs(holo):
    c, h, w = 1, 16, 16
    spec = holo.PropagationSpec((532e-9,), pad_factor=1)
    img = S.random_real(31, c, h, w, 0.0, 1.0)
    depth = S.random_real(130, 1, h, w, 0.0, 1.0)
    tgt = holo.make_target_stack(holo.RealField(c, h, w, img), holo.RealField(1, h, w, depth), 2, True)
    dist = S.make_depth_planes(2, 3e-3, 2e-3)
    re, im = field32(33, 1, 8, 8)
    with pytest.raises(ValueError):
        holo.convert_random_poh_field(holo.ComplexField(1, 8, 8, re, im), dist, tgt, spec)
    re, im = field32(34, c, h, w)
    ok = holo.ComplexField(c, h, w, re, im)
    with pytest.raises(ValueError):
        holo.convert_random_poh_field(ok, S.make_depth_planes(1, 3e-3, 0.0), tgt, spec)
    with pytest.raises(ValueError):
        holo.convert_random_poh_field(ok, dist, tgt, spec, holo.RandomPohOptions(steps=0))


# ---- end-of-run metrics (pipeline.cpp:135-163) -----------------------------
@pytest.mark.parametrize("L,c,h,w", [(2, 3, 32, 48), (1, 1, 40, 56)])
def test_compute_metrics(holo, ref, L, c, h, w):
    tgt = S.random_real(5, c, h, w, -0.1, 1.1).astype(np.float32).astype(np.float64)
    rec = np.stack([S.random_real(6 + l, c, h, w, -0.2, 1.2) for l in range(L)]).astype(np.float32).astype(
        np.float64)
    m = holo.compute_metrics([holo.RealField(c, h, w, rec[l]) for l in range(L)], holo.RealField(c, h, w, tgt))
    rp, rs = ref.compute_metrics(rec, tgt)
    np.testing.assert_allclose(m.psnr, rp, atol=1e-4)
    np.testing.assert_allclose(m.ssim, rs, atol=1e-5)
    assert m.mean_psnr == pytest.approx(float(np.mean(rp)), abs=1e-4)
    same = holo.compute_metrics([holo.RealField(c, h, w, tgt)], holo.RealField(c, h, w, tgt))
    assert same.psnr[0] == float("inf") and same.ssim[0] == pytest.approx(1.0, abs=1e-6)
    assert holo.psnr_value(holo.RealField(c, h, w, rec[0]), holo.RealField(c, h, w, tgt)) == pytest.approx(
        rp[0], abs=1e-9)
