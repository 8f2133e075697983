"""CPU: pin the oracle restatement (oracle/holo_oracle.py) against
(1) the known-answer tests of the reference's own test-suite and
(2) golden vectors produced by the reference itself (tests/golden/golden.npz,
    generated from oracle/_ref by tests/golden/make_golden.py).
"""
import math
import os

import numpy as np
import pytest

from oracle import holo_oracle as O

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def rel_l2(a, b):
    a, b = np.ravel(a), np.ravel(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ---- known-answer tests (proj/tests/*.cpp) -------------------------------------------------
def test_activation_kats():
    # test_field_core.cpp:13-14, :43-44, :54-55
    assert O.activate_position(1.0, 100.0) == pytest.approx(88.079707797788245, rel=1e-12)
    assert O.activate_position(-1.0, 100.0) == pytest.approx(11.920292202211758, rel=1e-12)
    assert O.activate_position(0.0, 64.0) == pytest.approx(32.0)
    assert O.activate_position(-30.0, 41.0) == 0.0 and O.activate_position(30.0, 41.0) == 41.0
    assert O.activate_scale(-3.0) == pytest.approx(0.14978706836786394, rel=1e-12)
    assert O.activate_scale(2.0) == pytest.approx(7.489056098930650, rel=1e-12)
    assert O.activate_opacity(-0.5) == pytest.approx(0.37754066879814541, rel=1e-12)
    assert O.activate_opacity(10.0) == pytest.approx(0.99995460213129761, rel=1e-12)
    assert O.activate_amplitude(-0.3) == 0.0 and O.activate_amplitude(1.7) == 1.0
    assert O.activate_amplitude_deriv(0.4) == 1.0 and O.activate_amplitude_deriv(1.7) == 0.0
    for bad in (O.activate_position, O.activate_opacity):
        with pytest.raises(ValueError):
            bad(float("nan"), 10.0) if bad is O.activate_position else bad(float("nan"))


def test_covariance_kats():
    # test_field_core.cpp:74-88, :92-116
    sxx, sxy, syy = O.covariance(2.0, 3.0, math.pi / 6.0)
    assert sxx == pytest.approx(5.35, rel=1e-12)
    assert sxy == pytest.approx(-2.1650635094610964, rel=1e-12)
    assert syy == pytest.approx(7.85, rel=1e-12)
    (i00, i01, i11), r = O.invert_covariance(4.1, 0.0, 9.1)
    assert i00 == pytest.approx(1 / 4.1, rel=1e-12) and i11 == pytest.approx(1 / 9.1, rel=1e-12)
    assert r == pytest.approx(3.0 * math.sqrt(9.1), rel=1e-12)
    (t00, _, _), _ = O.invert_covariance(1e-6, 0.0, 1e-6)
    assert t00 == pytest.approx(1e-6 / 1e-10, rel=1e-9)


def test_adan_frozen_trajectories():
    # test_optimizer.cpp:43-71 (1e-14) and the bowl :81
    exp = [0.09999999981818182, 0.19986158511773655, 0.29964122486116573, 0.39933228830259548,
           0.49891560514694228]
    a = O.Adan()
    a.add_group("x", 1, 0.1)
    x = np.array([0.0])
    for e in exp:
        a.step("x", x, np.array([2.0 * (x[0] - 3.0) + 0.5]))
        assert x[0] == pytest.approx(e, rel=1e-14)
    exp2 = [(0.65000000035714278, -0.34999999947662419), (0.60020923125793246, -0.39997688814024729),
            (0.55056102825700071, -0.4499359681375078), (0.50108443403293712, -0.49987253298970658)]
    a = O.Adan()
    a.add_group("xy", 2, 0.05)
    x = np.array([0.7, -0.3])
    for e0, e1 in exp2:
        a.step("xy", x, np.array([2.0 * x[0], math.cos(x[1])]))
        assert x[0] == pytest.approx(e0, rel=1e-14) and x[1] == pytest.approx(e1, rel=1e-14)
    a = O.Adan()
    a.add_group("x", 1, 0.1)
    x = np.array([1.0])
    for _ in range(200):
        a.step("x", x, np.array([2.0 * x[0]]))
    assert abs(x[0]) == pytest.approx(2.19957082432718e-4, rel=1e-9)
    with pytest.raises(RuntimeError, match="params"):
        b = O.Adan()
        b.add_group("params", 2, 0.1)
        b.step("params", np.zeros(2), np.array([np.nan, 0.0]))


def test_cosine_and_planes_kats():
    # test_optimizer.cpp:11-14, test_loss.cpp:31-43
    assert O.cosine_lr(0, 2000, 1e-2, 1e-3) == pytest.approx(1e-2, rel=1e-12)
    assert O.cosine_lr(2000, 2000, 1e-2, 1e-3) == pytest.approx(1e-3, rel=1e-12)
    assert O.cosine_lr(1000, 2000, 1e-2, 1e-3) == pytest.approx(5.5e-3, rel=1e-12)
    with pytest.raises(ValueError):
        O.cosine_lr(101, 100, 1e-2, 1e-3)
    assert O.make_depth_planes(3, 3e-3, 2e-3) == pytest.approx([1e-3, 3e-3, 5e-3])
    d = np.array([[0.0, 0.2, 0.45], [0.55, 0.9, 1.0]])
    m = O.build_masks(d, 2, True)
    assert m[0].ravel().tolist() == [0, 0, 0, 1, 1, 1]
    assert m[1].ravel().tolist() == [1, 1, 1, 0, 0, 0]


def test_transfer_function_dc():
    # test_propagation.cpp:53-68
    b = O.make_band_limit((532e-9,), 3.74e-6, 3e-3, 0, 16, 12)
    H = O.transfer(b, 12, 16, 3e-3, 0.0)
    k = 2 * math.pi / 532e-9
    assert H[0, 0] == pytest.approx(complex(math.cos(k * 3e-3), math.sin(k * 3e-3)), rel=1e-9)


def test_plane_wave_phase():
    # test_propagation.cpp:159-171
    u = np.full((1, 16, 16), 0.7 + 0j)
    out = O.propagate(u, (532e-9,), 3.74e-6, 1, 0.0, 2.5e-3)
    k = 2 * math.pi / 532e-9
    assert np.allclose(out, 0.7 * np.exp(1j * k * 2.5e-3), rtol=1e-9, atol=0)


# ---- golden vectors from the reference -----------------------------------------------------------
@pytest.mark.parametrize("i", range(4))
def test_golden_tile_index(i):
    n, c, w, h = GOLD[f"r{i}_meta"]
    g = O.split(GOLD[f"r{i}_params"], n, c)
    ti = O.build_tile_index(g, n, c, w, h)
    assert np.array_equal(ti["tiles"], GOLD[f"r{i}_tiles"])
    assert np.array_equal(ti["ids"], GOLD[f"r{i}_ids"])
    assert np.array_equal(ti["ranges"], GOLD[f"r{i}_ranges"])


@pytest.mark.parametrize("i", range(4))
def test_golden_raster(i):
    n, c, w, h = GOLD[f"r{i}_meta"]
    g = O.split(GOLD[f"r{i}_params"], n, c)
    re, im = O.rasterize_forward(g, n, c, w, h)
    assert np.max(np.abs(np.stack([re, im]) - GOLD[f"r{i}_fwd"])) <= 1e-12
    gf = GOLD[f"r{i}_gfield"]
    gr = O.rasterize_backward(g, n, c, gf[0], gf[1])
    flat = np.concatenate([gr[k] for k in O.GROUPS])
    assert rel_l2(flat, GOLD[f"r{i}_bwd"]) <= 1e-12


@pytest.mark.parametrize("i", range(4))
def test_golden_propagation(i):
    c, h, w, pad, ap, d = GOLD[f"p{i}_meta"]
    c, h, w, pad = int(c), int(h), int(w), int(pad)
    wl = {1: (532e-9,), 3: (639e-9, 532e-9, 473e-9)}[c]
    u = GOLD[f"p{i}_in"][0] + 1j * GOLD[f"p{i}_in"][1]
    out = O.propagate(u, wl, 3.74e-6, pad, ap, d)
    ref = GOLD[f"p{i}_out"]
    assert np.max(np.abs(out.real - ref[0])) <= 1e-10 and np.max(np.abs(out.imag - ref[1])) <= 1e-10
    back = O.propagate_backward(u, wl, 3.74e-6, pad, ap, d)
    ref = GOLD[f"p{i}_back"]
    assert np.max(np.abs(back.real - ref[0])) <= 1e-10


def test_golden_propagate_multi():
    wl = (639e-9, 532e-9, 473e-9)
    dist = [1e-3, 3e-3, 5e-3]
    u = GOLD["pm_in"][0] + 1j * GOLD["pm_in"][1]
    out = O.propagate_multi(u, wl, 3.74e-6, 2, 0.0, dist)
    assert np.max(np.abs(out.real - GOLD["pm_out"][0])) <= 1e-10
    g = GOLD["pmb_in"][0] + 1j * GOLD["pmb_in"][1]
    back = O.propagate_multi_backward(g, wl, 3.74e-6, 2, 0.0, dist)
    assert np.max(np.abs(back.real - GOLD["pmb_out"][0])) <= 1e-10
    assert np.max(np.abs(back.imag - GOLD["pmb_out"][1])) <= 1e-10


@pytest.mark.parametrize("i", range(2))
def test_golden_loss(i):
    t, m, r = GOLD[f"l{i}_target"], GOLD[f"l{i}_masks"], GOLD[f"l{i}_recon"]
    fns = dict(training=O.training_loss_grad, recon=O.loss_recon_grad, mse=O.loss_mse_grad,
               ssim=lambda r, t, m: O.loss_ssim_grad(r, t, m)[:2])
    for kind, fn in fns.items():
        v, g = fn(r, t, m)
        assert v == pytest.approx(float(GOLD[f"l{i}_{kind}_value"][0]), rel=1e-12, abs=1e-15)
        assert rel_l2(g, GOLD[f"l{i}_{kind}_grad"]) <= 1e-10


def test_golden_full_step():
    n, c, w, h, L = GOLD["step_meta"]
    g = O.split(GOLD["step_params"], n, c)
    masks = O.build_masks(GOLD["step_depth"], L, True)
    dist = O.make_depth_planes(L, 3e-3, 2e-3)
    r = O.step_grads(g, n, c, w, h, GOLD["step_target"], masks, dist, (639e-9, 532e-9, 473e-9))
    loss = r["recon_sum"] / (GOLD["step_target"].size * L) + O.kSsimWeight * (1 - r["ssim_sum"] / r["count"])
    assert loss == pytest.approx(float(GOLD["step_loss"][0]), rel=1e-10)
    flat = np.concatenate([r["grads"][k] for k in O.GROUPS])
    assert rel_l2(flat, GOLD["step_grads"]) <= 1e-9


def test_canonicalize_phase_known_answers():
    """test_convert.cpp:34-48 on the host-side fp64 canonicalisation of the drop-in."""
    from paper_2511_15022_b200 import holo
    tau = 2.0 * np.pi
    assert holo.canonicalize_phase(7.5) == pytest.approx(1.2168146928204138, rel=1e-13)
    assert holo.canonicalize_phase(-np.pi / 2.0) == pytest.approx(3.0 * np.pi / 2.0, rel=1e-13)
    assert holo.canonicalize_phase(0.0) == 0.0
    assert holo.canonicalize_phase(tau) == 0.0
    assert holo.canonicalize_phase(-1e-18) < tau
    for v in (-25.0, -3.2, 0.1, 6.2, 100.0):
        c = holo.canonicalize_phase(v)
        assert 0.0 <= c < tau
        assert abs(np.remainder(c - v + np.pi, tau) - np.pi) <= 1e-9
