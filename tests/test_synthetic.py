"""CPU: host-side input generators restate the reference's fixtures
(holo::Rng, test_util.hpp, pipeline.cpp:165-200) bit-for-bit."""
import numpy as np
import pytest

from paper_2511_15022_b200 import synthetic as S


def test_rng_mt19937_64_known_values():
    # std::mt19937_64 default-seed (5489) 10000th output is 9981545732273789042 (C++ standard)
    r = S.Rng(5489)
    assert int(r.raw(10000)[-1]) == 9981545732273789042


def test_generators_match_reference(ref):
    a = S.init_gaussians(2000, 3, 1920, 1080, 42)
    b = ref.init_gaussians(2000, 3, 1920, 1080, 42)
    for k in ref.GROUPS:
        np.testing.assert_allclose(a[k], getattr(b, k), rtol=0, atol=1e-15)
    assert np.array_equal(a["amplitude"], b.amplitude)
    r = S.random_set(7, 50, 3)
    rb = ref.random_set(7, 50, 3, 10, 10)
    for k in ref.GROUPS:
        assert np.array_equal(r[k], getattr(rb, k)), k
    assert np.abs(S.synthetic_image(42, 3, 64, 96) - ref.synthetic_image(42, 3, 64, 96)).max() < 1e-15
    assert np.abs(S.synthetic_depth(43, 64, 96) - ref.synthetic_depth(43, 64, 96)).max() < 1e-15
    fr = S.random_field(5, 2, 8, 9)
    fb = ref.random_field(5, 2, 8, 9)
    assert np.array_equal(fr[0], fb[0]) and np.array_equal(fr[1], fb[1])
    assert S.resolve_gaussian_count(3, 1920, 1080, 0, 5.0) == ref.resolve_gaussian_count(5.0, 0, 3, 1920, 1080)


def test_resolve_gaussian_count_kats():
    # test_pipeline.cpp:99-116: N = round(2CHW / (12 r))
    assert S.resolve_gaussian_count(1, 160, 256, 0, 2.0) == 3413
    assert S.resolve_gaussian_count(3, 1920, 1080, 0, 5.0) == 207360
    assert S.resolve_gaussian_count(3, 10, 10, 77, 5.0) == 77
