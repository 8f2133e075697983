"""CPU: the artifact formats of the reference (io.hpp and
io.cpp:237-335): CGHF complex fields and CGGS Gaussian sets.  Pinned against
the reference's own io.cpp (compiled unmodified into oracle/_ref with a libpng
stand-in): files written by the reference and by this repo -- the Python
mirror and the C++ drop-in (libholo_b200.so, include/holo/io.hpp) -- are
byte-identical, and each side reads the other's files to the same values."""
import os
import struct
import subprocess

import numpy as np
import pytest

from paper_2511_15022_b200 import holo

TOOL = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cxx", "bin", "io_tool")


def test_cghf_layout_and_roundtrip(tmp_path):
    re = np.arange(30, dtype=np.float64).reshape(2, 3, 5) * 0.1 - 1.0 / 3.0
    im = -0.25 * np.arange(30, dtype=np.float64).reshape(2, 3, 5) + 1e-9
    f = holo.ComplexField(2, 3, 5, re, im)
    for as_f64, item in ((True, 8), (False, 4)):
        p = str(tmp_path / f"f{item}.cghf")
        holo.write_field(p, f, as_f64)
        data = open(p, "rb").read()
        assert data[:4] == b"CGHF"
        assert struct.unpack_from("<HIIIB", data, 4) == (1, 2, 3, 5, 1 if as_f64 else 0)
        assert len(data) == 19 + 2 * 30 * item
        g = holo.read_field(p)
        if as_f64:  # bit-exact persist/load (io.hpp: writers default to f64)
            assert np.array_equal(g.real, re) and np.array_equal(g.imag, im)
        else:
            assert np.array_equal(g.real, re.astype(np.float32)) and np.array_equal(g.imag, im.astype(np.float32))
    assert not os.path.exists(str(tmp_path / "f8.cghf.tmp"))


def test_cggs_layout_and_roundtrip(tmp_path):
    n, c = 4, 3
    flat = np.linspace(-2.0, 3.0, (6 + 2 * c) * n)
    gs = holo.GaussianSet.from_flat(flat, n, c)
    p = str(tmp_path / "s.cggs")
    holo.write_gaussians(p, gs)
    data = open(p, "rb").read()
    assert data[:4] == b"CGGS" and struct.unpack_from("<HII", data, 4) == (1, n, c)
    assert len(data) == 14 + 4 * flat.size
    back = holo.read_gaussians(p)
    assert np.array_equal(back.flat(), flat.astype(np.float32))


def test_format_errors(tmp_path):
    p = str(tmp_path / "bad.cghf")
    open(p, "wb").write(b"XXXX")
    with pytest.raises(holo.HoloError):
        holo.read_field(p)
    f = holo.ComplexField(1, 2, 2)
    q = str(tmp_path / "t.cghf")
    holo.write_field(q, f)
    open(q, "ab").write(b"\0")
    with pytest.raises(holo.HoloError, match="trailing"):
        holo.read_field(q)


@pytest.mark.skipif(not os.path.exists(TOOL), reason="tests/cxx/bin/io_tool not built")
def test_cpp_dropin_and_python_interoperate(tmp_path):
    d = str(tmp_path)
    assert subprocess.run([TOOL, "write", d]).returncode == 0
    f64 = holo.read_field(os.path.join(d, "field64.cghf"))
    i = np.arange(30, dtype=np.float64).reshape(2, 3, 5)
    assert np.array_equal(f64.real, 0.1 * i - 1.0 / 3.0) and np.array_equal(f64.imag, -0.25 * i + 1e-9)
    f32 = holo.read_field(os.path.join(d, "field32.cghf"))
    assert np.array_equal(f32.real, (0.1 * i - 1.0 / 3.0).astype(np.float32))
    s = holo.read_gaussians(os.path.join(d, "set.cggs"))
    assert s.count == 4 and s.channels == 3
    assert np.array_equal(s.pre_scale, (0.25 + 0.5 * np.arange(8)).astype(np.float32))
    # Python writes, C++ reads
    f = holo.ComplexField(1, 4, 6, np.linspace(0, 1, 24), np.linspace(-1, 0, 24))
    holo.write_field(os.path.join(d, "py_field.cghf"), f)
    g = holo.GaussianSet.from_flat(np.linspace(-1, 1, 8 * 5), 5, 1)
    holo.write_gaussians(os.path.join(d, "py_set.cggs"), g)
    out = subprocess.run([TOOL, "read", d], capture_output=True, text=True, check=True).stdout.split()
    k = np.arange(1, 25)
    a = float(np.sum(f.real.ravel() * k + 2.0 * f.imag.ravel() * k))
    flat = g.flat().astype(np.float32).astype(np.float64)
    b = sum(float(np.sum(getattr(g, grp).astype(np.float32).astype(np.float64) * np.arange(1, getattr(g, grp).size + 1)))
            for grp in ("pre_position", "pre_scale", "rotation", "amplitude", "phase", "pre_opacity"))
    assert [int(x) for x in out[:3]] == [1, 4, 6] and float(out[3]) == pytest.approx(a, rel=1e-14)
    assert [int(x) for x in out[4:6]] == [5, 1] and float(out[6]) == pytest.approx(b, rel=1e-12)


def _fixture_field(c=3, h=7, w=11, seed=5):
    rng = np.random.default_rng(seed)
    re = rng.standard_normal((c, h, w)) * 10.0 ** rng.integers(-6, 6, (c, h, w))
    im = rng.standard_normal((c, h, w))
    re[0, 0, 0], im[0, 0, 1] = -0.0, np.inf  # signed zero, non-finite: bit patterns must survive
    return re, im


@pytest.mark.parametrize("as_f64", [True, False])
def test_cghf_byte_identical_with_the_reference_writer(tmp_path, ref, as_f64):
    re, im = _fixture_field()
    pr, po = str(tmp_path / "ref.cghf"), str(tmp_path / "ours.cghf")
    ref.write_field(pr, re, im, as_f64)
    holo.write_field(po, holo.ComplexField(*re.shape, re, im), as_f64)
    assert open(pr, "rb").read() == open(po, "rb").read()
    # each side reads the other's file to the same values
    a = holo.read_field(pr)
    b_re, b_im = ref.read_field(po)
    assert np.array_equal(a.real, b_re, equal_nan=True) and np.array_equal(a.imag, b_im, equal_nan=True)
    assert np.signbit(a.real[0, 0, 0]) and np.isinf(a.imag[0, 0, 1])


def test_cggs_byte_identical_with_the_reference_writer(tmp_path, ref):
    n, c = 37, 3
    g = ref.random_set(11, n, c, 64, 48)
    pr, po = str(tmp_path / "ref.cggs"), str(tmp_path / "ours.cggs")
    ref.write_gaussians(pr, g)
    holo.write_gaussians(po, holo.GaussianSet(n, c, **{k: getattr(g, k) for k in ref.GROUPS}))
    assert open(pr, "rb").read() == open(po, "rb").read()
    back = ref.read_gaussians(po)
    ours = holo.read_gaussians(pr)
    for k in ref.GROUPS:
        assert np.array_equal(getattr(back, k), getattr(ours, k))
        assert np.array_equal(getattr(ours, k), getattr(g, k).astype(np.float32))


@pytest.mark.skipif(not os.path.exists(TOOL), reason="tests/cxx/bin/io_tool not built")
def test_cpp_dropin_files_read_by_the_reference(tmp_path, ref):
    d = str(tmp_path)
    assert subprocess.run([TOOL, "write", d]).returncode == 0
    i = np.arange(30, dtype=np.float64).reshape(2, 3, 5)
    re, im = 0.1 * i - 1.0 / 3.0, -0.25 * i + 1e-9
    ref.write_field(os.path.join(d, "ref64.cghf"), re, im, True)
    ref.write_field(os.path.join(d, "ref32.cghf"), re, im, False)
    assert open(os.path.join(d, "field64.cghf"), "rb").read() == open(os.path.join(d, "ref64.cghf"), "rb").read()
    assert open(os.path.join(d, "field32.cghf"), "rb").read() == open(os.path.join(d, "ref32.cghf"), "rb").read()
    s = ref.read_gaussians(os.path.join(d, "set.cggs"))
    assert s.count == 4 and s.channels == 3
    assert np.array_equal(s.pre_scale, (0.25 + 0.5 * np.arange(8)).astype(np.float32))


def test_format_errors_match_the_reference(tmp_path, ref):
    """Truncated, trailing-byte and wrong-magic files fail on both sides with
    the reference's messages."""
    re, im = _fixture_field(1, 2, 3)
    good = str(tmp_path / "g.cghf")
    ref.write_field(good, re, im, True)
    data = open(good, "rb").read()
    cases = {"trunc.cghf": data[:-3], "trail.cghf": data + b"\0", "magic.cghf": b"XGHF" + data[4:],
             "ver.cghf": data[:4] + b"\2\0" + data[6:]}
    for name, blob in cases.items():
        p = str(tmp_path / name)
        open(p, "wb").write(blob)
        with pytest.raises(ref.RefError) as e_ref:
            ref.read_field(p)
        with pytest.raises(holo.HoloError) as e_ours:
            holo.read_field(p)
        assert str(e_ours.value) == str(e_ref.value), name
