"""CPU: the artifact formats of the reference (io.hpp and
io.cpp:237-335): CGHF complex fields and CGGS Gaussian sets.  The reference's
io.cpp needs libpng (absent here) so it is not compiled; the layout is pinned
by golden header bytes restated from io.cpp:249-335, and the C++ drop-in
(libholo_b200.so, include/holo/io.hpp) and the Python mirror interoperate both
ways."""
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
