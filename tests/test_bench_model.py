"""bench.py's byte model: the per-step algorithmic bytes the
roofline fraction divides by, and the per-kernel split, on CPU."""
import importlib.util
import os

import pytest

from paper_2511_15022_b200 import synthetic as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_step_bytes_match_survey_numbers():
    b = _bench()
    # cfg2 1.41 GB (K = 1.91M pairs at init), cfg3 5.59 GB, cfg4 5.79 GB
    assert b.algorithmic_bytes(S.CONFIGS["cfg2"], 1_910_593) == pytest.approx(1.41e9, rel=5e-3)
    assert b.algorithmic_bytes(S.CONFIGS["cfg3"], 1_910_593) == pytest.approx(5.59e9, rel=5e-3)
    assert b.algorithmic_bytes(S.CONFIGS["cfg4"], 7_868_668) == pytest.approx(5.79e9, rel=1e-2)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4"])
def test_kernel_bytes_cover_the_field_passes(name):
    """The ASM and loss slots of kernel_bytes add up to the C (13 + 12 L) A field
    term of the step model (raster fwd/bwd carry one A each), less the target
    read the model books twice (in F3's loss epilogue and in SSIM) and the
    fused loss kernel reads once."""
    b = _bench()
    cfg = S.CONFIGS[name]
    A = 8.0 * cfg["height"] * cfg["width"]
    c, L = cfg["channels"], cfg["planes"]
    kb = b.kernel_bytes(cfg, 0)
    field = sum(kb[k] for k in ("rows_fwd", "cols_fwd", "rows_inv", "loss_ssim", "rows_fwd_bwd", "cols_bwd",
                                "rows_inv_bwd"))
    field -= L * cfg["height"] * cfg["width"]  # the masks ride with the loss slot
    assert field + 2 * c * A + 0.5 * c * A == pytest.approx(c * (13 + 12 * L) * A, rel=1e-12)


def test_bench_refuses_more_gpus_than_visible():
    """`bench.py --gpus N` with fewer than N visible GPUs exits non-zero with a
    clear message instead of silently running one rank."""
    import subprocess
    import sys
    import torch
    n = max(2, torch.cuda.device_count() + 1)
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0
    assert f"--gpus {n} needs {n} visible GPUs" in r.stderr


def test_fft_adjusted_estimate_charges_the_steps_fft2s_at_pocketfft_speed():
    import bench
    st = {"raster_fwd": 270.0, "propagate_multi": 2300.0, "training_loss_grad": 790.0,
          "propagate_multi_backward": 2300.0, "rasterize_backward": 250.0, "adan": 17.0, "total": 5927.0}
    fft = {"shim_fft2_ifft2_ms_1core": 800.0, "numpy_pocketfft_fft2_ifft2_ms_1core": 600.0}
    est = bench.fft_adjusted(st, fft, 3, 1)  # cfg2: 3 channels x (1 forward + 1 inverse) x 2 directions
    assert est["fft2_per_step"] == 12
    assert abs(est["ms_per_step"] - (5927.0 - 12 * 100.0)) < 0.1
    assert abs(est["value"] - 1e3 / est["ms_per_step"]) < 1e-3
    assert "estimate" in est["note"]
    assert bench.fft_adjusted(st, fft, 3, 8)["fft2_per_step"] == 54
    assert bench.fft_adjusted({"total": 1.0}, {}, 3, 1) is None
