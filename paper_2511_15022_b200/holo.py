"""Python mirror of the reference's hot-path API (namespace holo), backed by the
B200 kernels through the C ABI (include/holosplat.h).

Names, argument meaning and error behaviour follow
/root/reference/proj/core/include/holo/{gaussian_set,complex_field,rasterizer,
propagation,loss,optimizer}.hpp so that tests read like the reference's own
tests.  Host containers are fp64 numpy arrays like the reference's
std::vector<double>; the device computes in fp32 (values are rounded to fp32
on upload).  Device-level entry points (``*_device``) take/return torch CUDA
tensors and skip the host round trip.

There is no CPU fallback: every call goes through libholosplat.so on a GPU.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import (HoloError, HoloInvalidArgument, HoloNonFinite, check, hs_adan_config,
                   hs_poh_config, hs_prop_spec, hs_trainer_config)

__all__ = [
    "GaussianSet", "ComplexField", "RealField", "TileIndex", "PropagationSpec", "TargetStack",
    "DepthPlaneSet", "build_tile_index", "rasterize_forward", "rasterize_backward",
    "propagate", "propagate_with_mask_distance", "propagate_backward", "propagate_multi",
    "propagate_multi_backward", "intensity_of", "make_depth_planes", "build_masks",
    "make_target_stack", "loss_mse", "loss_recon", "loss_ssim", "training_loss",
    "loss_mse_grad", "loss_recon_grad", "loss_ssim_grad", "training_loss_grad", "cosine_lr",
    "Adan", "AdanConfig", "Trainer", "HoloError", "HoloInvalidArgument", "HoloNonFinite",
    "kTileSize", "GROUPS",
]

kTileSize = 16
GROUPS = ("pre_position", "pre_scale", "rotation", "amplitude", "phase", "pre_opacity")


# ---------------------------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------------------------
class _Ctx:
    def __init__(self, device: int):
        self.device = device
        h = C.c_void_p()
        check(_lib.load().hs_ctx_create(device, C.byref(h)))
        self.h = h

    def bind_stream(self):
        s = torch.cuda.current_stream(self.device)
        check(_lib.load().hs_ctx_set_stream(self.h, C.c_void_p(s.cuda_stream)))
        return self.h


_ctxs = {}


def _ctx(device=None):
    if not torch.cuda.is_available():
        raise HoloError("holosplat-b200 needs a CUDA device (B200); no CPU fallback")
    dev = torch.cuda.current_device() if device is None else int(device)
    if dev not in _ctxs:
        _ctxs[dev] = _Ctx(dev)
    return _ctxs[dev]


def ctx_handle(device=None):
    return _ctx(device).bind_stream()


def kernel_launch_count() -> int:
    return int(_lib.load().hs_kernel_launch_count())


def _dev(device=None):
    if not torch.cuda.is_available():
        raise HoloError("holosplat-b200 needs a CUDA device (B200); no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device() if device is None else device)


def _ptr(t: torch.Tensor):
    return C.c_void_p(t.data_ptr())


# ---------------------------------------------------------------------------------------------
# data model (gaussian_set.hpp:12-33, complex_field.hpp:11-63)
# ---------------------------------------------------------------------------------------------
@dataclass
class GaussianSet:
    count: int
    channels: int
    pre_position: np.ndarray = None
    pre_scale: np.ndarray = None
    rotation: np.ndarray = None
    amplitude: np.ndarray = None
    phase: np.ndarray = None
    pre_opacity: np.ndarray = None

    def __post_init__(self):
        if self.count < 0 or self.channels <= 0:
            raise HoloInvalidArgument("GaussianSet: invalid N or C")
        n, c = self.count, self.channels
        sizes = dict(pre_position=2 * n, pre_scale=2 * n, rotation=n, amplitude=n * c, phase=n * c,
                     pre_opacity=n)
        for g in GROUPS:
            if getattr(self, g) is None:
                setattr(self, g, np.zeros(sizes[g]))
            else:
                setattr(self, g, np.asarray(getattr(self, g), dtype=np.float64))

    def validate(self):
        """gaussian_set.cpp:30-39."""
        n, c = self.count, self.channels
        sizes = dict(pre_position=2 * n, pre_scale=2 * n, rotation=n, amplitude=n * c, phase=n * c,
                     pre_opacity=n)
        for g in GROUPS:
            a = getattr(self, g)
            if a.size != sizes[g]:
                raise HoloInvalidArgument(f"GaussianSet: bad size for {g}")
            if not np.all(np.isfinite(a)):
                raise HoloInvalidArgument(f"GaussianSet: non-finite entry in {g}")

    def flat(self) -> np.ndarray:
        """The device parameter layout: six groups back to back."""
        return np.concatenate([np.ravel(getattr(self, g)) for g in GROUPS])

    @classmethod
    def from_flat(cls, flat, n, c) -> "GaussianSet":
        flat = np.asarray(flat, dtype=np.float64)
        sizes = [2 * n, 2 * n, n, n * c, n * c, n]
        out, o = {}, 0
        for g, s in zip(GROUPS, sizes):
            out[g] = flat[o:o + s].copy()
            o += s
        return cls(n, c, **out)

    def to_device(self, device=None) -> torch.Tensor:
        return torch.from_numpy(self.flat().astype(np.float32)).to(_dev(device))

    @staticmethod
    def concat(a: "GaussianSet", b: "GaussianSet") -> "GaussianSet":
        if a.channels != b.channels:
            raise HoloInvalidArgument("GaussianSet::concat: channel mismatch")
        return GaussianSet(a.count + b.count, a.channels,
                           **{g: np.concatenate([getattr(a, g), getattr(b, g)]) for g in GROUPS})


GaussianSetGrads = GaussianSet


@dataclass
class ComplexField:
    channels: int
    height: int
    width: int
    real: np.ndarray = None
    imag: np.ndarray = None

    def __post_init__(self):
        if self.channels <= 0 or self.height <= 0 or self.width <= 0:
            raise HoloInvalidArgument("ComplexField: non-positive dims")
        shape = (self.channels, self.height, self.width)
        self.real = np.zeros(shape) if self.real is None else np.asarray(self.real, np.float64).reshape(shape)
        self.imag = np.zeros(shape) if self.imag is None else np.asarray(self.imag, np.float64).reshape(shape)

    def size(self):
        return self.real.size

    def same_shape(self, o):
        return (self.channels, self.height, self.width) == (o.channels, o.height, o.width)

    def to_device(self, device=None) -> torch.Tensor:
        z = np.stack([self.real, self.imag], axis=-1).astype(np.float32)
        return torch.from_numpy(np.ascontiguousarray(z)).to(_dev(device))

    @classmethod
    def from_device(cls, t: torch.Tensor) -> "ComplexField":
        a = t.detach().to("cpu").numpy().astype(np.float64)
        return cls(a.shape[0], a.shape[1], a.shape[2], a[..., 0], a[..., 1])


@dataclass
class RealField:
    channels: int
    height: int
    width: int
    values: np.ndarray = None

    def __post_init__(self):
        if self.channels <= 0 or self.height <= 0 or self.width <= 0:
            raise HoloInvalidArgument("RealField: non-positive dims")
        shape = (self.channels, self.height, self.width)
        self.values = np.zeros(shape) if self.values is None else np.asarray(self.values, np.float64).reshape(shape)

    def same_shape(self, o):
        return (self.channels, self.height, self.width) == (o.channels, o.height, o.width)


def intensity_of(u: ComplexField) -> RealField:
    """field_core.cpp:88-93 (on the device)."""
    d = u.to_device()
    out = torch.empty(d.shape[:-1], dtype=torch.float32, device=d.device)
    check(_lib.load().hs_intensity(ctx_handle(), _ptr(d), C.c_int64(u.size()), _ptr(out)))
    return RealField(u.channels, u.height, u.width, out.cpu().numpy())


# ---------------------------------------------------------------------------------------------
# rasterizer (rasterizer.hpp:12-36)
# ---------------------------------------------------------------------------------------------
@dataclass
class TileIndex:
    tiles_x: int
    tiles_y: int
    pairs: np.ndarray   # K x 2 uint32 (tile, id), sorted
    ranges: np.ndarray  # T x 2 uint64 [begin, end), {0,0} when empty


def build_tile_index_device(params: torch.Tensor, n, c, width, height):
    lib = _lib.load()
    h = ctx_handle()
    k = C.c_int64(0)
    txy = (C.c_int * 2)()
    check(lib.hs_build_tile_index(h, _ptr(params), n, c, width, height, None, None, None,
                                  C.c_int64(-1), C.byref(k), txy))
    tiles = max(txy[0] * txy[1], 1)
    dev = params.device
    t_tiles = torch.empty(max(k.value, 1), dtype=torch.int32, device=dev)
    t_ids = torch.empty(max(k.value, 1), dtype=torch.int32, device=dev)
    t_ranges = torch.empty(2 * tiles, dtype=torch.int64, device=dev)
    check(lib.hs_build_tile_index(h, _ptr(params), n, c, width, height, _ptr(t_tiles), _ptr(t_ids),
                                  _ptr(t_ranges), C.c_int64(k.value), C.byref(k), txy))
    return txy[0], txy[1], t_tiles[:k.value], t_ids[:k.value], t_ranges.view(-1, 2)


def build_tile_index(s: GaussianSet, width: int, height: int) -> TileIndex:
    if width <= 0 or height <= 0:
        raise HoloInvalidArgument("build_tile_index: empty canvas")
    tx, ty, tiles, ids, ranges = build_tile_index_device(s.to_device(), s.count, s.channels, width, height)
    pairs = np.stack([tiles.cpu().numpy().view(np.uint32), ids.cpu().numpy().view(np.uint32)], axis=1)
    return TileIndex(tx, ty, pairs, ranges[: tx * ty].cpu().numpy().view(np.uint64))


def rasterize_forward_device(params: torch.Tensor, n, c, width, height) -> torch.Tensor:
    if width <= 0 or height <= 0:
        raise HoloInvalidArgument("rasterize_forward: empty canvas")
    out = torch.empty((c, height, width, 2), dtype=torch.float32, device=params.device)
    check(_lib.load().hs_rasterize_forward(ctx_handle(), _ptr(params), n, c, width, height, _ptr(out)))
    return out


def rasterize_forward(s: GaussianSet, width: int, height: int) -> ComplexField:
    return ComplexField.from_device(rasterize_forward_device(s.to_device(), s.count, s.channels, width, height))


def set_backward_deterministic(on: bool = True):
    """Backward form of the stand-alone rasterize_backward on this context:
    the bit-reproducible per-Gaussian gather (default) or the per-tile backward
    with vector atomics (hs_ctx_set_deterministic)."""
    check(_lib.load().hs_ctx_set_deterministic(ctx_handle(), int(on)))


def rasterize_backward_device(params: torch.Tensor, n, c, grad_field: torch.Tensor) -> torch.Tensor:
    cc, h, w, _ = grad_field.shape
    if cc != c:
        raise HoloInvalidArgument("rasterize_backward: gradient shape mismatch")
    out = torch.zeros_like(params)
    check(_lib.load().hs_rasterize_backward(ctx_handle(), _ptr(params), n, c, w, h,
                                            _ptr(grad_field.contiguous()), _ptr(out)))
    return out


def rasterize_backward(s: GaussianSet, grad_real: RealField, grad_imag: RealField) -> GaussianSet:
    if not grad_real.same_shape(grad_imag) or grad_real.channels != s.channels:
        raise HoloInvalidArgument("rasterize_backward: gradient shape mismatch")
    gf = ComplexField(grad_real.channels, grad_real.height, grad_real.width, grad_real.values,
                      grad_imag.values).to_device()
    g = rasterize_backward_device(s.to_device(), s.count, s.channels, gf)
    return GaussianSet.from_flat(g.cpu().numpy(), s.count, s.channels)


# ---------------------------------------------------------------------------------------------
# propagation (propagation.hpp:9-49)
# ---------------------------------------------------------------------------------------------
@dataclass
class PropagationSpec:
    wavelengths: Sequence[float] = (639e-9, 532e-9, 473e-9)
    pixel_pitch: float = 3.74e-6
    pad_factor: int = 2
    aperture_radius: float = 0.0

    def c_struct(self):
        wl = (C.c_double * len(self.wavelengths))(*self.wavelengths)
        s = hs_prop_spec(C.cast(wl, C.POINTER(C.c_double)), len(self.wavelengths), float(self.pixel_pitch),
                         int(self.pad_factor), float(self.aperture_radius))
        s._keep = wl
        return s


def propagate_device(field: torch.Tensor, spec: PropagationSpec, distance, mode=0, mask_distance=0.0):
    c, h, w, _ = field.shape
    out = torch.empty_like(field)
    s = spec.c_struct()
    check(_lib.load().hs_propagate(ctx_handle(), C.byref(s), mode, float(distance), float(mask_distance),
                                   _ptr(field.contiguous()), c, h, w, _ptr(out)))
    return out


def propagate(field: ComplexField, spec: PropagationSpec, distance: float) -> ComplexField:
    return ComplexField.from_device(propagate_device(field.to_device(), spec, distance, 0))


def propagate_with_mask_distance(field: ComplexField, spec: PropagationSpec, distance: float,
                                 mask_distance: float) -> ComplexField:
    return ComplexField.from_device(propagate_device(field.to_device(), spec, distance, 1, mask_distance))


def propagate_backward(grad_out: ComplexField, spec: PropagationSpec, distance: float) -> ComplexField:
    return ComplexField.from_device(propagate_device(grad_out.to_device(), spec, distance, 2))


def propagate_multi_device(field: torch.Tensor, spec: PropagationSpec, distances) -> torch.Tensor:
    c, h, w, _ = field.shape
    L = len(distances)
    out = torch.empty((L, c, h, w, 2), dtype=torch.float32, device=field.device)
    d = (C.c_double * max(L, 1))(*distances)
    s = spec.c_struct()
    check(_lib.load().hs_propagate_multi(ctx_handle(), C.byref(s), d, L, _ptr(field.contiguous()), c, h, w,
                                         _ptr(out)))
    return out


def propagate_multi(field: ComplexField, spec: PropagationSpec, distances) -> List[ComplexField]:
    out = propagate_multi_device(field.to_device(), spec, list(distances))
    return [ComplexField.from_device(out[l]) for l in range(out.shape[0])]


def propagate_multi_backward_device(grads: torch.Tensor, spec: PropagationSpec, distances) -> torch.Tensor:
    L, c, h, w, _ = grads.shape
    out = torch.empty((c, h, w, 2), dtype=torch.float32, device=grads.device)
    d = (C.c_double * max(L, 1))(*distances)
    s = spec.c_struct()
    check(_lib.load().hs_propagate_multi_backward(ctx_handle(), C.byref(s), d, len(distances),
                                                  _ptr(grads.contiguous()), c, h, w, _ptr(out)))
    return out


def propagate_multi_backward(grads: List[ComplexField], spec: PropagationSpec, distances) -> ComplexField:
    if not grads or len(grads) != len(distances):
        raise HoloInvalidArgument("propagate_multi_backward: plane count mismatch")
    for g in grads:
        if not g.same_shape(grads[0]):
            raise HoloInvalidArgument("propagate_multi_backward: gradient shape mismatch")
    stack = torch.stack([g.to_device() for g in grads])
    return ComplexField.from_device(propagate_multi_backward_device(stack, spec, list(distances)))


# ---------------------------------------------------------------------------------------------
# loss (loss.hpp:10-67)
# ---------------------------------------------------------------------------------------------
kSsimWindow, kSsimSigma, kSsimC1, kSsimC2, kSsimWeight = 11, 1.5, 0.01 ** 2, 0.03 ** 2, 0.005


# ---- artifact formats (io.hpp; io.cpp:237-335) -----------------------------------------------------
def atomic_write(path: str, data: bytes) -> None:
    """Temp file in the same directory, then rename (io.cpp:237-247)."""
    import os
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(data)
    os.replace(tmp, path)


def write_field(path: str, field: ComplexField, as_f64: bool = True) -> None:
    """CGHF: magic, u16 1, u32 C/H/W, u8 dtype, planar real then imag, little-endian."""
    import struct
    dt = "<f8" if as_f64 else "<f4"
    head = b"CGHF" + struct.pack("<HIIIB", 1, field.channels, field.height, field.width, 1 if as_f64 else 0)
    body = np.ascontiguousarray(field.real, dtype=dt).tobytes() + np.ascontiguousarray(field.imag, dtype=dt).tobytes()
    atomic_write(path, head + body)


def read_field(path: str) -> ComplexField:
    import struct
    data = open(path, "rb").read()
    if len(data) < 4 or data[:4] != b"CGHF":
        raise HoloError(f"{path}: not a CGHF file")
    if len(data) < 19:
        raise HoloError("truncated file")  # io.cpp:44-47 (no path)
    ver, c, h, w, dtype = struct.unpack_from("<HIIIB", data, 4)
    if ver != 1:
        raise HoloError(f"{path}: unsupported CGHF version")
    if dtype > 1:
        raise HoloError(f"{path}: unknown CGHF dtype")
    n = c * h * w
    item = 8 if dtype else 4
    if len(data) < 19 + 2 * n * item:
        raise HoloError("truncated file")  # io.cpp:44-47 (no path)
    if len(data) != 19 + 2 * n * item:
        raise HoloError(f"{path}: trailing bytes")
    v = np.frombuffer(data, dtype="<f8" if dtype else "<f4", offset=19, count=2 * n).astype(np.float64)
    return ComplexField(c, h, w, v[:n].reshape(c, h, w), v[n:].reshape(c, h, w))


def write_gaussians(path: str, gs: GaussianSet) -> None:
    """CGGS: magic, u16 1, u32 N, u32 C, the six groups in declaration order as f32."""
    import struct
    head = b"CGGS" + struct.pack("<HII", 1, gs.count, gs.channels)
    atomic_write(path, head + np.asarray(gs.flat(), dtype="<f4").tobytes())


def read_gaussians(path: str) -> GaussianSet:
    import struct
    data = open(path, "rb").read()
    if len(data) < 4 or data[:4] != b"CGGS":
        raise HoloError(f"{path}: not a CGGS file")
    if len(data) < 14:
        raise HoloError("truncated file")  # io.cpp:44-47 (no path)
    ver, n, c = struct.unpack_from("<HII", data, 4)
    if ver != 1:
        raise HoloError(f"{path}: unsupported CGGS version")
    count = (6 + 2 * c) * n
    if len(data) < 14 + 4 * count:
        raise HoloError("truncated file")  # io.cpp:44-47 (no path)
    if len(data) != 14 + 4 * count:
        raise HoloError(f"{path}: trailing bytes")
    flat = np.frombuffer(data, dtype="<f4", offset=14, count=count).astype(np.float64)
    return GaussianSet.from_flat(flat, n, c)


# ---- end-of-run metrics (pipeline.hpp:47-57, pipeline.cpp:135-163) --------------------------------
@dataclass
class Metrics:
    psnr: List[float]
    ssim: List[float]
    mean_psnr: float
    mean_ssim: float


def psnr_value(recon: RealField, target: RealField) -> float:
    """pipeline.cpp:135-147 (host fp64, like the reference's scalar helper)."""
    if not recon.same_shape(target):
        raise HoloInvalidArgument("psnr: shape mismatch")
    d = np.clip(recon.values, 0.0, 1.0) - np.clip(target.values, 0.0, 1.0)
    mse = float(np.mean(d * d))
    return math.inf if mse <= 0.0 else -10.0 * math.log10(mse)


def compute_metrics(recon: List[RealField], target: RealField) -> Metrics:
    """pipeline.cpp:149-163 on the B200 (hs_compute_metrics)."""
    if not recon:
        raise HoloInvalidArgument("compute_metrics: no planes")
    for r in recon:
        if not r.same_shape(target):
            raise HoloInvalidArgument("psnr: shape mismatch")
    L = len(recon)
    dev = _dev()
    t = torch.from_numpy(np.ascontiguousarray(target.values, dtype=np.float32)).to(dev)
    r = torch.from_numpy(np.stack([np.asarray(x.values, dtype=np.float32) for x in recon])).to(dev)
    ps, ss = (C.c_double * L)(), (C.c_double * L)()
    check(_lib.load().hs_compute_metrics(ctx_handle(), L, target.channels, target.height, target.width,
                                         _ptr(r.contiguous()), _ptr(t), ps, ss))
    p, s = list(ps), list(ss)
    return Metrics(p, s, sum(p) / L, sum(s) / L)


# ---- phase-only hologram conversion (convert.hpp, convert.cpp:20-184) -------------------------
TWO_PI = 2.0 * math.pi


def canonicalize_phase(value):
    """convert.cpp:20-25 in fp64 (scalar or array) -> [0, 2 pi)."""
    r = np.fmod(np.asarray(value, dtype=np.float64), TWO_PI)
    r = np.where(r < 0.0, r + TWO_PI, r)
    r = np.where(r >= TWO_PI, r - TWO_PI, r)
    return float(r) if np.ndim(r) == 0 else r


DPAC_DIRECT, DPAC_CLASSICAL = 0, 1
POH_SMOOTH, POH_RANDOM = "smooth", "random"


@dataclass
class PhaseOnlyHologram:
    phase: RealField
    format: str = POH_SMOOTH


def dpac_encode(field: ComplexField, mode: int = DPAC_DIRECT) -> PhaseOnlyHologram:
    """convert.cpp:31-60 on the B200; canonicalised in fp64 like the reference."""
    d = field.to_device()
    out = torch.empty((field.channels, field.height, field.width), dtype=torch.float32, device=d.device)
    check(_lib.load().hs_dpac_encode(ctx_handle(), _ptr(d), field.channels, field.height, field.width, int(mode),
                                     _ptr(out)))
    ph = canonicalize_phase(out.cpu().numpy().astype(np.float64))
    return PhaseOnlyHologram(RealField(field.channels, field.height, field.width, ph), POH_SMOOTH)


def poh_field(poh: PhaseOnlyHologram) -> ComplexField:
    """convert.cpp:62-69: e^{i phase}."""
    ph = poh.phase
    d = torch.from_numpy(np.ascontiguousarray(ph.values, dtype=np.float32)).to(_dev())
    out = torch.empty((ph.channels, ph.height, ph.width, 2), dtype=torch.float32, device=d.device)
    check(_lib.load().hs_poh_field(ctx_handle(), _ptr(d), int(d.numel()), _ptr(out)))
    return ComplexField.from_device(out)


@dataclass
class RandomPohOptions:
    steps: int = 600
    seed: int = 0
    lambda_comp: float = 0.1
    lambda_field: float = 0.01
    lr: float = 2.5e-3
    log_every: int = 50


@dataclass
class RandomPohResult:
    poh: PhaseOnlyHologram
    loss_history: List[float]


def random_phase(seed: int, n: int) -> np.ndarray:
    """Rng(seed).uniform(-pi, pi) in element order (rng.hpp: mt19937_64, 53-bit),
    drawn by std::mt19937_64 in the native library (hs_random_uniform)."""
    out = np.empty(int(n), dtype=np.float64)
    check(_lib.load().hs_random_uniform(C.c_uint64(int(seed) & 0xFFFFFFFFFFFFFFFF), C.c_int64(int(n)), -math.pi,
                                        math.pi, out.ctypes.data_as(C.c_void_p)))
    return out


def convert_random_poh_field(guide_field: ComplexField, planes, target: "TargetStack", spec: PropagationSpec,
                             opt: RandomPohOptions = RandomPohOptions()) -> RandomPohResult:
    """convert.cpp:71-174, device resident (hs_convert_random_poh_field)."""
    c, h, w = guide_field.channels, guide_field.height, guide_field.width
    ti = target.intensity
    if (c, h, w) != (ti.channels, ti.height, ti.width):
        raise HoloInvalidArgument("convert_random_poh: guide/target shape mismatch")
    dists = list(planes.distances if hasattr(planes, "distances") else planes)
    if not dists:
        raise HoloInvalidArgument("convert_random_poh: no depth planes")
    masks = np.ascontiguousarray(target.masks, dtype=np.uint8)
    if masks.shape[0] != len(dists):
        raise HoloInvalidArgument("convert_random_poh: plane/mask count mismatch")
    if opt.steps < 1:
        raise HoloInvalidArgument("convert_random_poh: steps must be >= 1")
    phase = torch.from_numpy(random_phase(opt.seed, c * h * w).astype(np.float32)).to(_dev())
    tgt = np.ascontiguousarray(ti.values, dtype=np.float32)
    d = (C.c_double * len(dists))(*dists)
    s = spec.c_struct()
    cfg = hs_poh_config(c, h, w, len(dists), C.cast(d, C.POINTER(C.c_double)), s,
                        tgt.ctypes.data_as(C.POINTER(C.c_float)), masks.ctypes.data_as(C.POINTER(C.c_uint8)),
                        int(opt.steps), float(opt.lambda_comp), float(opt.lambda_field), float(opt.lr))
    loss = (C.c_double * opt.steps)()
    g = guide_field.to_device()
    check(_lib.load().hs_convert_random_poh_field(ctx_handle(), C.byref(cfg), _ptr(g), _ptr(phase), loss))
    hist = [loss[i] for i in range(opt.steps)
            if (opt.log_every > 0 and (i + 1) % opt.log_every == 0) or i + 1 == opt.steps]
    ph = canonicalize_phase(phase.cpu().numpy().astype(np.float64))
    return RandomPohResult(PhaseOnlyHologram(RealField(c, h, w, ph), POH_RANDOM), hist)


def convert_random_poh(guide: GaussianSet, planes, target: "TargetStack", spec: PropagationSpec,
                       opt: RandomPohOptions = RandomPohOptions()) -> RandomPohResult:
    """convert.cpp:176-182."""
    field = rasterize_forward(guide, target.intensity.width, target.intensity.height)
    return convert_random_poh_field(field, planes, target, spec, opt)


@dataclass
class DepthPlaneSet:
    count: int
    center_distance: float
    spacing: float
    distances: List[float] = field(default_factory=list)


def make_depth_planes(count: int, center_distance: float, spacing: float) -> DepthPlaneSet:
    """make_depth_planes, loss.cpp:154-164."""
    if count < 1:
        raise HoloInvalidArgument("make_depth_planes: count must be >= 1")
    return DepthPlaneSet(count, center_distance, spacing,
                         [center_distance + (l - (count - 1) * 0.5) * spacing for l in range(count)])


def build_masks(depth: RealField, plane_count: int, near_is_high: bool) -> np.ndarray:
    """build_masks, loss.cpp:166-180 (via the C ABI, bit-exact); returns L x H x W uint8."""
    if plane_count < 1:
        raise HoloInvalidArgument("build_masks: plane count must be >= 1")
    if depth.channels != 1:
        raise HoloInvalidArgument("build_masks: depth must be a single plane")
    d = np.ascontiguousarray(depth.values.reshape(depth.height, depth.width), dtype=np.float64)
    out = np.zeros((plane_count, depth.height, depth.width), dtype=np.uint8)
    check(_lib.load().hs_build_masks(d.ctypes.data_as(C.c_void_p), depth.height, depth.width, plane_count,
                                     int(bool(near_is_high)), out.ctypes.data_as(C.c_void_p)))
    return out


@dataclass
class TargetStack:
    intensity: RealField
    depth: RealField
    masks: np.ndarray  # L x H x W uint8


def make_target_stack(intensity: RealField, depth: RealField, plane_count: int, near_is_high: bool):
    if depth.height != intensity.height or depth.width != intensity.width:
        raise HoloInvalidArgument("make_target_stack: depth/intensity size mismatch")
    return TargetStack(intensity, depth, build_masks(depth, plane_count, near_is_high))


_KIND = dict(training=0, recon=1, ssim=2, mse=3)


def _check_pair(recon: List[RealField], target: TargetStack):
    if not recon:
        raise HoloInvalidArgument("loss: no reconstruction planes")
    if len(recon) != target.masks.shape[0]:
        raise HoloInvalidArgument("loss: plane count does not match masks")
    for r in recon:
        if not r.same_shape(target.intensity):
            raise HoloInvalidArgument("loss: reconstruction shape mismatch")


def loss_device(kind: str, recon: torch.Tensor, target: torch.Tensor, masks: torch.Tensor,
                want_grad=True):
    L, c, h, w = recon.shape
    g = torch.empty_like(recon) if want_grad else None
    v = C.c_double(0.0)
    check(_lib.load().hs_loss(ctx_handle(), _KIND[kind], L, c, h, w, _ptr(recon.contiguous()),
                              _ptr(target.contiguous()), _ptr(masks.contiguous()),
                              _ptr(g) if g is not None else None, C.byref(v)))
    return v.value, g


def _loss(kind, recon, target, grads=None):
    _check_pair(recon, target)
    dev = _dev()
    r = torch.from_numpy(np.stack([x.values for x in recon]).astype(np.float32)).to(dev)
    t = torch.from_numpy(target.intensity.values.astype(np.float32)).to(dev)
    m = torch.from_numpy(np.ascontiguousarray(target.masks)).to(dev)
    v, g = loss_device(kind, r, t, m, grads is not None)
    if grads is not None:
        gh = g.cpu().numpy().astype(np.float64)
        grads.clear()
        for l in range(len(recon)):
            grads.append(RealField(recon[0].channels, recon[0].height, recon[0].width, gh[l]))
    return v


def loss_mse(recon, target):
    return _loss("mse", recon, target)


def loss_recon(recon, target):
    return _loss("recon", recon, target)


def loss_ssim(recon, target):
    return _loss("ssim", recon, target)


def training_loss(recon, target):
    return _loss("training", recon, target)


def loss_mse_grad(recon, target, grads: list):
    return _loss("mse", recon, target, grads)


def loss_recon_grad(recon, target, grads: list):
    return _loss("recon", recon, target, grads)


def loss_ssim_grad(recon, target, grads: list):
    return _loss("ssim", recon, target, grads)


def training_loss_grad(recon, target, grads: list):
    return _loss("training", recon, target, grads)


# ---------------------------------------------------------------------------------------------
# optimizer (optimizer.hpp:10-49)
# ---------------------------------------------------------------------------------------------
def cosine_lr(step: int, total_steps: int, lr_max: float, lr_min: float) -> float:
    out = C.c_double(0.0)
    check(_lib.load().hs_cosine_lr(int(step), int(total_steps), float(lr_max), float(lr_min), C.byref(out)))
    return out.value


@dataclass
class AdanConfig:
    beta1: float = 0.98
    beta2: float = 0.92
    beta3: float = 0.99
    eps: float = 1e-8


class Adan:
    """holo::Adan with device-resident fp32 state (optimizer.cpp:15-72)."""

    def __init__(self, cfg: AdanConfig = None):
        self.cfg = cfg or AdanConfig()
        self._groups = {}

    def add_group(self, name: str, size: int, lr: float):
        if name in self._groups:
            raise HoloInvalidArgument("Adan: duplicate group " + name)
        self._groups[name] = dict(lr=float(lr), t=0, size=int(size),
                                  state=torch.zeros(4 * max(int(size), 1), dtype=torch.float32, device=_dev()))

    def _find(self, name):
        if name not in self._groups:
            raise HoloInvalidArgument("Adan: unknown group " + name)
        return self._groups[name]

    def set_lr(self, name, lr):
        self._find(name)["lr"] = float(lr)

    def lr(self, name):
        return self._find(name)["lr"]

    def step_count(self, name):
        return self._find(name)["t"]

    def step_device(self, name, params: torch.Tensor, grads: torch.Tensor):
        g = self._find(name)
        if params.numel() != g["size"] or grads.numel() != g["size"]:
            raise HoloInvalidArgument("Adan: size mismatch for group " + name)
        c = self.cfg
        cfg = hs_adan_config(c.beta1, c.beta2, c.beta3, c.eps)
        check(_lib.load().hs_adan_step(ctx_handle(), C.byref(cfg), name.encode(), _ptr(params),
                                       _ptr(grads.contiguous()), _ptr(g["state"]), C.c_int64(g["size"]),
                                       g["t"] + 1, g["lr"]))
        g["t"] += 1

    def step(self, name, params: np.ndarray, grads: np.ndarray):
        """In place on a host fp64 array, like holo::Adan::step on a span."""
        p = torch.from_numpy(np.asarray(params, dtype=np.float32)).to(_dev())
        gr = torch.from_numpy(np.asarray(grads, dtype=np.float32)).to(_dev())
        self.step_device(name, p, gr)
        params[...] = p.cpu().numpy().astype(np.float64)


# ---------------------------------------------------------------------------------------------
# trainer: the fused step loop (pipeline.cpp:243-297)
# ---------------------------------------------------------------------------------------------
class Trainer:
    """Device-resident replacement of the reference step-loop body.

    ``step()`` runs rasterize_forward -> propagate_multi -> training_loss_grad ->
    dU = 2 U g -> propagate_multi_backward -> rasterize_backward -> Adan x 6
    with the reference's group learning rates and cosine position schedule.
    """

    def __init__(self, gaussians: GaussianSet, width: int, height: int, target: RealField,
                 masks: np.ndarray, distances: Sequence[float], spec: PropagationSpec, total_steps: int,
                 plane_range=None, device=None, channels_total=None):
        self.n, self.c = gaussians.count, gaussians.channels
        self.width, self.height = width, height
        self.L = len(distances)
        self._spec = spec.c_struct()
        self._dist = (C.c_double * self.L)(*distances)
        tgt = np.ascontiguousarray(target.values, dtype=np.float32)
        msk = np.ascontiguousarray(masks, dtype=np.uint8)
        self._keep = (tgt, msk)
        pb, pe = plane_range if plane_range else (0, 0)
        cfg = hs_trainer_config(self.n, self.c, width, height, self.L,
                                C.cast(self._dist, C.POINTER(C.c_double)), self._spec, int(total_steps),
                                tgt.ctypes.data_as(C.POINTER(C.c_float)),
                                msk.ctypes.data_as(C.POINTER(C.c_uint8)), pb, pe,
                                int(channels_total or 0))
        h = C.c_void_p()
        self._ctx = ctx_handle(device)
        check(_lib.load().hs_trainer_create(self._ctx, C.byref(cfg), C.byref(h)))
        self.h = h
        self.set_params(gaussians.flat().astype(np.float32))

    def __del__(self):
        if getattr(self, "h", None):
            try:
                _lib.load().hs_trainer_destroy(self.h)
            except Exception:
                pass
            self.h = None

    @property
    def param_count(self):
        return int(_lib.load().hs_trainer_param_count(self.h))

    def set_params(self, flat):
        if isinstance(flat, torch.Tensor):
            check(_lib.load().hs_trainer_set_params(self.h, _ptr(flat), 1 if flat.is_cuda else 0))
        else:
            a = np.ascontiguousarray(flat, dtype=np.float32)
            check(_lib.load().hs_trainer_set_params(self.h, a.ctypes.data_as(C.c_void_p), 0))

    def params(self) -> np.ndarray:
        out = np.zeros(self.param_count, dtype=np.float32)
        check(_lib.load().hs_trainer_get_params(self.h, out.ctypes.data_as(C.c_void_p), 0))
        return out

    def params_tensor(self) -> torch.Tensor:
        """Zero-copy view of the device parameter buffer (fp32)."""
        return _wrap(self, _lib.load().hs_trainer_params_ptr(self.h), self.param_count)

    def grads_tensor(self) -> torch.Tensor:
        return _wrap(self, _lib.load().hs_trainer_grads_ptr(self.h), self.param_count)

    def flags_tensor(self) -> torch.Tensor:
        """The device word of non-finite gradient groups (int32 view, bit g = group g)."""
        return _wrap(self, _lib.load().hs_trainer_flags_ptr(self.h), 1, "<i4")

    def slab_error_tensor(self):
        """The device peer-put timeout word (int32 view), None without row slabs."""
        p = _lib.load().hs_trainer_slab_error_ptr(self.h)
        return _wrap(self, p, 1, "<i4") if p else None

    def gaussians(self) -> GaussianSet:
        return GaussianSet.from_flat(self.params(), self.n, self.c)

    def use_graph(self, on=True):
        check(_lib.load().hs_trainer_use_graph(self.h, int(on)))

    def set_deterministic(self, on=True):
        """Raster backward as the bit-reproducible per-Gaussian gather (on) or the
        faster per-tile backward with atomics (off, the default)."""
        check(_lib.load().hs_trainer_set_deterministic(self.h, int(on)))

    def set_profiling(self, on=True):
        check(_lib.load().hs_trainer_set_profiling(self.h, int(on)))

    STAGES = ("binning", "raster_fwd", "rows_fwd", "cols_fwd", "rows_inv", "loss_ssim",
              "rows_fwd_bwd", "cols_bwd", "rows_inv_bwd", "raster_bwd", "adan", "total")

    def stage_ms(self):
        out = (C.c_double * 12)()
        check(_lib.load().hs_trainer_stage_ms(self.h, out))
        return dict(zip(self.STAGES, list(out)))

    def step_host(self, params_in, params_out=None) -> float:
        """One step with host-resident parameters (hs_trainer_step_host): H2D of
        params_in, the step, D2H of the updated parameters into params_out and of
        the loss, one synchronisation.  Pass pinned torch tensors (fp32, CPU) for
        full copy bandwidth; numpy arrays work too."""
        self._ctx = ctx_handle()

        def addr(x):
            if x is None:
                return None
            if isinstance(x, torch.Tensor):
                if x.is_cuda or x.dtype != torch.float32 or not x.is_contiguous() or x.numel() != self.param_count:
                    raise HoloInvalidArgument("step_host: need a contiguous fp32 host tensor of param_count floats")
                return C.c_void_p(x.data_ptr())
            if x.dtype != np.float32 or not x.flags.c_contiguous or x.size != self.param_count:
                raise HoloInvalidArgument("step_host: need a contiguous fp32 array of param_count floats")
            return x.ctypes.data_as(C.c_void_p)

        v = C.c_double(0.0)
        check(_lib.load().hs_trainer_step_host(self.h, addr(params_in), addr(params_out), C.byref(v)))
        return v.value

    def run_host(self, params, steps: int):
        """`steps` steps with host-resident parameters (hs_trainer_run_host):
        `params` (pinned fp32 torch tensor or numpy array of param_count floats)
        is uploaded before and overwritten with the updated parameters after
        every step, the copies pipelined across steps.  Returns the per-step
        losses (numpy float64)."""
        self._ctx = ctx_handle()
        if isinstance(params, torch.Tensor):
            if params.is_cuda or params.dtype != torch.float32 or not params.is_contiguous() \
                    or params.numel() != self.param_count:
                raise HoloInvalidArgument("run_host: need a contiguous fp32 host tensor of param_count floats")
            ptr = C.c_void_p(params.data_ptr())
        else:
            if params.dtype != np.float32 or not params.flags.c_contiguous or params.size != self.param_count:
                raise HoloInvalidArgument("run_host: need a contiguous fp32 array of param_count floats")
            ptr = params.ctypes.data_as(C.c_void_p)
        losses = np.zeros(max(int(steps), 0), np.float64)
        check(_lib.load().hs_trainer_run_host(self.h, ptr, int(steps),
                                              losses.ctypes.data_as(C.POINTER(C.c_double))))
        return losses

    def step(self, sync_loss=True):
        self._ctx = ctx_handle()
        if sync_loss:
            v = C.c_double(0.0)
            check(_lib.load().hs_trainer_step(self.h, C.byref(v)))
            return v.value
        check(_lib.load().hs_trainer_step(self.h, None))
        return None

    def forward_backward(self):
        ctx_handle()
        check(_lib.load().hs_trainer_forward_backward(self.h))

    def apply_update(self):
        ctx_handle()
        check(_lib.load().hs_trainer_apply_update(self.h))

    def check_grads(self):
        """After a cross-rank sum of grads_tensor(): recompute the non-finite group bits."""
        ctx_handle()
        check(_lib.load().hs_trainer_check_grads(self.h))

    def check_grads_range(self, begin: int, end: int):
        """Non-finite group bits of grads[begin, end) only (a rank's shard after a
        reduce-scatter; agree on them across ranks afterwards)."""
        ctx_handle()
        check(_lib.load().hs_trainer_check_grads_range(self.h, int(begin), int(end)))

    def apply_update_range(self, begin: int, end: int):
        """Adan over params[begin, end) only (sharded update; all-gather after)."""
        ctx_handle()
        check(_lib.load().hs_trainer_apply_update_range(self.h, int(begin), int(end)))

    def last_loss(self):
        v = C.c_double(0.0)
        k = C.c_int64(0)
        check(_lib.load().hs_trainer_last_loss(self.h, C.byref(v), C.byref(k)))
        return v.value, k.value

    def loss_partials(self):
        out = (C.c_double * 2)()
        check(_lib.load().hs_trainer_loss_partials(self.h, out))
        return out[0], out[1]

    def reserve_pairs(self, cap):
        check(_lib.load().hs_trainer_reserve_pairs(self.h, C.c_int64(int(cap))))

    # ---- row-slab sharding (cfg4: distributed 2D FFT, parallel.SlabShardedStep) ----
    def set_row_slab(self, rank: int, ranks: int):
        """Make this trainer rank `rank` of `ranks` row slabs (hs_trainer_set_row_slab)."""
        check(_lib.load().hs_trainer_set_row_slab(self.h, int(rank), int(ranks)))
        self.slab = (int(rank), int(ranks))
        counts = [self.slab_counts(e) for e in range(4)]
        size = max(max(sum(s), sum(r)) for s, r in counts)
        lib = _lib.load()
        self._slab_send = _wrap(self, lib.hs_trainer_slab_send_ptr(self.h), size)
        self._slab_recv = _wrap(self, lib.hs_trainer_slab_recv_ptr(self.h), size)

    def slab_counts(self, exchange: int):
        """(send counts, recv counts) in floats per peer of all-to-all `exchange` (0..3)."""
        R = self.slab[1]
        out = (C.c_int64 * (2 * R))()
        check(_lib.load().hs_trainer_slab_counts(self.h, int(exchange), out))
        return list(out[:R]), list(out[R:])

    def slab_buffers(self):
        """(send, recv) fp32 device views of the exchange buffers."""
        return self._slab_send, self._slab_recv

    def slab_stage(self, stage: int):
        ctx_handle()
        check(_lib.load().hs_trainer_slab_stage(self.h, int(stage)))

    def slab_peer_buffers(self):
        """Device addresses (recv0, recv1, flags) a peer stores into in the peer-put exchange."""
        lib = _lib.load()
        return (int(lib.hs_trainer_slab_recv_ptr(self.h)), int(lib.hs_trainer_slab_recv2_ptr(self.h)),
                int(lib.hs_trainer_slab_flags_ptr(self.h)))

    def slab_set_peers(self, recv0, recv1, flags):
        """Peer-put exchange: per-rank device addresses valid in this context (same
        device, P2P or CUDA IPC mapped); this rank's own entries are its own buffers."""
        R = self.slab[1]
        arr = lambda v: (C.c_void_p * R)(*[C.c_void_p(int(x)) for x in v])
        self._peer_arrays = (arr(recv0), arr(recv1), arr(flags))
        check(_lib.load().hs_trainer_slab_set_peers(self.h, *self._peer_arrays))

    def slab_forward_backward(self):
        """Peer-put mode: all five stages in one call (one CUDA graph with use_graph)."""
        ctx_handle()
        check(_lib.load().hs_trainer_slab_forward_backward(self.h))

    def sharded_step(self, with_loss: bool = True):
        """One sharded step over the context's NCCL communicator
        (hs_trainer_sharded_step): exchanges, gradient all-reduce, agreement on
        the first non-finite group, Adan, loss sums -- all inside the library."""
        self._ctx = ctx_handle()
        if with_loss:
            v = C.c_double(0.0)
            check(_lib.load().hs_trainer_sharded_step(self.h, C.byref(v)))
            return v.value
        check(_lib.load().hs_trainer_sharded_step(self.h, None))
        return None

    def slab_status(self) -> int:
        v = C.c_uint32(0)
        check(_lib.load().hs_trainer_slab_status(self.h, C.byref(v)))
        return int(v.value)


def comm_unique_id() -> bytes:
    """ncclGetUniqueId (hs_comm_unique_id): 128 bytes to ship to every rank."""
    buf = (C.c_char * 128)()
    check(_lib.load().hs_comm_unique_id(buf))
    return bytes(buf)


def ctx_comm_init(uid: bytes, nranks: int, rank: int, device=None):
    """Creates the NCCL communicator inside this device's context (hs_ctx_comm_init)."""
    buf = (C.c_char * 128).from_buffer_copy(uid)
    check(_lib.load().hs_ctx_comm_init(ctx_handle(device), buf, int(nranks), int(rank)))


def ctx_comm_destroy(device=None):
    check(_lib.load().hs_ctx_comm_destroy(ctx_handle(device)))


def ipc_handle(d_ptr: int) -> bytes:
    """cudaIpcGetMemHandle of a device allocation (64 bytes)."""
    buf = C.create_string_buffer(64)
    check(_lib.load().hs_ipc_get_handle(C.c_void_p(int(d_ptr)), buf))
    return buf.raw


def ipc_open(handle: bytes) -> int:
    """cudaIpcOpenMemHandle (lazy peer access): the peer allocation mapped here."""
    p = C.c_void_p()
    buf = C.create_string_buffer(bytes(handle), 64)
    check(_lib.load().hs_ipc_open_handle(buf, C.byref(p)))
    return int(p.value)


def _wrap(owner, ptr, count, typestr="<f4") -> torch.Tensor:
    """torch view over trainer-owned device memory (kept alive by owner)."""
    class _Holder:
        pass

    dev = torch.cuda.current_device()
    iface = {"shape": (count,), "typestr": typestr, "data": (int(ptr), False), "version": 3,
             "strides": None}
    holder = _Holder()
    holder.__cuda_array_interface__ = iface
    holder.owner = owner
    t = torch.as_tensor(holder, device=f"cuda:{dev}")
    return t
