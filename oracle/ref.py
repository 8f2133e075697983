"""Test infrastructure (oracle) -- NOT part of the product path.

ctypes binding of oracle/_ref/libholoref.so, i.e. the UNMODIFIED reference
library (/root/reference/proj/core) compiled by oracle/Makefile, through the
extern "C" adaptor oracle/ref_capi.cpp.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference leg import this module.

Arrays follow the reference layouts (proj/core/include/holo/*.hpp):
GaussianSet = six fp64 arrays (pre_position 2N xy-interleaved, pre_scale 2N,
rotation N, amplitude N*C, phase N*C, pre_opacity N); fields planar C*H*W.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libholoref.so")

_lib = None

GROUPS = ("pre_position", "pre_scale", "rotation", "amplitude", "phase", "pre_opacity")


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run make -C oracle)")
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_build_tile_index.restype = C.c_int64
        _lib.ref_cosine_lr.restype = C.c_double
        _lib.ref_adan_create.restype = C.c_void_p
        _lib.ref_trainer_create.restype = C.c_void_p
        for name in ("ref_adan_destroy", "ref_trainer_destroy", "ref_trainer_step",
                     "ref_trainer_params", "ref_trainer_stage_ms", "ref_adan_add_group",
                     "ref_adan_set_lr", "ref_adan_step"):
            getattr(_lib, name).argtypes = None
    return _lib


class RefError(RuntimeError):
    pass


class RefInvalidArgument(RefError, ValueError):
    pass


def _check(rc):
    if rc < 0:
        msg = lib().ref_last_error().decode()
        if rc == -1:
            raise RefInvalidArgument(msg)
        raise RefError(msg)
    return rc


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _d(x):
    return C.c_double(float(x))


@dataclass
class GaussianSet:
    """fp64 host mirror of holo::GaussianSet (gaussian_set.hpp:12-30)."""
    count: int
    channels: int
    pre_position: np.ndarray
    pre_scale: np.ndarray
    rotation: np.ndarray
    amplitude: np.ndarray
    phase: np.ndarray
    pre_opacity: np.ndarray

    @classmethod
    def empty(cls, n, c):
        return cls(n, c, np.zeros(2 * n), np.zeros(2 * n), np.zeros(n), np.zeros(n * c),
                   np.zeros(n * c), np.zeros(n))

    def arrays(self):
        return [np.ascontiguousarray(getattr(self, g), dtype=np.float64) for g in GROUPS]

    def ptrs(self):
        self._keep = self.arrays()
        return [_p(a) for a in self._keep]

    def rounded_f32(self):
        """Same set with every value rounded to fp32 (the parity protocol)."""
        return GaussianSet(self.count, self.channels,
                           *[a.astype(np.float32).astype(np.float64) for a in self.arrays()])

    def flat(self):
        return np.concatenate(self.arrays())


def random_set(seed, count, channels, width, height) -> GaussianSet:
    s = GaussianSet.empty(count, channels)
    _check(lib().ref_random_set(C.c_uint64(seed), count, channels, width, height, *s.ptrs()))
    return s


def init_gaussians(count, channels, width, height, seed) -> GaussianSet:
    s = GaussianSet.empty(count, channels)
    _check(lib().ref_init_gaussians(count, channels, width, height, C.c_uint64(seed), *s.ptrs()))
    return s


def random_field(seed, c, h, w, amp=1.0):
    re = np.zeros(c * h * w)
    im = np.zeros(c * h * w)
    _check(lib().ref_random_field(C.c_uint64(seed), c, h, w, _d(amp), _p(re), _p(im)))
    return re.reshape(c, h, w), im.reshape(c, h, w)


def random_real(seed, c, h, w, lo, hi):
    out = np.zeros(c * h * w)
    _check(lib().ref_random_real(C.c_uint64(seed), c, h, w, _d(lo), _d(hi), _p(out)))
    return out.reshape(c, h, w)


def synthetic_image(seed, c, h, w):
    out = np.zeros(c * h * w)
    _check(lib().ref_synthetic_image(C.c_uint64(seed), c, h, w, _p(out)))
    return out.reshape(c, h, w)


def synthetic_depth(seed, h, w):
    out = np.zeros(h * w)
    _check(lib().ref_synthetic_depth(C.c_uint64(seed), h, w, _p(out)))
    return out.reshape(h, w)


def resolve_gaussian_count(ratio, count, c, w, h):
    return lib().ref_resolve_gaussian_count(_d(ratio), count, c, w, h)


def activations(pre, extent):
    out = np.zeros(8)
    _check(lib().ref_activations(_d(pre), _d(extent), _p(out)))
    return out


def covariance(sx, sy, theta):
    out = np.zeros(7)
    _check(lib().ref_covariance(_d(sx), _d(sy), _d(theta), _p(out)))
    return out


def build_tile_index(s: GaussianSet, width, height):
    txy = np.zeros(2, dtype=np.int32)
    tiles_n = ((width + 15) // 16) * ((height + 15) // 16) if width > 0 and height > 0 else 0
    ranges = np.zeros(2 * max(tiles_n, 1), dtype=np.uint64)
    ptrs = s.ptrs()
    k = lib().ref_build_tile_index(s.count, s.channels, *ptrs, width, height, None, None,
                                   _p(ranges), C.c_int64(-1), _p(txy))
    _check(k)
    tiles = np.zeros(max(k, 1), dtype=np.uint32)
    ids = np.zeros(max(k, 1), dtype=np.uint32)
    k2 = lib().ref_build_tile_index(s.count, s.channels, *ptrs, width, height, _p(tiles), _p(ids),
                                    _p(ranges), C.c_int64(k), _p(txy))
    _check(k2)
    return dict(tiles_x=int(txy[0]), tiles_y=int(txy[1]), tiles=tiles[:k], ids=ids[:k],
                ranges=ranges[:2 * tiles_n].reshape(-1, 2))


def rasterize_forward(s: GaussianSet, width, height):
    re = np.zeros(s.channels * height * width)
    im = np.zeros_like(re)
    _check(lib().ref_rasterize_forward(s.count, s.channels, *s.ptrs(), width, height, _p(re), _p(im)))
    return re.reshape(s.channels, height, width), im.reshape(s.channels, height, width)


def brute_rasterize(s: GaussianSet, width, height):
    re = np.zeros(s.channels * height * width)
    im = np.zeros_like(re)
    cnt = np.zeros(3, dtype=np.int64)
    _check(lib().ref_brute_rasterize(s.count, s.channels, *s.ptrs(), width, height, _p(re), _p(im),
                                     _p(cnt)))
    return re.reshape(s.channels, height, width), im.reshape(s.channels, height, width), cnt


def rasterize_backward(s: GaussianSet, grad_re, grad_im) -> GaussianSet:
    c, h, w = grad_re.shape
    gre = np.ascontiguousarray(grad_re, dtype=np.float64)
    gim = np.ascontiguousarray(grad_im, dtype=np.float64)
    out = GaussianSet.empty(s.count, s.channels)
    _check(lib().ref_rasterize_backward(s.count, s.channels, *s.ptrs(), w, h, _p(gre), _p(gim),
                                        *out.ptrs()))
    for g, a in zip(GROUPS, out._keep):
        setattr(out, g, a)
    return out


@dataclass
class PropagationSpec:
    """holo::PropagationSpec (propagation.hpp:9-14)."""
    wavelengths: tuple = (639e-9, 532e-9, 473e-9)
    pixel_pitch: float = 3.74e-6
    pad_factor: int = 2
    aperture_radius: float = 0.0


def _spec_args(spec: PropagationSpec):
    wl = np.ascontiguousarray(spec.wavelengths, dtype=np.float64)
    return wl, [_p(wl), _d(spec.pixel_pitch), int(spec.pad_factor), _d(spec.aperture_radius)]


def propagate(re, im, spec, distance, mode=0, mask_distance=0.0):
    """mode 0 propagate, 1 propagate_with_mask_distance, 2 propagate_backward,
    3 oracle::direct_dft_propagate."""
    c, h, w = re.shape
    re = np.ascontiguousarray(re, dtype=np.float64)
    im = np.ascontiguousarray(im, dtype=np.float64)
    ore = np.zeros_like(re)
    oim = np.zeros_like(im)
    wl, sa = _spec_args(spec)
    _check(lib().ref_propagate(mode, c, h, w, _p(re), _p(im), *sa, _d(distance), _d(mask_distance),
                               _p(ore), _p(oim)))
    return ore, oim


def propagate_multi(re, im, spec, distances):
    c, h, w = re.shape
    L = len(distances)
    re = np.ascontiguousarray(re, dtype=np.float64)
    im = np.ascontiguousarray(im, dtype=np.float64)
    ore = np.zeros((L, c, h, w))
    oim = np.zeros((L, c, h, w))
    d = np.ascontiguousarray(distances, dtype=np.float64)
    wl, sa = _spec_args(spec)
    _check(lib().ref_propagate_multi(c, h, w, _p(re), _p(im), *sa, _p(d), L, _p(ore), _p(oim)))
    return ore, oim


def propagate_multi_backward(gre, gim, spec, distances):
    L, c, h, w = gre.shape
    gre = np.ascontiguousarray(gre, dtype=np.float64)
    gim = np.ascontiguousarray(gim, dtype=np.float64)
    ore = np.zeros((c, h, w))
    oim = np.zeros((c, h, w))
    d = np.ascontiguousarray(distances, dtype=np.float64)
    wl, sa = _spec_args(spec)
    _check(lib().ref_propagate_multi_backward(c, h, w, _p(gre), _p(gim), *sa, _p(d), L, _p(ore),
                                              _p(oim)))
    return ore, oim


def transfer_function(spec, distance, channel, pnx, pny):
    out = np.zeros((pny * pnx, 4))
    wl, _ = _spec_args(spec)
    _check(lib().ref_transfer_function(_p(wl), len(wl), _d(spec.pixel_pitch), int(spec.pad_factor),
                                       _d(spec.aperture_radius), _d(distance), channel, pnx, pny,
                                       _p(out)))
    return out


def build_masks(depth, L, near_is_high=True):
    h, w = depth.shape
    d = np.ascontiguousarray(depth, dtype=np.float64)
    out = np.zeros((L, h, w), dtype=np.uint8)
    _check(lib().ref_build_masks(_p(d), h, w, L, int(near_is_high), _p(out)))
    return out


def make_depth_planes(count, d0, dz):
    out = np.zeros(count)
    _check(lib().ref_make_depth_planes(count, _d(d0), _d(dz), _p(out)))
    return out


LOSS_KINDS = dict(training=0, recon=1, ssim=2, mse=3, training_value=10, recon_value=11,
                  ssim_value=12, mse_value=13, loop_recon=20, loop_ssim=21, loop_mse=22)


def loss(kind, recon, target, depth, near_is_high=True):
    """recon: (L,C,H,W) intensities; target (C,H,W); depth (H,W). Returns (loss, grads)."""
    L, c, h, w = recon.shape
    r = np.ascontiguousarray(recon, dtype=np.float64)
    t = np.ascontiguousarray(target, dtype=np.float64)
    d = np.ascontiguousarray(depth, dtype=np.float64)
    g = np.zeros_like(r)
    v = C.c_double(0.0)
    _check(lib().ref_loss(LOSS_KINDS[kind], L, c, h, w, _p(r), _p(t), _p(d), int(near_is_high),
                          _p(g), C.byref(v)))
    return v.value, g


def cosine_lr(step, total, lr_max, lr_min):
    rc = C.c_int(0)
    v = lib().ref_cosine_lr(step, total, _d(lr_max), _d(lr_min), C.byref(rc))
    _check(rc.value)
    return v


class Adan:
    """holo::Adan (optimizer.hpp:23-49) driven through the adaptor."""

    def __init__(self):
        self._h = C.c_void_p(lib().ref_adan_create())

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ref_adan_destroy(self._h)
            self._h = None

    def add_group(self, name, size, lr):
        _check(lib().ref_adan_add_group(self._h, name.encode(), C.c_int64(size), _d(lr)))

    def set_lr(self, name, lr):
        _check(lib().ref_adan_set_lr(self._h, name.encode(), _d(lr)))

    def step(self, name, params: np.ndarray, grads: np.ndarray):
        assert params.dtype == np.float64 and params.flags.c_contiguous
        g = np.ascontiguousarray(grads, dtype=np.float64)
        _check(lib().ref_adan_step(self._h, name.encode(), _p(params), _p(g),
                                   C.c_int64(params.size), C.c_int64(g.size)))


class Trainer:
    """Reference step loop (pipeline.cpp:243-297) over given inputs."""

    def __init__(self, s: GaussianSet, width, height, target, depth, L, d0, dz, spec,
                 total_steps, near_is_high=True):
        self.s = s
        t = np.ascontiguousarray(target, dtype=np.float64)
        d = np.ascontiguousarray(depth, dtype=np.float64)
        wl, sa = _spec_args(spec)
        h = lib().ref_trainer_create(s.count, s.channels, *s.ptrs(), width, height, _p(t), _p(d),
                                     L, _d(d0), _d(dz), int(near_is_high), *sa, total_steps)
        if not h:
            raise RefError(lib().ref_last_error().decode())
        self._h = C.c_void_p(h)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ref_trainer_destroy(self._h)
            self._h = None

    def step(self, want_grads=False):
        v = C.c_double(0.0)
        if want_grads:
            g = GaussianSet.empty(self.s.count, self.s.channels)
            _check(lib().ref_trainer_step(self._h, C.byref(v), *g.ptrs()))
            for name, a in zip(GROUPS, g._keep):
                setattr(g, name, a)
            return v.value, g
        _check(lib().ref_trainer_step(self._h, C.byref(v), *([None] * 6)))
        return v.value

    def params(self) -> GaussianSet:
        g = GaussianSet.empty(self.s.count, self.s.channels)
        _check(lib().ref_trainer_params(self._h, *g.ptrs()))
        for name, a in zip(GROUPS, g._keep):
            setattr(g, name, a)
        return g

    def stage_ms(self):
        out = np.zeros(7)
        lib().ref_trainer_stage_ms(self._h, _p(out))
        return out


def set_thread_count(n):
    lib().ref_set_thread_count(int(n))


# ---- POH conversion (convert.cpp) ---------------------------------------------------------------
def dpac_encode(re, im, mode=0):
    c, h, w = re.shape
    re = np.ascontiguousarray(re, dtype=np.float64)
    im = np.ascontiguousarray(im, dtype=np.float64)
    out = np.zeros((c, h, w))
    _check(lib().ref_dpac_encode(c, h, w, _p(re), _p(im), int(mode), _p(out)))
    return out


def poh_field(phase):
    c, h, w = phase.shape
    phase = np.ascontiguousarray(phase, dtype=np.float64)
    re, im = np.zeros((c, h, w)), np.zeros((c, h, w))
    _check(lib().ref_poh_field(c, h, w, _p(phase), _p(re), _p(im)))
    return re, im


def convert_random_poh_field(gre, gim, target, depth, L, distances, spec, steps, seed=0,
                             lambda_comp=0.1, lambda_field=0.01, lr=2.5e-3, log_every=50, near_is_high=True):
    """The reference's convert_random_poh_field; target stack = make_target_stack(target, depth, L)."""
    c, h, w = gre.shape
    gre = np.ascontiguousarray(gre, dtype=np.float64)
    gim = np.ascontiguousarray(gim, dtype=np.float64)
    target = np.ascontiguousarray(target, dtype=np.float64)
    depth = np.ascontiguousarray(depth, dtype=np.float64)
    d = np.ascontiguousarray(distances, dtype=np.float64)
    wl, sa = _spec_args(spec)
    phase = np.zeros((c, h, w))
    loss = np.zeros(steps + 1)
    n = _check(lib().ref_convert_random_poh_field(
        c, h, w, _p(gre), _p(gim), _p(target), _p(depth), int(near_is_high), _p(d), int(L), *sa, int(steps),
        C.c_uint64(seed), _d(lambda_comp), _d(lambda_field), _d(lr), int(log_every), _p(phase), _p(loss),
        len(loss)))
    return phase, loss[:n]


def compute_metrics(recon, target):
    """pipeline.cpp:149-163: per-plane (psnr, ssim) of clipped reconstructions."""
    L, c, h, w = recon.shape
    recon = np.ascontiguousarray(recon, dtype=np.float64)
    target = np.ascontiguousarray(target, dtype=np.float64)
    psnr, ssim = np.zeros(L), np.zeros(L)
    _check(lib().ref_compute_metrics(L, c, h, w, _p(recon), _p(target), _p(psnr), _p(ssim)))
    return psnr, ssim


# ---- artifact formats (io.cpp:237-335: the reference's own CGHF / CGGS code) --------------------
def write_field(path, re, im, as_f64=True):
    c, h, w = re.shape
    re = np.ascontiguousarray(re, dtype=np.float64)
    im = np.ascontiguousarray(im, dtype=np.float64)
    _check(lib().ref_write_field(str(path).encode(), c, h, w, _p(re), _p(im), int(as_f64)))


def read_field(path):
    chw = (C.c_int * 3)()
    _check(lib().ref_read_field(str(path).encode(), chw, None, None))
    c, h, w = chw
    re, im = np.zeros((c, h, w)), np.zeros((c, h, w))
    _check(lib().ref_read_field(str(path).encode(), chw, _p(re), _p(im)))
    return re, im


def write_gaussians(path, s: GaussianSet):
    _check(lib().ref_write_gaussians(str(path).encode(), s.count, s.channels, *s.ptrs()))


def read_gaussians(path) -> GaussianSet:
    nc = (C.c_int * 2)()
    _check(lib().ref_read_gaussians(str(path).encode(), nc, *([None] * 6)))
    g = GaussianSet.empty(nc[0], nc[1])
    _check(lib().ref_read_gaussians(str(path).encode(), nc, *g.ptrs()))
    for name, a in zip(GROUPS, g._keep):
        setattr(g, name, a)
    return g
