"""Deterministic synthetic inputs, restating the reference's generators.

* ``Rng``            holo::Rng (proj/core/include/holo/rng.hpp:11-24): std::mt19937_64
                     with the 53-bit mapping ``(x >> 11) * 2^-53``.
* ``init_gaussians`` pipeline.cpp:175-200 (draw order x,y per n, then amplitudes).
* ``resolve_gaussian_count`` pipeline.cpp:165-173.
* ``synthetic_image`` / ``synthetic_depth`` / ``random_set`` / ``random_field`` /
  ``random_real``  tests/test_util.hpp:16-111.

Host-side input generation for bench.py and the tests (the reference's own
tests use the same fixtures); the draw sequences are bit-identical with the
reference (checked against oracle/_ref in tests/test_oracle_ref.py).
"""
from __future__ import annotations

import math

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_UM = np.uint64(0xFFFFFFFF80000000)
_LM = np.uint64(0x7FFFFFFF)
_MATA = np.uint64(0xB5026F5AA96619E9)


class Rng:
    """std::mt19937_64 + holo's uniform mapping (vectorised twist)."""

    NN, MM = 312, 156

    def __init__(self, seed: int):
        mt = [0] * self.NN
        mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, self.NN):
            prev = mt[i - 1]
            mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.mt = np.array(mt, dtype=np.uint64)
        self.idx = self.NN
        self.buf = np.empty(0, dtype=np.uint64)
        self.pos = 0

    def _twist(self):
        mt, NN, MM = self.mt, self.NN, self.MM
        with np.errstate(over="ignore"):
            def mix(a, b, c):  # new = c ^ (((a & UM) | (b & LM)) >> 1) ^ (odd * MATA)
                x = (a & _UM) | (b & _LM)
                xa = x >> np.uint64(1)
                xa = np.where((x & np.uint64(1)) != 0, xa ^ _MATA, xa)
                return c ^ xa
            mt[0:MM] = mix(mt[0:MM], mt[1:MM + 1], mt[MM:NN])
            mt[MM:NN - 1] = mix(mt[MM:NN - 1], mt[MM + 1:NN], mt[0:NN - MM - 1])
            mt[NN - 1:NN] = mix(mt[NN - 1:NN], mt[0:1], mt[MM - 1:MM])
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        return y

    def raw(self, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.uint64)
        got = 0
        while got < count:
            if self.pos >= self.buf.size:
                self.buf = self._twist()
                self.pos = 0
            take = min(count - got, self.buf.size - self.pos)
            out[got:got + take] = self.buf[self.pos:self.pos + take]
            self.pos += take
            got += take
        return out

    def uniform(self, count: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        u = (self.raw(count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        if lo == 0.0 and hi == 1.0:
            return u
        return lo + (hi - lo) * u


def unactivate_position(value, extent):
    """field_core.cpp:39-41."""
    return np.arctanh(2.0 * value / extent - 1.0)


def resolve_gaussian_count(channels: int, width: int, height: int, gaussian_count: int = 0,
                           parameter_ratio: float = 0.0) -> int:
    """pipeline.cpp:165-173: N = round(2 C H W / (12 r))."""
    if gaussian_count > 0:
        return gaussian_count
    if parameter_ratio > 0.0:
        dense = 2.0 * channels * width * height
        n = int(math.floor(dense / (12.0 * parameter_ratio) + 0.5))  # lround (positive)
        return max(n, 1)
    raise ValueError("config: neither gaussian_count nor parameter_ratio set")


def init_gaussians(count: int, channels: int, width: int, height: int, seed: int) -> dict:
    """pipeline.cpp:175-200; returns the six fp64 groups."""
    if count < 1:
        raise ValueError("init_gaussians: count must be >= 1")
    rng = Rng(seed)
    xy = rng.uniform(2 * count)
    x = 0.0 + (float(width) - 0.0) * xy[0::2]
    y = 0.0 + (float(height) - 0.0) * xy[1::2]
    nx, ny = 1e-6 * width, 1e-6 * height
    x = np.where(x <= 0.0, nx, x)
    x = np.where(x >= width, width - nx, x)
    y = np.where(y <= 0.0, ny, y)
    y = np.where(y >= height, height - ny, y)
    pos = np.empty(2 * count)
    pos[0::2] = unactivate_position(x, width)
    pos[1::2] = unactivate_position(y, height)
    scale = np.empty(2 * count)
    scale[0::2] = math.log(1.5)
    scale[1::2] = math.log(5.0)
    amp = rng.uniform(count * channels)
    return dict(pre_position=pos, pre_scale=scale, rotation=np.zeros(count), amplitude=amp,
                phase=np.zeros(count * channels), pre_opacity=np.full(count, -0.5))


def random_set(seed: int, count: int, channels: int) -> dict:
    """test_util.hpp:16-37."""
    rng = Rng(seed)
    per = 6 + 2 * channels
    u = rng.uniform(per * count).reshape(count, per)
    lo4, hi4 = math.log(0.5), math.log(4.0)
    pos = np.empty(2 * count)
    pos[0::2] = -1.5 + 3.0 * u[:, 0]
    pos[1::2] = -1.5 + 3.0 * u[:, 1]
    sc = np.empty(2 * count)
    sc[0::2] = lo4 + (hi4 - lo4) * u[:, 2]
    sc[1::2] = lo4 + (hi4 - lo4) * u[:, 3]
    rot = -3.2 + 6.4 * u[:, 4]
    op = -3.0 + 6.0 * u[:, 5]
    amp = -0.2 + (1.2 - -0.2) * u[:, 6::2]
    ph = -3.2 + 6.4 * u[:, 7::2]
    return dict(pre_position=pos, pre_scale=sc, rotation=rot, amplitude=amp.reshape(-1),
                phase=ph.reshape(-1), pre_opacity=op)


def random_field(seed: int, c: int, h: int, w: int, amp: float = 1.0):
    """test_util.hpp:39-48 -> (real, imag) C x H x W."""
    u = Rng(seed).uniform(2 * c * h * w)
    v = -amp + (amp - -amp) * u
    return v[0::2].reshape(c, h, w), v[1::2].reshape(c, h, w)


def random_real(seed: int, c: int, h: int, w: int, lo: float, hi: float):
    """test_util.hpp:50-55."""
    return (lo + (hi - lo) * Rng(seed).uniform(c * h * w)).reshape(c, h, w)


def synthetic_image(seed: int, channels: int, height: int, width: int) -> np.ndarray:
    """test_util.hpp:57-94, C x H x W in [0.02, 0.98]."""
    rng = Rng(seed)
    blobs = 6
    u = rng.uniform(blobs * (4 + channels)).reshape(blobs, 4 + channels)
    bx = (0.1 + 0.8 * u[:, 0]) * width
    by = (0.1 + 0.8 * u[:, 1]) * height
    bsx = (0.05 + 0.15 * u[:, 2]) * width
    bsy = (0.05 + 0.15 * u[:, 3]) * height
    ba = -0.25 + 0.6 * u[:, 4:]
    rx0, rx1 = 0.15 * width, 0.4 * width
    ry0, ry1 = 0.55 * height, 0.8 * height
    rcx, rcy = 0.7 * width, 0.35 * height
    rr0, rw = 0.18 * min(width, height), 0.05 * min(width, height)
    yy, xx = np.meshgrid(np.arange(height, dtype=np.float64), np.arange(width, dtype=np.float64),
                         indexing="ij")
    img = np.empty((channels, height, width))
    rect = (xx >= rx0) & (xx <= rx1) & (yy >= ry0) & (yy <= ry1)
    rr = np.hypot(xx - rcx, yy - rcy) - rr0
    ring = 0.22 * np.exp(-0.5 * (rr / rw) * (rr / rw))
    tex = 0.025 * np.sin(2.0 * 3.14159265358979 * xx / 31.0) * np.sin(2.0 * 3.14159265358979 * yy / 23.0)
    for c in range(channels):
        v = 0.3 + 0.35 * (xx / width) + 0.2 * (yy / height) + 0.04 * (c - (channels - 1) * 0.5)
        for k in range(blobs):
            dx = (xx - bx[k]) / bsx[k]
            dy = (yy - by[k]) / bsy[k]
            v = v + ba[k, c] * np.exp(-0.5 * (dx * dx + dy * dy))
        v = v + np.where(rect, 0.18, 0.0)
        v = v + ring
        v = v + tex
        img[c] = np.minimum(0.98, np.maximum(0.02, v))
    return img


def synthetic_depth(seed: int, height: int, width: int) -> np.ndarray:
    """test_util.hpp:97-111, H x W in [0, 1]."""
    u = Rng(seed).uniform(2)
    cx = (0.3 + 0.4 * u[0]) * width
    cy = (0.3 + 0.4 * u[1]) * height
    sx, sy = 0.25 * width, 0.25 * height
    yy, xx = np.meshgrid(np.arange(height, dtype=np.float64), np.arange(width, dtype=np.float64),
                         indexing="ij")
    ddx, ddy = (xx - cx) / sx, (yy - cy) / sy
    v = 0.25 + 0.45 * ((xx + yy) / (width + height)) + 0.4 * np.exp(-0.5 * (ddx * ddx + ddy * ddy))
    return np.minimum(1.0, np.maximum(0.0, v))


def build_masks(depth: np.ndarray, plane_count: int, near_is_high: bool = True) -> np.ndarray:
    """build_masks, loss.cpp:166-180 (host, bit-exact): L x H x W uint8."""
    if plane_count < 1:
        raise ValueError("build_masks: plane count must be >= 1")
    h, w = depth.shape
    b = np.floor(depth * plane_count).astype(np.int64)
    b = np.clip(b, 0, plane_count - 1)
    plane = plane_count - 1 - b if near_is_high else b
    out = np.zeros((plane_count, h, w), dtype=np.uint8)
    for l in range(plane_count):
        out[l][plane == l] = 1
    return out


def make_depth_planes(count: int, d0: float, dz: float):
    """make_depth_planes, loss.cpp:154-164."""
    return [d0 + (l - (count - 1) * 0.5) * dz for l in range(count)]


# Benchmark / parity workloads
CONFIGS = {
    "cfg1": dict(width=256, height=256, channels=1, count=10_000, planes=1, dz=2e-3),
    "cfg2": dict(width=1920, height=1080, channels=3, count=200_000, planes=1, dz=2e-3),
    "cfg3": dict(width=1920, height=1080, channels=3, count=200_000, planes=8, dz=4e-3 / 7),
    "cfg4": dict(width=3840, height=2160, channels=3, count=1_000_000, planes=1, dz=2e-3),
    "desk": dict(width=256, height=160, channels=1, count=3413, planes=2, dz=2e-3),
    # cfg5: one scene of the 64-scene conversion batch (N from ratio 5: round(2 C H W / 60))
    "cfg5": dict(width=1920, height=1080, channels=3, count=207_360, planes=2, dz=2e-3),
}
WAVELENGTHS = {1: (532e-9,), 2: (639e-9, 473e-9), 3: (639e-9, 532e-9, 473e-9)}


def workload(name: str, scene: int = 0):
    """Inputs of a named config: gaussians (dict of fp64 groups), target, depth,
    masks, distances, wavelengths.  Seeds follow SURVEY §8(d)."""
    cfg = dict(CONFIGS[name])
    w, h, c = cfg["width"], cfg["height"], cfg["channels"]
    target = synthetic_image(42 + 2 * scene, c, h, w)
    depth = synthetic_depth(43 + 2 * scene, h, w)
    masks = build_masks(depth, cfg["planes"], True)
    dist = make_depth_planes(cfg["planes"], 3e-3, cfg["dz"])
    g = init_gaussians(cfg["count"], c, w, h, 42 + scene)
    return dict(cfg=cfg, gaussians=g, target=target, depth=depth, masks=masks, distances=dist,
                wavelengths=WAVELENGTHS[c])


# ---- train()'s PNG round trip of its inputs (io.cpp:228-235, 337-395) ----------------------------
def srgb_to_linear(s):
    """io.cpp:228-230."""
    s = np.asarray(s, dtype=np.float64)
    return np.where(s <= 0.04045, s / 12.92, np.power((s + 0.055) / 1.055, 2.4))


def linear_to_srgb(v):
    """io.cpp:232-235."""
    v = np.clip(np.asarray(v, dtype=np.float64), 0.0, 1.0)
    return np.where(v <= 0.0031308, 12.92 * v, 1.055 * np.power(v, 1.0 / 2.4) - 0.055)


def _lround(x):
    return np.floor(np.asarray(x, dtype=np.float64) + 0.5)  # std::lround on non-negative values


def png8_srgb_roundtrip(img: np.ndarray) -> np.ndarray:
    """write_image_srgb (io.cpp:353-368: lround(srgb * 255) into 8 bits) followed by
    read_image_linear (io.cpp:337-351: srgb_to_linear(v / 255)): the intensity target
    train() sees for an image written by the reference's tests."""
    q = _lround(linear_to_srgb(img) * 255.0)
    return srgb_to_linear(q / 255.0)


def png16_depth_roundtrip(depth: np.ndarray) -> np.ndarray:
    """write_depth_png(..., 16) (io.cpp:378-390) followed by read_depth (io.cpp:370-376)."""
    q = _lround(np.clip(depth, 0.0, 1.0) * 65535.0)
    return q / 65535.0


def desk_scene(ratio: float):
    """The reference's end-to-end desk regression (acceptance.cpp:303-334, criteria 6/7):
    a 256x160 grayscale synthetic image (seed 42) and depth (seed 43) written as an 8-bit
    sRGB / 16-bit PNG and read back by train(), two planes (3 mm centre, 2 mm spacing),
    532 nm, N from the parameter ratio, Gaussians from seed 42, 2000 steps."""
    w, h, c, L = 256, 160, 1, 2
    target = png8_srgb_roundtrip(synthetic_image(42, c, h, w))
    depth = png16_depth_roundtrip(synthetic_depth(43, h, w))
    n = resolve_gaussian_count(c, w, h, parameter_ratio=ratio)
    return dict(width=w, height=h, channels=c, count=n, target=target, depth=depth,
                masks=build_masks(depth, L, True), distances=make_depth_planes(L, 3e-3, 2e-3),
                gaussians=init_gaussians(n, c, w, h, 42), steps=2000, wavelengths=(532e-9,))
