"""Test infrastructure (oracle) -- NOT part of the product path.

fp64 numpy restatement of the reference's optimisation hot path, written from
the reference sources (each function cites the file:line it follows, paths
relative to /root/reference/proj/core/src).  Used by the CPU tests to pin the
golden vectors / known-answer tests of the reference's own test-suite and to
cross-check oracle/_ref; the GPU parity tests compare the CUDA path against
oracle/_ref (the reference compiled from its own sources) and this module.

FFTW3 (the reference's third-party FFT, unpinned version) is restated by
numpy.fft (pocketfft): both compute the unnormalised DFT with the sign
conventions FFTW_FORWARD=-1 / FFTW_BACKWARD=+1 (propagation.cpp:27-39).
"""
from __future__ import annotations

import math

import numpy as np

GROUPS = ("pre_position", "pre_scale", "rotation", "amplitude", "phase", "pre_opacity")
kEpsScale, kEpsCov, kEpsDet = 0.1, 0.1, 1e-10          # field_core.hpp:10-12
kPowerFloor, kAlphaCap, kAlphaCutoff = -50.0, 0.99, 1.0 / 255.0  # field_core.hpp:13-15
kMahalSlack = 1e-9                                     # rasterizer.cpp:17
kTile = 16                                             # rasterizer.hpp:12
kSsimWin, kSsimSigma, kSsimC1, kSsimC2, kSsimWeight = 11, 1.5, 0.01 ** 2, 0.03 ** 2, 0.005  # loss.hpp:10-14


# ---- field_core.cpp ------------------------------------------------------------------
def activate_position(pre, extent):          # :11-14
    pre = np.asarray(pre, dtype=np.float64)
    if not np.all(np.isfinite(pre)):
        raise ValueError("activate_position: non-finite input")
    return (np.tanh(pre) + 1.0) * 0.5 * extent


def activate_position_deriv(pre, extent):    # :16-19
    t = np.tanh(pre)
    return 0.5 * extent * (1.0 - t * t)


def activate_scale(pre):                     # :21-24
    pre = np.asarray(pre, dtype=np.float64)
    if not np.all(np.isfinite(pre)):
        raise ValueError("activate_scale: non-finite input")
    return np.exp(pre) + kEpsScale


def activate_scale_deriv(pre):               # :26
    return np.exp(pre)


def activate_opacity(pre):                   # :28-31
    pre = np.asarray(pre, dtype=np.float64)
    if not np.all(np.isfinite(pre)):
        raise ValueError("activate_opacity: non-finite input")
    return 1.0 / (1.0 + np.exp(-pre))


def activate_opacity_deriv(pre):             # :33-36
    s = activate_opacity(pre)
    return s * (1.0 - s)


def activate_amplitude(raw):                 # :38
    return np.clip(raw, 0.0, 1.0)


def activate_amplitude_deriv(raw):           # :40
    raw = np.asarray(raw)
    return np.where((raw >= 0.0) & (raw <= 1.0), 1.0, 0.0)


def unactivate_position(value, extent):      # :42-44
    return np.arctanh(2.0 * value / extent - 1.0)


def covariance(sx, sy, theta):               # :46-54
    c, s = np.cos(theta), np.sin(theta)
    sx2, sy2 = sx * sx, sy * sy
    return (sx2 * c * c + sy2 * s * s + kEpsCov, (sx2 - sy2) * c * s, sx2 * s * s + sy2 * c * c + kEpsCov)


def invert_covariance(sxx, sxy, syy):        # :56-68
    det = sxx * syy - sxy * sxy
    det_safe = np.maximum(det, kEpsDet)
    inv = (syy / det_safe, -sxy / det_safe, sxx / det_safe)
    mid = 0.5 * (sxx + syy)
    half = 0.5 * (sxx - syy)
    lmax = mid + np.sqrt(np.maximum(half * half + sxy * sxy, 0.0))
    return inv, 3.0 * np.sqrt(np.maximum(lmax, 0.0))


# ---- rasterizer.cpp ---------------------------------------------------------------------
def split(flat, n, c):
    flat = np.asarray(flat, dtype=np.float64)
    sizes = [2 * n, 2 * n, n, n * c, n * c, n]
    out, o = {}, 0
    for g, s in zip(GROUPS, sizes):
        out[g] = flat[o:o + s]
        o += s
    return out


def activate_flat(g, n, c, width, height):   # rasterizer.cpp:33-88
    pp, ps = np.asarray(g["pre_position"]), np.asarray(g["pre_scale"])
    f = {}
    f["px"] = activate_position(pp[0::2], width)
    f["py"] = activate_position(pp[1::2], height)
    f["sx"] = activate_scale(ps[0::2])
    f["sy"] = activate_scale(ps[1::2])
    cov = covariance(f["sx"], f["sy"], np.asarray(g["rotation"], np.float64))
    f["cov"] = cov
    inv, rad3 = invert_covariance(*cov)
    f["inv"] = inv
    alpha = activate_opacity(np.asarray(g["pre_opacity"], np.float64))
    f["alpha"] = alpha
    with np.errstate(divide="ignore"):
        cutoff = 2.0 * np.maximum(np.log(255.0 * alpha), 0.0)
    f["mahal_cutoff"] = cutoff + kMahalSlack
    sigma = rad3 / 3.0
    f["radius"] = sigma * np.sqrt(np.maximum(9.0, cutoff)) + 1.0
    amp = activate_amplitude(np.asarray(g["amplitude"], np.float64)).reshape(n, c)
    ph = np.asarray(g["phase"], np.float64).reshape(n, c)
    f["amp"], f["cos"], f["sin"] = amp, np.cos(ph), np.sin(ph)
    return f


def build_tile_index(g, n, c, width, height):  # rasterizer.cpp:90-126
    if width <= 0 or height <= 0:
        raise ValueError("build_tile_index: empty canvas")
    f = activate_flat(g, n, c, width, height)
    tx_n, ty_n = (width + kTile - 1) // kTile, (height + kTile - 1) // kTile
    r = f["radius"]
    tx0 = np.maximum(np.floor((f["px"] - r) / kTile).astype(np.int64), 0)
    tx1 = np.minimum(np.floor((f["px"] + r) / kTile).astype(np.int64), tx_n - 1)
    ty0 = np.maximum(np.floor((f["py"] - r) / kTile).astype(np.int64), 0)
    ty1 = np.minimum(np.floor((f["py"] + r) / kTile).astype(np.int64), ty_n - 1)
    tiles, ids = [], []
    for gi in range(n):
        for ty in range(ty0[gi], ty1[gi] + 1):
            for tx in range(tx0[gi], tx1[gi] + 1):
                tiles.append(ty * tx_n + tx)
                ids.append(gi)
    tiles = np.asarray(tiles, dtype=np.uint32)
    ids = np.asarray(ids, dtype=np.uint32)
    order = np.lexsort((ids, tiles))
    tiles, ids = tiles[order], ids[order]
    ranges = np.zeros((tx_n * ty_n, 2), dtype=np.uint64)
    if tiles.size:
        starts = np.r_[0, np.nonzero(np.diff(tiles))[0] + 1]
        ends = np.r_[starts[1:], tiles.size]
        ranges[tiles[starts], 0] = starts
        ranges[tiles[starts], 1] = ends
    return dict(tiles_x=tx_n, tiles_y=ty_n, tiles=tiles, ids=ids, ranges=ranges)


def _footprint(f, gi, width, height, x0=0, x1=None, y0=0, y1=None):
    """Pixels of Gaussian gi inside [x0,x1) x [y0,y1) that contribute, with
    (dx, dy, G, aeff, saturated) -- rasterizer.cpp:157-176 / :209-228."""
    x1 = width if x1 is None else x1
    y1 = height if y1 is None else y1
    px, py, r = f["px"][gi], f["py"][gi], f["radius"][gi]
    gx0, gx1 = max(x0, int(math.ceil(px - r))), min(x1 - 1, int(math.floor(px + r)))
    gy0, gy1 = max(y0, int(math.ceil(py - r))), min(y1 - 1, int(math.floor(py + r)))
    if gx1 < gx0 or gy1 < gy0:
        return None
    ys, xs = np.meshgrid(np.arange(gy0, gy1 + 1, dtype=np.float64),
                         np.arange(gx0, gx1 + 1, dtype=np.float64), indexing="ij")
    dx, dy = xs - px, ys - py
    i00, i01, i11 = (f["inv"][k][gi] for k in range(3))
    mahal = dx * dx * i00 + 2.0 * dx * dy * i01 + dy * dy * i11
    keep = mahal <= f["mahal_cutoff"][gi]
    power = np.maximum(-0.5 * mahal, kPowerFloor)
    G = np.exp(power)
    aG = f["alpha"][gi] * G
    sat = aG > kAlphaCap
    aeff = np.where(sat, kAlphaCap, aG)
    keep &= ~(aeff < kAlphaCutoff)
    return (ys[keep].astype(np.int64), xs[keep].astype(np.int64), dx[keep], dy[keep], G[keep],
            aeff[keep], sat[keep])


def rasterize_forward(g, n, c, width, height):  # :128-190
    if width <= 0 or height <= 0:
        raise ValueError("rasterize_forward: empty canvas")
    re = np.zeros((c, height, width))
    im = np.zeros((c, height, width))
    if n == 0:
        return re, im
    f = activate_flat(g, n, c, width, height)
    for gi in range(n):  # ascending id per pixel, like the per-tile lists
        fp = _footprint(f, gi, width, height)
        if fp is None:
            continue
        ys, xs, _, _, _, aeff, _ = fp
        for ch in range(c):
            re[ch, ys, xs] += f["amp"][gi, ch] * f["cos"][gi, ch] * aeff
            im[ch, ys, xs] += f["amp"][gi, ch] * f["sin"][gi, ch] * aeff
    return re, im


def rasterize_backward(g, n, c, grad_re, grad_im):  # :192-286
    c2, height, width = grad_re.shape
    if grad_re.shape != grad_im.shape or c2 != c:
        raise ValueError("rasterize_backward: gradient shape mismatch")
    out = {k: np.zeros_like(np.asarray(g[k], np.float64)) for k in GROUPS}
    if n == 0:
        return out
    f = activate_flat(g, n, c, width, height)
    for gi in range(n):
        fp = _footprint(f, gi, width, height)
        d_amp = np.zeros(c)
        d_phase = np.zeros(c)
        d_alpha = gmx = gmy = ga = gb = gc = 0.0
        if fp is not None:
            ys, xs, dx, dy, G, aeff, sat = fp
            s_amp = np.zeros(ys.size)
            for ch in range(c):
                gr, gi_ = grad_re[ch, ys, xs], grad_im[ch, ys, xs]
                cs, sn, a = f["cos"][gi, ch], f["sin"][gi, ch], f["amp"][gi, ch]
                common = cs * gr + sn * gi_
                d_amp[ch] = np.sum(aeff * common)
                d_phase[ch] = np.sum(a * aeff * (-sn * gr + cs * gi_))
                s_amp += a * common
            ns = ~sat
            alpha = f["alpha"][gi]
            i00, i01, i11 = (f["inv"][k][gi] for k in range(3))
            w = s_amp * alpha * G * -0.5
            d_alpha = np.sum((s_amp * G)[ns])
            gmx = np.sum((w * -2.0 * (dx * i00 + dy * i01))[ns])
            gmy = np.sum((w * -2.0 * (dx * i01 + dy * i11))[ns])
            ga = np.sum((w * dx * dx)[ns])
            gb = np.sum((2.0 * w * dx * dy)[ns])
            gc = np.sum((w * dy * dy)[ns])
        amp_raw = np.asarray(g["amplitude"], np.float64)[gi * c:(gi + 1) * c]
        out["amplitude"][gi * c:(gi + 1) * c] = d_amp * activate_amplitude_deriv(amp_raw)
        out["phase"][gi * c:(gi + 1) * c] = d_phase
        out["pre_opacity"][gi] = d_alpha * activate_opacity_deriv(g["pre_opacity"][gi])
        out["pre_position"][2 * gi] = gmx * activate_position_deriv(g["pre_position"][2 * gi], width)
        out["pre_position"][2 * gi + 1] = gmy * activate_position_deriv(g["pre_position"][2 * gi + 1], height)
        c00, c01, c11 = (f["cov"][k][gi] for k in range(3))
        det = c00 * c11 - c01 * c01
        dsafe = max(det, kEpsDet)
        t_adj = ga * c11 - gb * c01 + gc * c00
        cl = 1.0 if det > kEpsDet else 0.0
        d2 = dsafe * dsafe
        gS00 = gc / dsafe - t_adj * (cl * c11) / d2
        gS01 = -gb / dsafe - t_adj * (cl * -2.0 * c01) / d2
        gS11 = ga / dsafe - t_adj * (cl * c00) / d2
        th = g["rotation"][gi]
        ct, st = math.cos(th), math.sin(th)
        sx, sy = f["sx"][gi], f["sy"][gi]
        dsx = 2.0 * sx * (ct * ct * gS00 + ct * st * gS01 + st * st * gS11)
        dsy = 2.0 * sy * (st * st * gS00 - ct * st * gS01 + ct * ct * gS11)
        out["pre_scale"][2 * gi] = dsx * activate_scale_deriv(g["pre_scale"][2 * gi])
        out["pre_scale"][2 * gi + 1] = dsy * activate_scale_deriv(g["pre_scale"][2 * gi + 1])
        out["rotation"][gi] = (2.0 * (sy * sy - sx * sx) * ct * st * gS00
                               + (sx * sx - sy * sy) * (ct * ct - st * st) * gS01
                               + 2.0 * (sx * sx - sy * sy) * ct * st * gS11)
    return out


# ---- propagation.cpp ----------------------------------------------------------------------
def wrapped_freq_index(k, n):                # :44
    k = np.asarray(k)
    return np.where(k < n - n // 2, k, k - n)


def make_band_limit(wavelengths, pitch, mask_distance, channel, pnx, pny):  # make_band_limit :54-70, kz_of :72-75
    if channel < 0 or channel >= len(wavelengths):
        raise ValueError("propagation: channel has no wavelength")
    lam = wavelengths[channel]
    if lam <= 0.0 or pitch <= 0.0:
        raise ValueError("propagation: non-positive wavelength or pitch")
    lx, ly = pnx * pitch, pny * pitch
    return dict(k=2.0 * math.pi / lam, inv_lx=1.0 / lx, inv_ly=1.0 / ly,
                fx_max=1.0 / (lam * math.sqrt((2.0 * mask_distance / lx) ** 2 + 1.0)),
                fy_max=1.0 / (lam * math.sqrt((2.0 * mask_distance / ly) ** 2 + 1.0)))


def transfer(b, ny, nx, phase_distance, aperture):  # apply_transfer :79-109 as a multiplier
    my = wrapped_freq_index(np.arange(ny), ny)[:, None]
    mx = wrapped_freq_index(np.arange(nx), nx)[None, :]
    fy, fx = my * b["inv_ly"], mx * b["inv_lx"]
    inside = (np.abs(fy) < b["fy_max"]) & (np.abs(fx) < b["fx_max"])
    kz2 = b["k"] ** 2 - (2.0 * math.pi) ** 2 * (fx * fx + fy * fy)
    kz = np.where(kz2 > 0.0, np.sqrt(np.maximum(kz2, 0.0)), 0.0)
    ph = kz * phase_distance
    H = np.where(inside, np.cos(ph) + 1j * np.sin(ph), 0.0)
    if aperture > 0.0:
        a2 = aperture * aperture
        H = np.where((mx + 0.5) ** 2 + (my + 0.5) ** 2 >= a2, 0.0, H)
    return H


def _pad(u, py, px):                         # pad_center :111-117
    h, w = u.shape
    buf = np.zeros((py, px), dtype=np.complex128)
    oy, ox = (py - h) // 2, (px - w) // 2
    buf[oy:oy + h, ox:ox + w] = u
    return buf


def _crop(buf, h, w):                        # crop_center :119-127
    py, px = buf.shape
    oy, ox = (py - h) // 2, (px - w) // 2
    return buf[oy:oy + h, ox:ox + w]


def _check_spec(c, wavelengths, pad):        # check_spec :129-133
    if c != len(wavelengths):
        raise ValueError("propagation: channel count does not match wavelengths")
    if pad < 1:
        raise ValueError("propagation: pad_factor must be >= 1")


def propagate_impl(u, wavelengths, pitch, pad, aperture, phase_d, mask_d):  # :135-153
    c, h, w = u.shape
    _check_spec(c, wavelengths, pad)
    px, py = w * pad, h * pad
    out = np.zeros_like(u, dtype=np.complex128)
    for ch in range(c):
        b = make_band_limit(wavelengths, pitch, mask_d, ch, px, py)
        spec = np.fft.fft2(_pad(u[ch], py, px))
        out[ch] = _crop(np.fft.ifft2(spec * transfer(b, py, px, phase_d, aperture)), h, w)
    return out


def propagate(u, wavelengths, pitch, pad, aperture, d):  # :174-177
    if not math.isfinite(d):
        raise ValueError("propagate: non-finite distance")
    return propagate_impl(u, wavelengths, pitch, pad, aperture, d, d)


def propagate_backward(g, wavelengths, pitch, pad, aperture, d):  # :184-187
    return propagate_impl(g, wavelengths, pitch, pad, aperture, -d, d)


def propagate_multi(u, wavelengths, pitch, pad, aperture, distances):  # :189-212
    c, h, w = u.shape
    _check_spec(c, wavelengths, pad)
    px, py = w * pad, h * pad
    out = np.zeros((len(distances), c, h, w), dtype=np.complex128)
    for ch in range(c):
        spec = np.fft.fft2(_pad(u[ch], py, px))
        for l, d in enumerate(distances):
            b = make_band_limit(wavelengths, pitch, d, ch, px, py)
            out[l, ch] = _crop(np.fft.ifft2(spec * transfer(b, py, px, d, aperture)), h, w)
    return out


def propagate_multi_backward(grads, wavelengths, pitch, pad, aperture, distances):  # :214-243
    L, c, h, w = grads.shape
    if L == 0 or L != len(distances):
        raise ValueError("propagate_multi_backward: plane count mismatch")
    _check_spec(c, wavelengths, pad)
    px, py = w * pad, h * pad
    out = np.zeros((c, h, w), dtype=np.complex128)
    for ch in range(c):
        acc = np.zeros((py, px), dtype=np.complex128)
        for l, d in enumerate(distances):
            b = make_band_limit(wavelengths, pitch, d, ch, px, py)
            acc += np.fft.fft2(_pad(grads[l, ch], py, px)) * transfer(b, py, px, -d, aperture)
        out[ch] = _crop(np.fft.ifft2(acc), h, w)
    return out


# ---- loss.cpp -------------------------------------------------------------------------------
def make_depth_planes(count, d0, dz):        # :154-164
    if count < 1:
        raise ValueError("make_depth_planes: count must be >= 1")
    return [d0 + (l - (count - 1) * 0.5) * dz for l in range(count)]


def build_masks(depth, L, near_is_high=True):  # :166-180
    if L < 1:
        raise ValueError("build_masks: plane count must be >= 1")
    b = np.clip(np.floor(depth * L).astype(np.int64), 0, L - 1)
    plane = L - 1 - b if near_is_high else b
    return np.stack([(plane == l).astype(np.uint8) for l in range(L)])


def ssim_window():                           # :20-31
    d = np.arange(kSsimWin) - kSsimWin // 2
    g = np.exp(-d * d / (2.0 * kSsimSigma ** 2))
    return g / g.sum()


def _corr_valid(img, g):                     # window_mean :56-62 (corr_x :34-42, then corr_y :45-53)
    h, w = img.shape
    vw, vh = w - g.size + 1, h - g.size + 1
    tmp = sum(g[j] * img[:, j:j + vw] for j in range(g.size))
    return sum(g[i] * tmp[i:i + vh, :] for i in range(g.size))


def _spread(valid, h, w, g):                 # spread_t :66-83
    vh, vw = valid.shape
    tmp = np.zeros((h, vw))
    for i in range(g.size):
        tmp[i:i + vh, :] += g[i] * valid
    out = np.zeros((h, w))
    for j in range(g.size):
        out[:, j:j + vw] += g[j] * tmp
    return out


def ssim_channel(x, y, want_grad):           # :91-145
    h, w = x.shape
    if h < kSsimWin or w < kSsimWin:
        raise ValueError("ssim: image smaller than the 11x11 window")
    g = ssim_window()
    mu1, mu2 = _corr_valid(x, g), _corr_valid(y, g)
    exx, eyy, exy = _corr_valid(x * x, g), _corr_valid(y * y, g), _corr_valid(x * y, g)
    s12, s11, s22 = exy - mu1 * mu2, exx - mu1 * mu1, eyy - mu2 * mu2
    a1, a2 = 2.0 * mu1 * mu2 + kSsimC1, 2.0 * s12 + kSsimC2
    b1, b2 = mu1 * mu1 + mu2 * mu2 + kSsimC1, s11 + s22 + kSsimC2
    s = (a1 * a2) / (b1 * b2)
    grad = None
    if want_grad:
        g1 = (s / a1) * 2.0 * mu2 - (s / b1) * 2.0 * mu1 + (s / b2) * 2.0 * mu1 - (s / a2) * 2.0 * mu2
        g2, g3 = -s / b2, 2.0 * s / a2
        grad = _spread(g1, h, w, g) + 2.0 * x * _spread(g2, h, w, g) + y * _spread(g3, h, w, g)
    return float(s.sum()), s.size, grad


def _check_pair(recon, target, masks):       # check_pair :11-18
    if len(recon) == 0:
        raise ValueError("loss: no reconstruction planes")
    if len(recon) != masks.shape[0]:
        raise ValueError("loss: plane count does not match masks")
    for r in recon:
        if r.shape != target.shape:
            raise ValueError("loss: reconstruction shape mismatch")


def loss_recon_grad(recon, target, masks, L_norm=None, C_norm=None):  # :248-272
    _check_pair(recon, target, masks)
    L = len(recon) if L_norm is None else L_norm
    n = target.size if C_norm is None else target.size // target.shape[0] * C_norm  # channel shard: global C
    w = 2.0 / (n * L)
    k = 1.0 + masks[:, None, :, :].astype(np.float64) + target[None] ** 2
    d = recon - target[None]
    return float(np.sum(d * d * k) / (n * L)), w * d * k


def loss_mse_grad(recon, target, masks):     # loss.cpp:208-225
    _check_pair(recon, target, masks)
    L, n = len(recon), target.size
    d = recon - target[None]
    return float(np.sum(d * d) / (n * L)), (2.0 / (n * L)) * d


def loss_ssim_grad(recon, target, masks, L_norm=None, C_norm=None):  # loss.cpp:292-314
    _check_pair(recon, target, masks)
    total, count = 0.0, 0
    grads = np.zeros_like(recon)
    for l in range(recon.shape[0]):
        for ch in range(recon.shape[1]):
            s, cnt, gr = ssim_channel(recon[l, ch], target[ch], True)
            total += s
            count += cnt
            grads[l, ch] = gr
    if L_norm is not None:  # plane shard: global normaliser
        count = count // recon.shape[0] * L_norm
    if C_norm is not None:  # channel shard: global normaliser
        count = count // recon.shape[1] * C_norm
    return 1.0 - total / count, grads * (-1.0 / count), total


def training_loss_grad(recon, target, masks):  # loss.cpp:320-329
    lr, gr = loss_recon_grad(recon, target, masks)
    ls, gs, _ = loss_ssim_grad(recon, target, masks)
    return lr + kSsimWeight * ls, gr + kSsimWeight * gs


# ---- optimizer.cpp -----------------------------------------------------------------------------
def cosine_lr(step, total, lr_max, lr_min):  # :8-13
    if total <= 0 or step < 0 or step > total:
        raise ValueError("cosine_lr: step outside [0, total_steps]")
    return lr_min + 0.5 * (lr_max - lr_min) * (1.0 + math.cos(math.pi * step / total))


class Adan:                                  # :15-72 (step :48-72)
    def __init__(self, beta1=0.98, beta2=0.92, beta3=0.99, eps=1e-8):
        self.b = (beta1, beta2, beta3)
        self.eps = eps
        self.groups = {}

    def add_group(self, name, size, lr):
        if name in self.groups:
            raise ValueError("Adan: duplicate group " + name)
        self.groups[name] = dict(lr=lr, t=0, m=np.zeros(size), v=np.zeros(size), n=np.zeros(size),
                                 gp=np.zeros(size))

    def set_lr(self, name, lr):
        self.groups[name]["lr"] = lr

    def step(self, name, params, grads):
        if name not in self.groups:
            raise ValueError("Adan: unknown group " + name)
        g = self.groups[name]
        grads = np.asarray(grads, dtype=np.float64)
        if params.size != g["m"].size or grads.size != g["m"].size:
            raise ValueError("Adan: size mismatch for group " + name)
        if not np.all(np.isfinite(grads)):
            raise RuntimeError("Adan: non-finite gradient in group " + name)
        g["t"] += 1
        b1, b2, b3 = self.b
        bc1, bc2, bc3 = 1.0 - b1 ** g["t"], 1.0 - b2 ** g["t"], 1.0 - b3 ** g["t"]
        diff = np.zeros_like(grads) if g["t"] == 1 else grads - g["gp"]
        g["m"] = b1 * g["m"] + (1.0 - b1) * grads
        g["v"] = b2 * g["v"] + (1.0 - b2) * diff
        upd = grads + b2 * diff
        g["n"] = b3 * g["n"] + (1.0 - b3) * upd * upd
        denom = np.sqrt(g["n"] / bc3) + self.eps
        params -= g["lr"] * (g["m"] / bc1 + b2 * g["v"] / bc2) / denom
        g["gp"] = grads.copy()


GROUP_LRS = (("position", 1e-2), ("scale", 5e-3), ("rotation", 1e-3), ("amplitude", 2.5e-3),
             ("phase", 2.5e-3), ("opacity", 2.5e-2))   # pipeline.cpp:243-249


def step_grads(g, n, c, width, height, target, masks, distances, wavelengths, pitch=3.74e-6, pad=2,
               aperture=0.0, planes=None, L_norm=None, C_norm=None):
    """Forward + backward of pipeline.cpp:256-279 for the planes in `planes`
    (all by default).  With a plane subset and L_norm (or a channel slice of
    the scene and C_norm) the loss normalisers are the global ones, so summing
    the per-shard results gives the full step."""
    L = len(distances)
    sel = list(range(L)) if planes is None else list(planes)
    re, im = rasterize_forward(g, n, c, width, height)
    d_sel = [distances[l] for l in sel]
    U = propagate_multi(re + 1j * im, wavelengths, pitch, pad, aperture, d_sel)
    I = np.abs(U) ** 2
    m_sel = masks[sel]
    Lg = L if L_norm is None else L_norm
    lr, gr = loss_recon_grad(I, target, m_sel, Lg, C_norm)
    _, gs, ssum = loss_ssim_grad(I, target, m_sel, Lg, C_norm)
    gi = gr + kSsimWeight * gs
    du = 2.0 * U * gi
    back = propagate_multi_backward(du, wavelengths, pitch, pad, aperture, d_sel)
    grads = rasterize_backward(g, n, c, back.real, back.imag)
    Cg = c if C_norm is None else C_norm
    count = Lg * Cg * (height - 10) * (width - 10)
    return dict(recon_sum=lr * (target.size // c * Cg) * Lg, ssim_sum=ssum, count=count, grads=grads)
