"""Synthetic ensembles for benchmarks and GPU tests (not the product path).

Per-member shape parameters are drawn on the host exactly like the reference
generators (/root/reference/pkg/src/fuzzdepth/synth.py:20-210: one Philox
stream per (seed, member)); the voxel fields of fuzzy disks / ellipsoids are
then evaluated on the GPU (libpidb ``pidb_synth_*``) straight into the
(n, ld) device layout — the 107 GB 200 x 512^3 ensemble is never built on the
host.  The binary Fourier contours are built on the host (as the reference
does) and uploaded.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .device import DeviceEnsemble, padded_ld, require_cuda, shard_bounds, stream_ptr
from .errors import ValidationError
from .grid import GridSpec, ProbMask


def member_rng(seed: int, index: int) -> np.random.Generator:
    """synth.py:20-22."""
    return np.random.Generator(np.random.Philox(key=[np.uint64(seed), np.uint64(index)]))


def ellipsoid_params(res, n_base, n_outliers, seed, *, axes_fractions=(0.30, 0.25, 0.20),
                     axis_jitter_sd=0.10, center_sd_fraction=0.01, falloff_fraction=0.02,
                     outlier_scales=(1.0,), outlier_offset_fraction=0.25):
    """Per-member (center, axes) of gen_ellipsoid_ensemble (synth.py:84-135)."""
    base_axes = np.array(axes_fractions, dtype=np.float64) * res
    grid_center = np.full(3, (res - 1) / 2.0)
    n = n_base + n_outliers
    prm = np.empty((n, 6), dtype=np.float64)
    ids = []
    for i in range(n):
        rng = member_rng(seed, i)
        out = i >= n_base
        axes = base_axes * rng.normal(1.0, axis_jitter_sd, size=3)
        center = grid_center + rng.normal(0.0, center_sd_fraction * res, size=3)
        if out:
            axes = axes * outlier_scales[int(rng.integers(len(outlier_scales)))]
            axis = int(rng.integers(3))
            sign = 1.0 if rng.integers(2) else -1.0
            center = center.copy()
            center[axis] += sign * outlier_offset_fraction * res
        prm[i, :3] = center
        prm[i, 3:] = axes
        ids.append(f"outlier_{i - n_base:04d}" if out else f"base_{i:04d}")
    return prm, falloff_fraction * res, ids


def disk_params(res, n, seed, *, radius_fraction=0.30, radius_sd=0.05,
                center_sd_fraction=0.01, sigma2=0.8):
    """Per-member (cy, cx, radius) of gen_disk_ensemble (synth.py:54-81)."""
    base = (res - 1) / 2.0
    prm = np.empty((n, 3), dtype=np.float64)
    for i in range(n):
        rng = member_rng(seed, i)
        radius = radius_fraction * res * rng.normal(1.0, radius_sd)
        cy, cx = np.array([base, base]) + rng.normal(0.0, center_sd_fraction * res, size=2)
        prm[i] = (cy, cx, max(radius, 1.0))
    return prm, sigma2, [f"disk_{i:04d}" for i in range(n)]


def contour_masks(n, res, seed, *, radius_fraction=0.35, amplitude_fraction=0.03, orders=5,
                  outlier_prob=0.2, outlier_amp_factor=3.0) -> np.ndarray:
    """Binary Fourier contours of gen_contour_ensemble_2d (synth.py:165-210) as
    an (n, res*res) float32 array."""
    yy, xx = np.ogrid[0:res, 0:res]
    c = (res - 1) / 2.0
    r = np.sqrt((yy - c) ** 2 + (xx - c) ** 2)
    theta = np.arctan2(xx - c, yy - c)
    cos_k = [np.cos(k * theta) for k in range(1, orders + 1)]
    sin_k = [np.sin(k * theta) for k in range(1, orders + 1)]
    out = np.empty((n, res * res), dtype=np.float32)
    for i in range(n):
        rng = member_rng(seed, i)
        is_out = rng.uniform() < outlier_prob
        ac = rng.normal(0.0, amplitude_fraction * res, size=orders)
        as_ = rng.normal(0.0, amplitude_fraction * res, size=orders)
        if is_out:
            ac = ac * outlier_amp_factor
            as_ = as_ * outlier_amp_factor
        radius = np.full((res, res), radius_fraction * res)
        for k in range(orders):
            radius = radius + ac[k] * cos_k[k]
            radius = radius + as_[k] * sin_k[k]
        np.maximum(radius, 0.02 * res, out=radius)
        out[i] = (r <= radius).reshape(-1)
    return out


def ellipsoids_device(res, n_base, n_outliers=0, seed=0, device=None,
                      shard: tuple[int, int] | None = None, process_group=None) -> DeviceEnsemble:
    """Fuzzy ellipsoid ensemble generated directly in HBM (optionally only
    this rank's cell slab)."""
    dev = require_cuda(device)
    prm, sigma, ids = ellipsoid_params(res, n_base, n_outliers, seed)
    n = prm.shape[0]
    m_full = res ** 3
    lo, hi = (0, m_full) if shard is None else shard_bounds(m_full, *shard)
    p = torch.from_numpy(prm).to(dev)
    if lo == 0 and hi == m_full:
        ld = padded_ld(m_full)
        out = torch.empty((n, ld), dtype=torch.float32, device=dev)
        N.call("pidb_synth_ellipsoids", out.data_ptr(), n, res, ld, p.data_ptr(), sigma,
               stream_ptr(dev))
    else:  # generate full rows in blocks and keep the slab
        ld = padded_ld(hi - lo)
        out = torch.zeros((n, ld), dtype=torch.float32, device=dev)
        ldf = padded_ld(m_full)
        blk = max(1, int((2 << 30) // (ldf * 4)))
        tmp = torch.empty((min(blk, n), ldf), dtype=torch.float32, device=dev)
        for i0 in range(0, n, blk):
            k = min(blk, n - i0)
            N.call("pidb_synth_ellipsoids", tmp.data_ptr(), k, res, ldf,
                   p[i0:i0 + k].contiguous().data_ptr(), sigma, stream_ptr(dev))
            out[i0:i0 + k, :hi - lo].copy_(tmp[:k, lo:hi])
        del tmp
    return DeviceEnsemble(out, hi - lo, (res, res, res), tuple(ids),
                          process_group=process_group if shard is not None else None,
                          cell_range=(lo, hi))


def disks_device(res, n, seed=0, device=None) -> DeviceEnsemble:
    dev = require_cuda(device)
    prm, sigma2, ids = disk_params(res, n, seed)
    ld = padded_ld(res * res)
    out = torch.empty((n, ld), dtype=torch.float32, device=dev)
    p = torch.from_numpy(prm).to(dev)
    N.call("pidb_synth_disks", out.data_ptr(), n, res, ld, p.data_ptr(), sigma2, stream_ptr(dev))
    return DeviceEnsemble(out, res * res, (res, res), tuple(ids), cell_range=(0, res * res))


def contours_device(n, res, seed=0, device=None) -> DeviceEnsemble:
    masks = contour_masks(n, res, seed)
    return DeviceEnsemble.from_tensor(torch.from_numpy(masks), ids=[f"contour_{i:04d}" for i in range(n)],
                                      dims=(res, res), validate=False, device=device)


# ------------------------------------------------- the reference's names


def gen_fuzzy_disk(grid2d: GridSpec, center, radius: float, sigma2: float) -> ProbMask:
    """One fuzzy disk mask (synth.py:30-51): 1 inside, Gaussian falloff
    exp(-(dist - radius)^2 / (2 sigma2)) outside (host, float64 -> float32)."""
    if len(grid2d.dims) != 2:
        raise ValidationError("gen_fuzzy_disk needs a 2D grid")
    if not radius > 0.0 or not sigma2 > 0.0:
        raise ValidationError("radius and sigma2 must be positive")
    yy, xx = np.meshgrid(*(np.arange(d, dtype=np.float64) for d in grid2d.dims), indexing="ij")
    dist = np.sqrt((yy - center[0]) ** 2 + (xx - center[1]) ** 2)
    u = np.where(dist <= radius, 1.0, np.exp(-((dist - radius) ** 2) / (2.0 * sigma2)))
    return ProbMask(grid2d, u.astype(np.float32))


def gen_disk_ensemble(res: int, n: int, seed: int, device=None, **kw) -> DeviceEnsemble:
    """gen_disk_ensemble (synth.py:54-81), generated in HBM."""
    if res < 8 or n < 1:
        raise ValidationError("need res >= 8 and n >= 1")
    if kw:
        raise ValidationError(f"unsupported generator options {sorted(kw)}")
    return disks_device(res, n, seed, device=device)


def gen_ellipsoid_ensemble(res: int, n_base: int, n_outliers: int, seed: int, device=None,
                           **kw) -> DeviceEnsemble:
    """gen_ellipsoid_ensemble (synth.py:84-135), generated in HBM."""
    if res < 8:
        raise ValidationError("need res >= 8")
    if n_base < 0 or n_outliers < 0 or n_base + n_outliers < 1:
        raise ValidationError("need n_base, n_outliers >= 0 and at least one member")
    if kw:
        raise ValidationError(f"unsupported generator options {sorted(kw)}")
    return ellipsoids_device(res, n_base, n_outliers, seed, device=device)


def gen_contour_ensemble_2d(n: int, res: int, seed: int, device=None, **kw) -> DeviceEnsemble:
    """gen_contour_ensemble_2d (synth.py:165-210): binary Fourier contours."""
    if n < 1 or res < 8:
        raise ValidationError("need n >= 1 and res >= 8")
    masks = contour_masks(n, res, seed, **kw)
    return DeviceEnsemble.from_tensor(torch.from_numpy(masks),
                                      ids=[f"contour_{i:04d}" for i in range(n)],
                                      dims=(res, res), validate=False, device=device)
