"""Pairwise operators on the GPU (K8): probabilistic inclusion, the binary
epsilon-subset and the symmetric Dice / IoU similarities,
/root/reference/pkg/src/fuzzdepth/inclusion.py:22-107.

Both take one fused pass over the cells (numerator and denominator together)
with fp64 accumulation, like the reference.  Inputs are the reference's mask
objects (or this package's mirrors); device tensors of shape (cells,) are
accepted too.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .device import require_cuda, stream_ptr
from .errors import ValidationError


def _dev_values(x, dev, dtype=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.reshape(-1)
    else:
        t = torch.from_numpy(np.array(np.asarray(x).reshape(-1)))  # writable copy
    if dtype is not None:
        t = t.to(dtype)
    elif t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float32)
    return t.to(dev).contiguous()


def _pair(u_vals, v_vals, weights, op: int) -> tuple[float, ...]:
    dev = require_cuda()
    dt = torch.float64 if (getattr(u_vals, "dtype", None) in (np.float64, torch.float64) or
                           getattr(v_vals, "dtype", None) in (np.float64, torch.float64)) else torch.float32
    u = _dev_values(u_vals, dev, dt)
    v = _dev_values(v_vals, dev, dt)
    w = None if weights is None else _dev_values(np.asarray(weights, dtype=np.float64), dev, torch.float64)
    m = u.numel()
    # a private ~20 KB workspace per call from the stream-aware caching
    # allocator: concurrent callers (any thread, same stream) never share the
    # partials buffer; the call synchronises before the block is released
    ws = torch.empty(8192 * 8, dtype=torch.uint8, device=dev)
    out = np.zeros(4, dtype=np.float64)
    N.call("pidb_pair_sums", u.data_ptr(), v.data_ptr(),
           N.PIDB_F64 if dt == torch.float64 else N.PIDB_F32, m,
           None if w is None else w.data_ptr(), int(op),
           out.ctypes.data, ws.data_ptr(), ws.numel(), stream_ptr(dev))
    return tuple(float(x) for x in out[:4 if op == N.PIDB_OP_MINMAX else 2])


def prob_inclusion(u, v) -> float:
    """(sum w u v) / (sum w u); 0 when u has zero mass (inclusion.py:22-40)."""
    u.grid.require_same(v.grid)
    num, den = _pair(u.values, v.values, u.grid.weights, N.PIDB_OP_INCLUSION)
    if den == 0.0:
        return 0.0
    return num / den


def subset_epsilon(a, b) -> float:
    """1 - |A \\ B| / |A|; 0 when |A| = 0 (inclusion.py:43-64)."""
    a.grid.require_same(b.grid)
    av = np.asarray(a.bits, dtype=np.float32)
    bv = np.asarray(b.bits, dtype=np.float32)
    excess, mass = _pair(av, bv, a.grid.weights, N.PIDB_OP_SUBSET)
    if mass == 0.0:
        return 0.0
    return 1.0 - excess / mass


def _min_max_terms(u, v) -> tuple[float, float, float, float]:
    """Fused sums of w*min(u,v), w*max(u,v), w*u, w*v (inclusion.py:67-88)."""
    u.grid.require_same(v.grid)
    return _pair(u.values, v.values, u.grid.weights, N.PIDB_OP_MINMAX)


def fuzzy_dice(u, v) -> float:
    """2 sum(w min(u,v)) / (sum(w u) + sum(w v)) (inclusion.py:91-96)."""
    s_min, _, s_u, s_v = _min_max_terms(u, v)
    if s_u + s_v == 0.0:
        raise ValidationError("fuzzy_dice is undefined for two zero-mass masks")
    return 2.0 * s_min / (s_u + s_v)


def prob_iou(u, v) -> float:
    """sum(w min(u,v)) / sum(w max(u,v)) (inclusion.py:99-107)."""
    s_min, s_max, _, _ = _min_max_terms(u, v)
    if s_max == 0.0:
        raise ValidationError("prob_iou is undefined for two zero-mass masks")
    return s_min / s_max
