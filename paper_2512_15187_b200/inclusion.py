"""Pairwise operators on the GPU (K8): probabilistic inclusion and the binary
epsilon-subset, /root/reference/pkg/src/fuzzdepth/inclusion.py:22-64.

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

_WS: dict = {}


def _dev_values(x, dev, dtype=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.reshape(-1)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x).reshape(-1)))
    if dtype is not None:
        t = t.to(dtype)
    elif t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float32)
    return t.to(dev).contiguous()


def _pair(u_vals, v_vals, weights, complement: bool) -> tuple[float, float]:
    dev = require_cuda()
    dt = torch.float64 if (getattr(u_vals, "dtype", None) in (np.float64, torch.float64) or
                           getattr(v_vals, "dtype", None) in (np.float64, torch.float64)) else torch.float32
    u = _dev_values(u_vals, dev, dt)
    v = _dev_values(v_vals, dev, dt)
    w = None if weights is None else _dev_values(np.asarray(weights, dtype=np.float64), dev, torch.float64)
    m = u.numel()
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    ws = _WS.get(key)
    if ws is None:
        ws = _WS[key] = torch.empty(8192 * 8, dtype=torch.uint8, device=dev)
    out = np.zeros(2, dtype=np.float64)
    N.call("pidb_pair_sums", u.data_ptr(), v.data_ptr(),
           N.PIDB_F64 if dt == torch.float64 else N.PIDB_F32, m,
           None if w is None else w.data_ptr(), int(complement),
           out.ctypes.data, ws.data_ptr(), ws.numel(), stream_ptr(dev))
    return float(out[0]), float(out[1])


def prob_inclusion(u, v) -> float:
    """(sum w u v) / (sum w u); 0 when u has zero mass (inclusion.py:22-40)."""
    u.grid.require_same(v.grid)
    num, den = _pair(u.values, v.values, u.grid.weights, complement=False)
    if den == 0.0:
        return 0.0
    return num / den


def subset_epsilon(a, b) -> float:
    """1 - |A \\ B| / |A|; 0 when |A| = 0 (inclusion.py:43-64)."""
    a.grid.require_same(b.grid)
    av = np.asarray(a.bits, dtype=np.float32)
    bv = np.asarray(b.bits, dtype=np.float32)
    excess, mass = _pair(av, bv, a.grid.weights, complement=True)
    if mass == 0.0:
        return 0.0
    return 1.0 - excess / mass
