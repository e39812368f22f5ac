"""Exact-summation oracle (TEST INFRASTRUCTURE).

Restates the reference test oracle /root/reference/pkg/tests/reference_impl.py
(every sum through math.fsum, i.e. exactly rounded) and adds ``eid_fast``:
the same ref_eid values computed from exact integer intersection counts, which
makes bit-exact eID checks feasible at the BASELINE sizes (500 x 512^2).
"""
from __future__ import annotations

import math

import numpy as np


def inclusion(u, v, w) -> float:
    """reference_impl.py:14-28."""
    u = np.asarray(u, dtype=np.float64).ravel()
    v = np.asarray(v, dtype=np.float64).ravel()
    w = np.asarray(w, dtype=np.float64).ravel()
    den = math.fsum((w * u).tolist())
    return 0.0 if den == 0.0 else math.fsum(((w * u) * v).tolist()) / den


def subset_eps(a, b, w) -> float:
    """reference_impl.py:31-40."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    w = np.asarray(w, dtype=np.float64).ravel()
    inside = a > 0
    mass = math.fsum(w[inside].tolist())
    if mass == 0.0:
        return 0.0
    return 1.0 - math.fsum(w[inside & (b == 0)].tolist()) / mass


def _pairwise(members, w, op):
    n = len(members)
    in_in, in_out = [], []
    for i in range(n):
        in_in.append(math.fsum(op(members[i], members[j], w) for j in range(n)) / n)
        in_out.append(math.fsum(op(members[j], members[i], w) for j in range(n)) / n)
    depth = [min(a, b) for a, b in zip(in_in, in_out)]
    return np.array(in_in), np.array(in_out), np.array(depth)


def pid(members, w):
    """reference_impl.py:47-57."""
    return _pairwise(members, w, inclusion)


def eid(members, w):
    """reference_impl.py:60-70."""
    return _pairwise(members, w, subset_eps)


def pid_mean(members, w):
    """reference_impl.py:73-81 (mean per cell via fsum / n)."""
    n = len(members)
    stack = np.stack([np.asarray(m, dtype=np.float64).ravel() for m in members])
    mean = np.array([math.fsum(stack[:, c].tolist()) / n for c in range(stack.shape[1])])
    in_in = np.array([inclusion(m, mean, w) for m in stack])
    in_out = np.array([inclusion(mean, m, w) for m in stack])
    return in_in, in_out, np.minimum(in_in, in_out)


def ranks(depth):
    """reference_impl.py:84-90."""
    order = sorted(range(len(depth)), key=lambda i: (-depth[i], i))
    r = [0] * len(depth)
    for k, i in enumerate(order):
        r[i] = k
    return np.array(r, dtype=np.int64)


def intersections(B: np.ndarray, chunk: int = 1 << 24) -> np.ndarray:
    """Exact |C_i ∩ C_j| for 0/1 rows: float32 BLAS over column chunks of at
    most 2^24 cells is exact (0/1 products, partial counts < 2^24), and the
    chunk counts are summed as int64."""
    B = np.asarray(B)
    n, m = B.shape
    I = np.zeros((n, n), dtype=np.int64)
    for lo in range(0, m, chunk):
        X = np.asarray(B[:, lo:lo + chunk], dtype=np.float32)
        I += np.rint(X @ X.T).astype(np.int64)
    return I


def eid_fast(B: np.ndarray):
    """ref_eid with unit weights from exact counts: per-pair IEEE terms
    1.0 - (m_i - I_ij) / m_i (reference_impl.py:36-40), fsum over j, / n."""
    I = intersections(B)
    n = I.shape[0]
    mass = np.diag(I).astype(np.float64)
    excess = mass[:, None] - I.astype(np.float64)      # (i, j): |A_i \ A_j|
    with np.errstate(divide="ignore", invalid="ignore"):
        T = 1.0 - excess / mass[:, None]
    T[mass == 0.0, :] = 0.0
    in_in = np.array([math.fsum(T[i].tolist()) / n for i in range(n)])
    in_out = np.array([math.fsum(T[:, i].tolist()) / n for i in range(n)])
    return in_in, in_out, np.minimum(in_in, in_out), I
