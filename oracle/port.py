"""numpy restatement of fuzzdepth's depth hot path (TEST INFRASTRUCTURE).

Works on a stacked (n, m) member matrix (float32 or float64) and optional
float64 weights instead of Ensemble objects.  Each function cites the
reference lines whose arithmetic it reproduces; the chunking (65 536 cells,
ascending), float64 accumulation and tile order are kept so results agree
with the reference to the last few ulps (pinned in tests/test_oracle.py).
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

CHUNK = 65536              # reduction.py:22
TILE_BYTES = 32 * 2**20    # depth.py:36


def _spans(m: int):
    """Ascending [lo, hi) chunk bounds (reduction.py:30-33)."""
    return [(lo, min(lo + CHUNK, m)) for lo in range(0, m, CHUNK)]


def _pmap(fn, items, workers):
    """Order-preserving map over a thread pool (reduction.py:115-127)."""
    items = list(items)
    if workers <= 1 or len(items) <= 1:
        return [fn(x) for x in items]
    with ThreadPoolExecutor(max_workers=workers) as ex:
        return list(ex.map(fn, items))


def _workers(workers):
    return int(workers) if workers else (os.cpu_count() or 1)


def weighted_sum(v: np.ndarray, w: np.ndarray | None) -> float:
    """sum w*v, chunked float64 (reduction.py:36-44 / grid.py:242-244)."""
    total = 0.0
    for lo, hi in _spans(v.shape[0]):
        c = v[lo:hi].astype(np.float64, copy=False)
        if w is not None:
            c = c * w[lo:hi]
        total += float(np.sum(c))
    return total


def masses(U, w=None, workers=None) -> np.ndarray:
    """member_masses (depth.py:88-102)."""
    return np.array(_pmap(lambda i: weighted_sum(U[i], w), range(len(U)), _workers(workers)),
                    dtype=np.float64)


def inverse(m: np.ndarray) -> np.ndarray:
    """_inverse_masses (depth.py:164-168)."""
    inv = np.zeros_like(m)
    pos = m > 0.0
    inv[pos] = 1.0 / m[pos]
    return inv


def mass_cv(m: np.ndarray) -> float:
    """depth.py:105-110."""
    mu = float(np.mean(m))
    return 0.0 if mu == 0.0 else float(np.std(m) / mu)


def ranks(depth: np.ndarray) -> np.ndarray:
    """depth.py:80-85: stable descending order, ties by index."""
    order = np.argsort(-depth, kind="stable")
    r = np.empty(depth.shape[0], dtype=np.int64)
    r[order] = np.arange(depth.shape[0])
    return r


def mean_values(U) -> np.ndarray:
    """mean_mask (grid.py:251-261): sequential float64 member sum, / n."""
    acc = np.zeros(np.asarray(U[0]).shape[0], dtype=np.float64)
    for i in range(len(U)):
        acc += U[i]
    acc /= len(U)
    return acc


def gram(rows: np.ndarray, cols: np.ndarray, w=None, complement=False) -> np.ndarray:
    """gram_block (reduction.py:75-97): per chunk, float64 (w*rows) @ cols^T."""
    out = np.zeros((rows.shape[0], cols.shape[0]), dtype=np.float64)
    for lo, hi in _spans(rows.shape[1]):
        a = rows[:, lo:hi].astype(np.float64, copy=False)
        if w is not None:
            a = a * w[lo:hi]
        b = cols[:, lo:hi].astype(np.float64, copy=False)
        if complement:
            b = 1.0 - b
        out += a @ b.T
    return out


def _tile(m: int, n: int) -> int:
    """depth.py:113-115."""
    return max(1, min(n, TILE_BYTES // (4 * m)))


def pairwise_sums(U, w, inv, complement, workers=None):
    """_pairwise_sums (depth.py:122-161): tile pairs (upper triangle for the
    symmetric product), fixed-order accumulation of row sums and
    inverse-mass-weighted column sums."""
    n, m = len(U), np.asarray(U[0]).shape[0]
    t = _tile(m, n)
    tiles = [(lo, min(lo + t, n)) for lo in range(0, n, t)]
    if complement:
        pairs = [(a, b) for a in tiles for b in tiles]
    else:
        pairs = [(a, b) for k, a in enumerate(tiles) for b in tiles[k:]]

    def block(pair):
        (il, ih), (jl, jh) = pair
        rows = np.stack([U[i] for i in range(il, ih)])
        cols = rows if (il, ih) == (jl, jh) else np.stack([U[j] for j in range(jl, jh)])
        return gram(rows, cols, w, complement)

    row = np.zeros(n)
    col = np.zeros(n)
    for ((il, ih), (jl, jh)), g in zip(pairs, _pmap(block, pairs, _workers(workers))):
        row[il:ih] += g.sum(axis=1)
        col[jl:jh] += inv[il:ih] @ g
        if not complement and (il, ih) != (jl, jh):
            row[jl:jh] += g.sum(axis=0)
            col[il:ih] += g @ inv[jl:jh]
    return row, col


def depth_pid(U, w=None, workers=None):
    """depth_pid (depth.py:213-228) -> dict of in_in, in_out, depth, rank, cv."""
    n = len(U)
    m_ = masses(U, w, workers)
    inv = inverse(m_)
    row, col = pairwise_sums(U, w, inv, False, workers)
    return _pack(inv * row / n, col / n, m_)


def depth_eid(U, w=None, workers=None):
    """depth_eid (depth.py:192-210) on 0/1 members."""
    n = len(U)
    m_ = masses(U, w, workers)
    inv = inverse(m_)
    row_x, col_inv = pairwise_sums(U, w, inv, True, workers)
    pos = m_ > 0.0
    n_pos = float(np.count_nonzero(pos))
    in_in = np.zeros(n)
    in_in[pos] = (n - inv[pos] * row_x[pos]) / n
    return _pack(in_in, (n_pos - col_inv) / n, m_)


def member_mean_terms(v, mean64, w):
    """_member_mean_terms (depth.py:231-243)."""
    num = 0.0
    mass = 0.0
    for lo, hi in _spans(v.shape[0]):
        c = v[lo:hi].astype(np.float64, copy=False)
        if w is not None:
            c = c * w[lo:hi]
        num += float(np.sum(c * mean64[lo:hi]))
        mass += float(np.sum(c))
    return num, mass


def depth_pid_mean(U, w=None, workers=None):
    """depth_pid_mean (depth.py:246-287); raises ValueError on a zero mean."""
    mean = mean_values(U)
    mean_mass = weighted_sum(mean, w)
    if mean_mass == 0.0:
        raise ValueError("ensemble mean mask is identically zero")
    terms = _pmap(lambda i: member_mean_terms(U[i], mean, w), range(len(U)), _workers(workers))
    num = np.array([t[0] for t in terms])
    m_ = np.array([t[1] for t in terms])
    inv = inverse(m_)
    return _pack(num * inv, num / mean_mass, m_)


def _pack(in_in, in_out, m_):
    depth = np.minimum(in_in, in_out)
    return {"in_in": in_in, "in_out": in_out, "depth": depth, "rank": ranks(depth),
            "cv": mass_cv(m_), "mass": m_}


def prob_inclusion(u, v, w=None) -> float:
    """inclusion.py:22-40."""
    num = den = 0.0
    for lo, hi in _spans(u.shape[0]):
        c = u[lo:hi].astype(np.float64, copy=False)
        if w is not None:
            c = c * w[lo:hi]
        num += float(np.sum(c * v[lo:hi]))
        den += float(np.sum(c))
    return 0.0 if den == 0.0 else num / den


def subset_epsilon(a, b, w=None) -> float:
    """inclusion.py:43-64 on boolean arrays."""
    excess = mass = 0.0
    for lo, hi in _spans(a.shape[0]):
        ac = a[lo:hi].astype(bool)
        out = ac & ~b[lo:hi].astype(bool)
        if w is not None:
            excess += float(np.sum(w[lo:hi] * out))
            mass += float(np.sum(w[lo:hi] * ac))
        else:
            excess += float(np.count_nonzero(out))
            mass += float(np.count_nonzero(ac))
    return 0.0 if mass == 0.0 else 1.0 - excess / mass


def min_max_terms(u, v, w=None):
    """_min_max_terms (inclusion.py:67-88)."""
    s_min = s_max = s_u = s_v = 0.0
    for lo, hi in _spans(u.shape[0]):
        uc = u[lo:hi].astype(np.float64, copy=False)
        vc = v[lo:hi].astype(np.float64, copy=False)
        lo_uv, hi_uv = np.minimum(uc, vc), np.maximum(uc, vc)
        if w is not None:
            wc = w[lo:hi]
            lo_uv, hi_uv, uc, vc = wc * lo_uv, wc * hi_uv, wc * uc, wc * vc
        s_min += float(np.sum(lo_uv))
        s_max += float(np.sum(hi_uv))
        s_u += float(np.sum(uc))
        s_v += float(np.sum(vc))
    return s_min, s_max, s_u, s_v


def fuzzy_dice(u, v, w=None) -> float:
    """inclusion.py:91-96; ValueError for two zero-mass masks."""
    s_min, _, s_u, s_v = min_max_terms(u, v, w)
    if s_u + s_v == 0.0:
        raise ValueError("fuzzy_dice is undefined for two zero-mass masks")
    return 2.0 * s_min / (s_u + s_v)


def prob_iou(u, v, w=None) -> float:
    """inclusion.py:99-107; ValueError for two zero-mass masks."""
    s_min, s_max, _, _ = min_max_terms(u, v, w)
    if s_max == 0.0:
        raise ValueError("prob_iou is undefined for two zero-mass masks")
    return s_min / s_max


def depth_similarity(U, measure, w=None, workers=None):
    """depth_similarity_baseline (depth.py:298-325): similarity to the mean mask."""
    fn = {"dice": fuzzy_dice, "fuzzy-dice": fuzzy_dice, "iou": prob_iou, "prob-iou": prob_iou}[measure]
    mean = mean_values(U)
    if weighted_sum(mean, w) == 0.0:
        raise ValueError("ensemble mean mask is identically zero")
    m_ = masses(U, w, workers)
    d = np.array(_pmap(lambda i: fn(U[i], mean, w), range(len(U)), _workers(workers)))
    return _pack(d, d.copy(), m_)
