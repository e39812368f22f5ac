"""Emulation of the K1x fixed-point Gram before it was built (numpy, CPU):
depth error of PID from the digit-level Gram (levels <= L of q = rint(u 2^31)
in base-256 digits) against the exact fp64 Gram, on ellipsoid (reference
generator), uniform and u^8 members.  Needs the reference importable
(baseline/_ref).  python tools/fixed_gram_emulation.py
Result recorded in csrc/gram_fixed.cu: levels <= 3 (10 digit pairs) ->
depth error <= 3.2e-9, 0 rank swaps; levels <= 4 -> ~1e-11."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
import numpy as np  # noqa: E402

import fuzzdepth as fd  # noqa: E402


def digits(U):
    q = np.rint(U.astype(np.float64) * 2.0 ** 31).astype(np.int64)
    return [((q >> (8 * (3 - k))) & 255).astype(np.float64) for k in range(4)]


def gram_fx(U, maxlevel):
    D = digits(U)
    G = np.zeros((U.shape[0],) * 2)
    for s in range(maxlevel + 1):
        L = np.zeros_like(G)
        for k in range(4):
            if 0 <= s - k < 4:
                L += D[k] @ D[s - k].T
        G += L * 2.0 ** (8 * (6 - s)) / 2.0 ** 62
    return G


def depth_from_gram(G, m):
    n = len(m)
    inv = np.where(m > 0, 1 / m, 0)
    return np.minimum(inv * G.sum(1) / n, (inv @ G) / n)


e = fd.gen_ellipsoid_ensemble(32, 300, 0, 3)
rng = np.random.default_rng(0)
for name, U in (("ellipsoids", np.stack([e.member(i).values for i in range(len(e))]).astype(np.float32)),
                ("uniform", rng.uniform(size=(300, 32768)).astype(np.float32)),
                ("u^8", (rng.uniform(size=(300, 32768)) ** 8).astype(np.float32))):
    X = U.astype(np.float64)
    G, m = X @ X.T, X.sum(1)
    d = depth_from_gram(G, m)
    for lv in (1, 2, 3, 4):
        df = depth_from_gram(gram_fx(U, lv), m)
        swaps = int((np.argsort(-df, kind="stable") != np.argsort(-d, kind="stable")).sum())
        print(f"{name}: levels <= {lv}: max depth err {np.abs(df - d).max():.2e}, "
              f"min gap {np.min(np.diff(np.sort(d))):.2e}, rank mismatches {swaps}")
