"""Randomised parity sweep of every streaming-kernel variant against the CPU
oracle: python tools/fuzz_parity.py SECONDS [seed]
(n log-uniform in 1..6000, cells log-uniform, fp32/fp64, weighted or not,
PID-mean / PID / dice / IoU / masses, binary eID, and -- round 2 -- the
tensor-core PID (K1x + certifier: depths within 1e-8, ranks equal), the
fp64 gram_block seam (rtol 1e-12) and, for pinned host inputs, the streamed
PID-mean, and binary eID on byte ensembles; depths within 1e-11, ranks
equal wherever the oracle's depth gaps exceed 1e-11)."""
import sys
import time
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_15187_b200 as pb  # noqa: E402
from oracle import exact, port  # noqa: E402

warnings.simplefilter("ignore", RuntimeWarning)  # the CV warning of skewed random draws
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
t_end = time.time() + budget
cases = fails = 0


def ranks_ok(got, want_depth, want_rank):
    if np.array_equal(got, want_rank):
        return True
    d = np.sort(want_depth)
    return np.min(np.diff(d)) < 1e-11 if d.size > 1 else False


while time.time() < t_end:
    n = int(np.exp(rng.uniform(0, np.log(6000))))
    m = int(np.exp(rng.uniform(0, np.log(min(200000, 4e7 / n)))))
    f64 = rng.uniform() < 0.25
    weighted = rng.uniform() < 0.4
    binary = rng.uniform() < 0.2
    U = rng.uniform(size=(n, m))
    if binary:
        U = (U < rng.uniform(0.2, 0.8)).astype(np.float64)
    U = U.astype(np.float64 if f64 else np.float32)
    w = rng.uniform(0.5, 2.0, size=m) if weighted else None
    de = pb.DeviceEnsemble.from_tensor(torch.from_numpy(U), w)
    checks = []
    try:
        if U.sum() > 0:
            r, ref = pb.depth_pid_mean(de), port.depth_pid_mean(U, w, workers=8)
            checks.append(("pid-mean", r, ref))
            for meas in ("dice", "iou"):
                checks.append((meas, pb.depth_similarity_baseline(de, meas),
                               port.depth_similarity(U, meas, w, workers=8)))
        if n * n * m <= 4e10:
            ref_pid = port.depth_pid(U, w, workers=8)
            checks.append(("pid", pb.depth_pid(de), ref_pid))
            if U.sum() > 0 and n <= 3000:
                g = pb.depth_pid(de, algorithm="gram")
                gerr = float(np.max(np.abs(g.depth - ref_pid["depth"])))
                if gerr > 1e-8 or not ranks_ok(g.rank, ref_pid["depth"], ref_pid["rank"]):
                    print(f"FAIL pid-gram n={n} m={m} f64={f64} w={weighted} err={gerr:.2e}",
                          flush=True)
                    fails += 1
        if rng.uniform() < 0.1 and n * m <= 4e6:
            from paper_2512_15187_b200.reduction import gram_block

            k = max(1, n // 2)
            got = gram_block(U[:k], U[k:] if n > 1 else U, w, complement_cols=binary)
            A = U[:k].astype(np.float64) * (1.0 if w is None else w)
            B = (U[k:] if n > 1 else U).astype(np.float64)
            want = A @ (1.0 - B if binary else B).T
            if not np.allclose(got, want, rtol=1e-12, atol=1e-300):
                print(f"FAIL gram_block n={n} m={m} f64={f64} w={weighted}", flush=True)
                fails += 1
        if not weighted and U.sum() > 0 and rng.uniform() < 0.15 and n * m * U.itemsize > 1 << 16:
            from paper_2512_15187_b200 import depth as D

            old = D.STREAM_SLAB_BYTES
            D.STREAM_SLAB_BYTES = max(4096, n * m * U.itemsize // int(rng.integers(3, 9)))
            try:
                r = pb.depth_pid_mean(torch.from_numpy(U).pin_memory())
            finally:
                D.STREAM_SLAB_BYTES = old
            checks.append(("pid-mean-streamed", r, port.depth_pid_mean(U, w, workers=8)))
        mass = pb.member_masses(de)
        ok = np.allclose(mass, port.masses(U, w), rtol=1e-12, atol=1e-9)
        if not ok:
            print(f"FAIL masses n={n} m={m} f64={f64} w={weighted}", flush=True)
            fails += 1
        if binary and not weighted and n * n * m <= 4e10:
            a, b, c, _ = exact.eid_fast(U.astype(np.float32))
            r = pb.depth_eid(de)
            if not (np.array_equal(r.depth, c) and np.array_equal(r.rank, exact.ranks(c))):
                print(f"FAIL eid n={n} m={m}", flush=True)
                fails += 1
            # the same members as a byte ensemble (K2 straight from the bytes)
            rb = pb.depth_eid(U != 0 if rng.uniform() < 0.5 else (U != 0).astype(np.uint8))
            if not (np.array_equal(rb.depth, c) and np.array_equal(rb.rank, r.rank)):
                print(f"FAIL eid-bytes n={n} m={m}", flush=True)
                fails += 1
        for name, r, ref in checks:
            err = float(np.max(np.abs(r.depth - ref["depth"]))) if n else 0.0
            if err > 1e-11 or not ranks_ok(r.rank, ref["depth"], ref["rank"]):
                print(f"FAIL {name} n={n} m={m} f64={f64} w={weighted} bin={binary} err={err:.2e}",
                      flush=True)
                fails += 1
    except Exception as exc:  # report and continue
        print(f"ERROR n={n} m={m} f64={f64} w={weighted}: {type(exc).__name__}: {exc}", flush=True)
        fails += 1
    cases += 1
    del de
print(f"fuzz_parity: {cases} cases, {fails} failures", flush=True)
sys.exit(1 if fails else 0)
