"""Generate the golden parity fixtures from the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports fuzzdepth from /root/reference/pkg/src and the reference test
oracle from /root/reference/pkg/tests/reference_impl.py, draws seeded
ensembles with the same recipes as the reference fixtures
(/root/reference/pkg/tests/conftest.py:20-42) and generators
(/root/reference/pkg/src/fuzzdepth/synth.py), and stores inputs and outputs
as compressed .npz files next to this script.  The GPU box never needs
/root/reference: the tests read these files only.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

import fuzzdepth as fd  # noqa: E402
from reference_impl import ref_eid, ref_pid, ref_pid_mean  # noqa: E402


def fuzzy(seed, n, dims, weighted):
    """Same draws as conftest.make_fuzzy_ensemble (conftest.py:20-29)."""
    rng = np.random.default_rng(seed)
    cells = int(np.prod(dims))
    w = rng.uniform(0.5, 2.0, size=cells) if weighted else None
    U = np.stack([rng.uniform(0.0, 1.0, size=cells).astype(np.float32) for _ in range(n)])
    return U, w


def binary(seed, n, dims, weighted):
    """Same draws as conftest.make_binary_ensemble (conftest.py:32-42)."""
    rng = np.random.default_rng(seed)
    cells = int(np.prod(dims))
    w = rng.uniform(0.5, 2.0, size=cells) if weighted else None
    rows = []
    for _ in range(n):
        density = rng.uniform(0.2, 0.8)
        rows.append((rng.uniform(0.0, 1.0, size=cells) < density).astype(np.float32))
    return np.stack(rows), w


def ensemble(U, w, dims):
    g = fd.GridSpec(tuple(dims), w)
    return fd.Ensemble(g, [fd.ProbMask(g, u) for u in U])


def result_arrays(prefix, r):
    return {
        f"{prefix}_in_in": r.in_in,
        f"{prefix}_in_out": r.in_out,
        f"{prefix}_depth": r.depth,
        f"{prefix}_rank": r.rank,
        f"{prefix}_cv": np.array(r.cv_mass),
    }


CMP_KEYS = ("max_abs_error", "mean_abs_error", "rank_pearson", "rank_kendall", "cv_mass")


def save(name, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(name, {k: v.shape for k, v in arrays.items()})


def main():
    import warnings

    warnings.simplefilter("ignore", RuntimeWarning)
    fuzzy_cases = [
        (11, 7, (4, 5), False), (11, 7, (4, 5), True), (21, 6, (3, 7), True),
        (3, 9, (6, 7), True), (5, 10, (9, 8), True),
        (0, 9, (4, 4, 4), False), (1, 9, (4, 4, 4), True),
        (77, 24, (17, 13, 7), True), (1, 20, (48, 48), False), (2, 12, (20, 20, 20), True),
    ]
    for k, (seed, n, dims, weighted) in enumerate(fuzzy_cases):
        U, w = fuzzy(seed, n, dims, weighted)
        e = ensemble(U, w, dims)
        arr = {"U": U, "dims": np.array(dims)}
        if w is not None:
            arr["w"] = w
        arr.update(result_arrays("pid", fd.depth_pid(e)))
        arr.update(result_arrays("pidmean", fd.depth_pid_mean(e)))
        arr.update(result_arrays("dice", fd.depth_similarity_baseline(e, "dice")))
        arr.update(result_arrays("iou", fd.depth_similarity_baseline(e, "iou")))
        if n >= 2:
            cmp = fd.compare_pid_vs_mean(e)
            arr["cmp"] = np.array([cmp[k] for k in CMP_KEYS])
        arr["mass"] = fd.member_masses(e)
        arr["mean"] = fd.mean_mask(e).values
        if int(np.prod(dims)) * n <= 4000:
            ww = w if w is not None else np.ones(int(np.prod(dims)))
            mem = [u.astype(np.float64) for u in U]
            a, b, c = ref_pid(mem, ww)
            arr.update(ref_pid_in_in=np.array(a), ref_pid_in_out=np.array(b), ref_pid_depth=np.array(c))
            a, b, c = ref_pid_mean(mem, ww)
            arr.update(ref_pm_in_in=np.array(a), ref_pm_in_out=np.array(b), ref_pm_depth=np.array(c))
        save(f"fuzzy_{k:02d}", **arr)

    binary_cases = [
        (13, 8, (5, 5), False), (13, 8, (5, 5), True), (78, 16, (17, 13, 7), True),
        (5, 40, (64, 64), False),
    ] + [(100 + s, 24, (12, 11), False) for s in range(8)]
    for k, (seed, n, dims, weighted) in enumerate(binary_cases):
        U, w = binary(seed, n, dims, weighted)
        e = ensemble(U, w, dims)
        arr = {"U": U, "dims": np.array(dims)}
        if w is not None:
            arr["w"] = w
        arr.update(result_arrays("eid", fd.depth_eid(e)))
        arr.update(result_arrays("pid", fd.depth_pid(e)))
        if int(np.prod(dims)) * n <= 4000:
            ww = w if w is not None else np.ones(int(np.prod(dims)))
            a, b, c = ref_eid([u.astype(np.float64) for u in U], ww)
            arr.update(ref_eid_in_in=np.array(a), ref_eid_in_out=np.array(b), ref_eid_depth=np.array(c))
        save(f"binary_{k:02d}", **arr)

    # reference generators (inputs for the synth restatement + depths)
    e = fd.gen_disk_ensemble(64, 12, 0)
    U = e.block_values(0, len(e))
    save("gen_disks", U=U, **result_arrays("pid", fd.depth_pid(e)),
         **result_arrays("pidmean", fd.depth_pid_mean(e)))
    e = fd.gen_ellipsoid_ensemble(16, 8, 2, 0)
    U = e.block_values(0, len(e))
    save("gen_ellipsoids", U=U, **result_arrays("pid", fd.depth_pid(e)),
         **result_arrays("pidmean", fd.depth_pid_mean(e)))
    e = fd.gen_contour_ensemble_2d(10, 32, 0)
    U = e.block_values(0, len(e))
    save("gen_contours", U=U, **result_arrays("eid", fd.depth_eid(e)),
         **result_arrays("pidmean", fd.depth_pid_mean(e)))

    # pairwise operators
    rng = np.random.default_rng(7)
    us = rng.uniform(size=(6, 50))
    vs = rng.uniform(size=(6, 50))
    ws = rng.uniform(0.5, 2.0, size=(6, 50))
    inc = []
    for k in range(6):
        w = ws[k] if k % 2 else None
        g = fd.GridSpec((50,), w)
        inc.append(fd.prob_inclusion(fd.ProbMask(g, us[k]), fd.ProbMask(g, vs[k])))
    a = rng.uniform(size=(6, 50)) < 0.5
    b = rng.uniform(size=(6, 50)) < 0.5
    sub = []
    for k in range(6):
        w = ws[k] if k % 2 else None
        g = fd.GridSpec((50,), w)
        sub.append(fd.subset_epsilon(fd.BinaryMask(g, a[k]), fd.BinaryMask(g, b[k])))
    dice, iou = [], []
    for k in range(6):
        w = ws[k] if k % 2 else None
        g = fd.GridSpec((50,), w)
        pu, pv = fd.ProbMask(g, us[k]), fd.ProbMask(g, vs[k])
        dice.append(fd.fuzzy_dice(pu, pv))
        iou.append(fd.prob_iou(pu, pv))
    save("pairs", u=us, v=vs, w=ws, inc=np.array(inc), a=a, b=b, sub=np.array(sub),
         dice=np.array(dice), iou=np.array(iou))


def tools_golden():
    """Host-side formats and callers of the depth path: CSV bytes, fuzzify,
    boxplot envelopes / slice images, stability and rank scatter."""
    import json
    import tempfile

    from fuzzdepth import boxplot as bx
    from fuzzdepth import consistency as cons
    from fuzzdepth import fuzzify as fz
    from fuzzdepth import io as fio

    z = np.load(OUT / "fuzzy_07.npz")
    U, w, dims = z["U"], z["w"], tuple(int(d) for d in z["dims"])
    e = ensemble(U, w, dims)
    pid = fd.depth_pid(e)
    pm = fd.depth_pid_mean(e)
    with tempfile.TemporaryDirectory() as td:
        fio.write_depth_csv(pid, f"{td}/d.csv", workers=1)
        csv_bytes = open(f"{td}/d.csv", "rb").read()
        art = bx.build_boxplot(e, pid, [0.25, 0.5, 1.0], 0.5, 2)
        pgms = [open(p, "rb").read() for p in bx.emit_slice_images(art, e, 2, 3, td)]
        pgms += [open(p, "rb").read() for p in bx.emit_slice_images(art, e, 0, 8, td)]
    (OUT / "tools_depth_pid.csv").write_bytes(csv_bytes)
    arrays = {"pgm_%d" % i: np.frombuffer(b, dtype=np.uint8) for i, b in enumerate(pgms)}
    for b, band in enumerate(art.bands):
        arrays[f"union_{b}"] = band.union.bits
        arrays[f"inter_{b}"] = band.intersection.bits
    rng = np.random.default_rng(11)
    field = rng.normal(size=(9, 10, 11))
    g = fd.GridSpec(field.shape)
    f = fz.ScalarField(g, field)
    arrays["field"] = field
    arrays["fz_iso"] = fz.fuzzy_isocontour(f, 0.3, 0.7).values
    arrays["fz_iso_default"] = fz.fuzzy_isocontour(f, -0.2, fz.default_width(f)).values
    arrays["fz_sub"] = fz.hard_isocontour(f, 0.1).bits
    arrays["fz_minmax"] = fz.normalize_density(f, "minmax").values
    arrays["fz_sbm"] = fz.normalize_density(fz.ScalarField(g, np.abs(field)), "scale-by-max").values
    planes = (rng.uniform(size=(4, 12, 13)) < 0.6)
    arrays["planes"] = planes
    arrays["edges"] = np.stack([bx._contour_cells(p) for p in planes])
    np.savez_compressed(OUT / "tools.npz", **arrays)
    meta = {
        "bands": [{"percentile": b.percentile, "member_ids": list(b.member_ids)} for b in art.bands],
        "median_id": art.median_id, "outlier_ids": list(art.outlier_ids),
        "stability_pid_3": cons.stability_test(e, "pid", 3),
        "stability_pidmean_0": cons.stability_test(e, "pid-mean", 0),
        "scatter": [list(r) for r in cons.rank_scatter(pid, pm).rows],
        "scatter_stats": [cons.rank_scatter(pid, pm).pearson, cons.rank_scatter(pid, pm).kendall],
        "ids": list(e.ids),
    }
    (OUT / "tools.json").write_text(json.dumps(meta, indent=1) + "\n")
    print("tools", sorted(arrays))


if __name__ == "__main__":
    main()
    tools_golden()
