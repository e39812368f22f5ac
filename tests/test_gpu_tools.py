"""GPU side of ingestion, the CLI and the callers around the depth path:
stage_manifest, K10 band envelopes (build_boxplot), slice images,
stability_test and the CLI subcommands, against fixtures produced by the
reference itself (tests/golden/make_golden.py: tools_golden)."""
from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN, golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pb():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2512_15187_b200 as pb

    return pb


def close(got, want, atol):
    np.testing.assert_allclose(got, want, rtol=0, atol=atol)


def fixture07(pb):
    z = golden("fuzzy_07")
    dims = tuple(int(d) for d in z["dims"])
    g = pb.GridSpec(dims, z["w"])
    return z, pb.Ensemble(g, [pb.ProbMask(g, u) for u in z["U"]])


def write_manifest_dir(pb, tmp_path, U, dims, weights=None, raw_every=3):
    (tmp_path / "members").mkdir(exist_ok=True)
    entries = []
    for i, u in enumerate(U):
        name = f"members/m{i:03d}" + (".raw" if i % raw_every == 1 else ".npy")
        pb.write_volume(u.reshape(dims), tmp_path / name)
        entries.append({"id": f"m{i:03d}", "path": name})
    wp = None
    if weights is not None:
        pb.write_volume(np.asarray(weights), tmp_path / "w.npy")
        wp = "w.npy"
    pb.write_manifest(tmp_path / "manifest.json", dims, entries, weights_path=wp)
    return tmp_path / "manifest.json"


def test_stage_manifest_matches_loader_path(pb, tmp_path):
    z, _ = fixture07(pb)
    dims = tuple(int(d) for d in z["dims"])
    m = write_manifest_dir(pb, tmp_path, z["U"], dims, z["w"])
    de = pb.stage_manifest(m)
    ref = pb.stage(pb.read_manifest(m))
    assert de.ids == ref.ids and de.dims == ref.dims
    assert torch.equal(de.values[:, :de.m], ref.values[:, :ref.m])
    assert np.array_equal(de.weights_host, z["w"])
    r = pb.depth_pid(de)
    close(r.depth, z["pid_depth"], 1e-13)
    np.testing.assert_array_equal(r.rank, z["pid_rank"])


def test_stage_manifest_binary_threshold(pb, tmp_path):
    rng = np.random.default_rng(4)
    (tmp_path / "v").mkdir()
    entries = []
    for i in range(3):
        pb.write_volume(rng.uniform(size=(6, 7)).astype(np.float32), tmp_path / f"v/u{i}.npy")
        entries.append({"id": f"u{i}", "path": f"v/u{i}.npy"})
    bits = (rng.uniform(size=(6, 7)) < 0.5).astype(np.uint8)
    pb.write_volume(bits, tmp_path / "v/b.npy")
    entries.append({"id": "b", "path": "v/b.npy"})
    pb.write_manifest(tmp_path / "m.json", (6, 7), entries)
    de = pb.stage_manifest(tmp_path / "m.json")
    e = pb.read_manifest(tmp_path / "m.json")
    want = np.stack([e.member(i).values for i in range(len(e))])
    assert np.array_equal(de.values[:, :de.m].cpu().numpy(), want)
    t = 0.7  # rounds down in float32: the comparison must be done in float32
    dt = pb.stage_manifest(tmp_path / "m.json", threshold=t)
    bw = np.stack([pb.binarize(e.member(i), t).bits for i in range(len(e))]).astype(np.float32)
    assert np.array_equal(dt.values[:, :dt.m].cpu().numpy(), bw)
    # out-of-range float member -> ValidationError from the device check
    pb.write_volume(np.full((6, 7), 1.5, dtype=np.float32), tmp_path / "v/bad.npy")
    pb.write_manifest(tmp_path / "bad.json", (6, 7), [{"id": "x", "path": "v/bad.npy"}])
    with pytest.raises(pb.ValidationError):
        pb.stage_manifest(tmp_path / "bad.json")


def test_stage_manifest_binary_is_byte_ensemble(pb, tmp_path):
    """A manifest of uint8 / bool masks stages as a byte ensemble: eID reads
    the bytes, the other methods its float32 view; results equal those of the
    reference-loaded (float32) ensemble; a 0/2 member raises with its id."""
    rng = np.random.default_rng(6)
    (tmp_path / "v").mkdir()
    entries = []
    for i in range(5):
        b = rng.uniform(size=(9, 11)) < rng.uniform(0.2, 0.8)
        pb.write_volume(b if i % 2 else b.astype(np.uint8), tmp_path / f"v/b{i}.npy")
        entries.append({"id": f"b{i}", "path": f"v/b{i}.npy"})
    pb.write_manifest(tmp_path / "m.json", (9, 11), entries)
    de = pb.stage_manifest(tmp_path / "m.json")
    assert de.is_bits
    e = pb.read_manifest(tmp_path / "m.json")
    for fn in (pb.depth_eid, pb.depth_pid, pb.depth_pid_mean):
        a, b = fn(de), fn(e)
        assert np.array_equal(a.depth, b.depth) and np.array_equal(a.rank, b.rank)
    from paper_2512_15187_b200.cli import main as cli_main

    for meth in ("eid", "pid", "pid-mean"):  # the CLI on the byte ensemble
        out = tmp_path / f"d_{meth}.csv"
        assert cli_main(["depth", "--manifest", str(tmp_path / "m.json"), "--method", meth,
                         "--out", str(out)]) == 0
        got = pb.read_depth_csv(out)
        assert np.array_equal(got.depth, pb.depth_by_method(e, meth).depth)
    bad = (rng.uniform(size=(9, 11)) < 0.5).astype(np.uint8) * 2
    pb.write_volume(bad, tmp_path / "v/bad.npy")
    pb.write_manifest(tmp_path / "bad.json", (9, 11), entries + [{"id": "two", "path": "v/bad.npy"}])
    with pytest.raises(pb.ValidationError, match="'two': binary mask values must be 0 or 1"):
        pb.stage_manifest(tmp_path / "bad.json")


def test_stage_manifest_rejects_non_binary_uint8(pb, tmp_path):
    """A 0/255 uint8 mask loads through BinaryMask in the reference, which
    raises ValidationError (grid.py:145-147); staging it must raise too (and
    a CLI depth run exit 1), not feed 255.0 into the kernels."""
    (tmp_path / "v").mkdir()
    ok = (np.arange(42).reshape(6, 7) % 2).astype(np.uint8)
    np.save(tmp_path / "v/ok.npy", ok)
    np.save(tmp_path / "v/b255.npy", ok * 255)
    np.save(tmp_path / "v/f.npy", np.full((6, 7), 0.5, dtype=np.float32))
    pb.write_manifest(tmp_path / "m.json", (6, 7), [{"id": "ok", "path": "v/ok.npy"},
                                                     {"id": "f", "path": "v/f.npy"},
                                                     {"id": "bad", "path": "v/b255.npy"}])
    with pytest.raises(pb.ValidationError, match="binary mask values must be 0 or 1"):
        pb.stage_manifest(tmp_path / "m.json")
    from paper_2512_15187_b200.cli import main as cli_main

    rc = cli_main(["depth", "--manifest", str(tmp_path / "m.json"), "--method", "pid",
                   "--out", str(tmp_path / "d.csv")])
    assert rc == 1


def test_build_boxplot_matches_reference(pb, tmp_path):
    z, e = fixture07(pb)
    t, meta = golden("tools"), json.loads((GOLDEN / "tools.json").read_text())
    result = pb.read_depth_csv(GOLDEN / "tools_depth_pid.csv")
    art = pb.build_boxplot(e, result, [0.25, 0.5, 1.0], 0.5, 2)
    assert art.median_id == meta["median_id"]
    assert list(art.outlier_ids) == meta["outlier_ids"]
    for b, band in enumerate(art.bands):
        assert np.array_equal(band.union.bits, t[f"union_{b}"])
        assert np.array_equal(band.intersection.bits, t[f"inter_{b}"])
        assert list(band.member_ids) == meta["bands"][b]["member_ids"]
    imgs = [open(f, "rb").read() for f in pb.emit_slice_images(art, e, 2, 3, tmp_path)]
    imgs += [open(f, "rb").read() for f in pb.emit_slice_images(art, e, 0, 8, tmp_path)]
    for i, img in enumerate(imgs):  # same file names per call: read before the next one
        assert np.array_equal(np.frombuffer(img, np.uint8), t[f"pgm_{i}"])
    with pytest.raises(pb.ValidationError):
        pb.build_boxplot(e, result, [0.5, 0.25])
    with pytest.raises(pb.ValidationError):
        pb.build_boxplot(e, result, [0.5], outlier_count=24)


def test_band_envelopes_vs_numpy(pb):
    rng = np.random.default_rng(9)
    for n, m, dt in ((37, 1001, np.float32), (300, 4099, np.float64), (5, 3, np.float32)):
        U = rng.uniform(size=(n, m)).astype(dt)
        rank = rng.permutation(n)
        cut = sorted({max(1, int(np.ceil(p * n))) for p in (0.1, 0.5, 0.9, 1.0)})
        uni, inter = pb.boxplot.band_envelopes(torch.from_numpy(U), rank, cut, 0.45)
        bits = U >= dt(0.45)
        for b, k in enumerate(cut):
            sel = bits[rank < k]
            assert np.array_equal(uni[b], sel.any(0)) and np.array_equal(inter[b], sel.all(0))


def test_stability_matches_reference(pb):
    _, e = fixture07(pb)
    meta = json.loads((GOLDEN / "tools.json").read_text())
    for key, method, k in (("stability_pid_3", "pid", 3), ("stability_pidmean_0", "pid-mean", 0)):
        got, want = pb.stability_test(e, method, k), meta[key]
        assert got["removed_ids"] == want["removed_ids"]
        assert got["pearson"] == pytest.approx(want["pearson"], abs=1e-12)
        assert got["kendall"] == pytest.approx(want["kendall"], abs=1e-12)
    with pytest.raises(pb.ValidationError):
        pb.stability_test(e, "pid", 24)


def test_cli_end_to_end(pb, tmp_path, capsys):
    from paper_2512_15187_b200.cli import main

    z, _ = fixture07(pb)
    dims = tuple(int(d) for d in z["dims"])
    m = write_manifest_dir(pb, tmp_path, z["U"], dims, z["w"])
    out = tmp_path / "d.csv"
    assert main(["depth", "--manifest", str(m), "--method", "pid", "--out", str(out)]) == 0
    r = pb.read_depth_csv(out)
    close(r.depth, z["pid_depth"], 1e-13)
    np.testing.assert_array_equal(r.rank, z["pid_rank"])
    assert main(["depth", "--manifest", str(m), "--method", "eid", "--out", str(out)]) == 2
    assert main(["depth", "--manifest", str(m), "--method", "eid", "--threshold", "0.5",
                 "--out", str(tmp_path / "e.csv")]) == 0
    assert main(["depth", "--manifest", str(m), "--method", "dice", "--out",
                 str(tmp_path / "dice.csv")]) == 0
    close(pb.read_depth_csv(tmp_path / "dice.csv").depth, z["dice_depth"], 1e-13)
    assert main(["boxplot", "--manifest", str(m), "--depths", str(out), "--percentiles",
                 "0.5,1.0", "--outliers", "1", "--slice", "2,3", "--out-dir",
                 str(tmp_path / "bx")]) == 0
    doc = json.loads((tmp_path / "bx" / "boxplot.json").read_text())
    assert len(doc["bands"]) == 2 and len(doc["slices"]) == 2
    assert main(["consistency", "--stability", "--manifest", str(m), "--method", "pid",
                 "--remove", "2", "--out", str(tmp_path / "st.json")]) == 0
    assert main(["synth", "disks", "--res", "16", "--n", "6", "--out-dir",
                 str(tmp_path / "syn")]) == 0
    assert main(["depth", "--manifest", str(tmp_path / "syn" / "manifest.json"), "--method",
                 "pid-mean", "--out", str(tmp_path / "s.csv")]) == 0
    assert main(["synth", "contours2d", "--res", "16", "--n", "5", "--out-dir",
                 str(tmp_path / "c2")]) == 0
    assert pb.manifest_guarantees_binary(tmp_path / "c2" / "manifest.json")
    assert main(["depth", "--manifest", str(tmp_path / "c2" / "manifest.json"), "--method",
                 "eid", "--out", str(tmp_path / "c.csv")]) == 0
