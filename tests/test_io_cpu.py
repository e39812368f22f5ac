"""Host side of the drop-in's ingestion / output formats and of the callers
around the depth path (io, boxplot images, consistency, CLI exit
codes), checked against fixtures produced by the reference itself
(tests/golden/make_golden.py: tools_golden).  No GPU needed."""
from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN, golden

pb = pytest.importorskip("paper_2512_15187_b200")
from paper_2512_15187_b200 import boxplot as bx  # noqa: E402
from paper_2512_15187_b200 import consistency as cons  # noqa: E402
from paper_2512_15187_b200 import io as pio  # noqa: E402
from paper_2512_15187_b200.cli import main as cli_main  # noqa: E402


def tools():
    return golden("tools"), json.loads((GOLDEN / "tools.json").read_text())


def test_field_members_are_out_of_scope(tmp_path):
    """Field-role members need fuzzification (fuzzify.py), input preparation
    outside the depth path: the manifest still parses, loading one raises."""
    np.save(tmp_path / "f.npy", np.ones((3, 4)))
    m = _manifest(tmp_path, [{"id": "f", "path": "f.npy", "role": "field",
                              "fuzzify": {"mode": "sublevel", "q": 0.0}}])
    e = pio.read_manifest(m)
    with pytest.raises(pb.ManifestError, match="fuzzif"):
        e.member(0)


def test_contour_cells_and_pgm(tmp_path):
    z, _ = tools()
    for p, want in zip(z["planes"], z["edges"]):
        assert np.array_equal(bx._edge(p), want)
    img = np.arange(12, dtype=np.uint8).reshape(3, 4)
    bx.write_pgm(tmp_path / "a.pgm", img)
    assert (tmp_path / "a.pgm").read_bytes() == b"P5\n4 3\n255\n" + img.tobytes()
    with pytest.raises(pb.ValidationError):
        bx.write_pgm(tmp_path / "b.pgm", img.astype(np.int16))


def test_depth_csv_is_byte_compatible(tmp_path):
    want = (GOLDEN / "tools_depth_pid.csv").read_bytes()
    r = pio.read_depth_csv(GOLDEN / "tools_depth_pid.csv")
    assert r.method == "pid" and len(r) == 24
    pio.write_depth_csv(r, tmp_path / "d.csv", workers=1)
    assert (tmp_path / "d.csv").read_bytes() == want
    meta = json.loads((tmp_path / "d.csv.json").read_text())
    assert list(meta) == ["method", "cv_mass", "elapsed_seconds", "n", "workers"]
    (tmp_path / "bad.csv").write_text("id,in_in\nx,1\n")
    with pytest.raises(pb.ValidationError):
        pio.read_depth_csv(tmp_path / "bad.csv")


def test_rank_scatter_and_correlations():
    z07 = golden("fuzzy_07")
    _, meta = tools()
    ids = tuple(meta["ids"])
    a = pb.DepthResult(ids, z07["pid_in_in"], z07["pid_in_out"], z07["pid_depth"], z07["pid_rank"],
                       "pid", 0.0, 0.0)
    b = pb.DepthResult(ids, z07["pidmean_in_in"], z07["pidmean_in_out"], z07["pidmean_depth"],
                       z07["pidmean_rank"], "pid-mean", 0.0, 0.0)
    sc = cons.rank_scatter(a, b)
    assert [list(r) for r in sc.rows] == meta["scatter"]
    assert sc.pearson == pytest.approx(meta["scatter_stats"][0], abs=1e-15)
    assert sc.kendall == pytest.approx(meta["scatter_stats"][1], abs=1e-15)
    with pytest.raises(pb.ValidationError):
        cons.pearson([1, 1, 1], [1, 2, 3])
    with pytest.raises(pb.ValidationError):
        cons.kendall_tau([1], [1])


def test_volumes_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    for arr in (rng.uniform(size=(4, 5)).astype(np.float32), rng.uniform(size=7),
                (rng.uniform(size=(2, 3, 4)) < 0.5).astype(np.uint8)):
        for name in ("v.npy", "v.raw"):
            pio.write_volume(arr, tmp_path / name)
            assert pio.volume_header(tmp_path / name) == (arr.shape, arr.dtype.name)
            back = pio._load_array(tmp_path / name)
            assert back.dtype == arr.dtype and np.array_equal(back, arr)
            mm = pio._load_array(tmp_path / name, mmap=True)
            assert np.array_equal(np.asarray(mm), arr)
    np.save(tmp_path / "be.npy", np.arange(4, dtype=">f4"))
    with pytest.raises(pb.VolumeFormatError):
        pio.read_volume(tmp_path / "be.npy")
    np.save(tmp_path / "i.npy", np.arange(4, dtype=np.int32))
    with pytest.raises(pb.VolumeFormatError):
        pio.read_volume(tmp_path / "i.npy")
    (tmp_path / "orphan.raw").write_bytes(b"\0" * 8)
    with pytest.raises(pb.VolumeFormatError):
        pio.volume_header(tmp_path / "orphan.raw")


def _manifest(tmp_path, entries, dims=(3, 4), weights=None):
    doc = {"grid": {"dims": list(dims)}, "members": entries}
    if weights is not None:
        np.save(tmp_path / "w.npy", weights)
        doc["grid"]["weights_path"] = "w.npy"
    (tmp_path / "m.json").write_text(json.dumps(doc))
    return tmp_path / "m.json"


def test_manifest_rules(tmp_path):
    rng = np.random.default_rng(1)
    np.save(tmp_path / "a.npy", rng.uniform(size=(3, 4)).astype(np.float32))
    np.save(tmp_path / "b.npy", (rng.uniform(size=12) < 0.5).astype(np.uint8))
    np.save(tmp_path / "f.npy", rng.normal(size=(3, 4)))
    m = _manifest(tmp_path, [{"id": "a", "path": "a.npy"}, {"id": "b", "path": "b.npy"}],
                  weights=rng.uniform(0.5, 2, size=12))
    e = pio.read_manifest(m)
    assert e.ids == ("a", "b") and e.is_lazy()
    assert np.array_equal(e.member(0).values, np.load(tmp_path / "a.npy").reshape(-1))
    assert np.array_equal(e.member(1).values, np.load(tmp_path / "b.npy").astype(np.float32))
    assert e.grid.weights is not None
    assert not pio.manifest_guarantees_binary(m)
    mb = _manifest(tmp_path, [{"id": "b", "path": "b.npy"}])
    assert pio.manifest_guarantees_binary(mb)
    bad = [
        [{"id": "a", "path": "a.npy"}, {"id": "a", "path": "b.npy"}],          # duplicate id
        [{"id": "x", "path": "missing.npy"}],                                    # no file
        [{"id": "f", "path": "f.npy", "role": "field"}],                         # no fuzzify
        [{"id": "f", "path": "f.npy", "role": "field", "fuzzify": {"mode": "isovalue"}}],
        [{"id": "a", "path": "a.npy", "fuzzify": {"mode": "minmax"}}],          # mask + fuzzify
        [{"id": "a", "path": "a.npy", "role": "shape"}],
        [],
    ]
    for entries in bad:
        with pytest.raises(pb.ManifestError):
            pio.read_manifest(_manifest(tmp_path, entries))
    with pytest.raises(pb.ManifestError):  # shape mismatch
        pio.read_manifest(_manifest(tmp_path, [{"id": "a", "path": "a.npy"}], dims=(4, 4)))


def test_cli_exit_codes(tmp_path, capsys):
    assert cli_main(["depth", "--manifest", str(tmp_path / "none.json"), "--method", "pid",
                     "--out", str(tmp_path / "o.csv")]) == 1
    with pytest.raises(SystemExit) as ex:
        cli_main(["depth", "--manifest", "m.json", "--method", "band", "--out", "o.csv"])
    assert ex.value.code == 2
    assert cli_main(["consistency", str(tmp_path / "a.csv")]) == 2
    assert cli_main(["consistency", "--stability"]) == 2
    # rank scatter between two CSVs is host-only
    src = GOLDEN / "tools_depth_pid.csv"
    assert cli_main(["consistency", str(src), str(src), "--out", str(tmp_path / "s.csv")]) == 0
    lines = (tmp_path / "s.csv").read_text().splitlines()
    assert lines[0] == "# pearson=1.0 kendall=1.0" and lines[1] == "id,rank_a,rank_b,abs_delta"
