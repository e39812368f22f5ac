"""Host-side logic of the drop-in (CPU only): containers, validation, error
types, rank/CV helpers, sharding bounds, and the no-CPU-fallback rule."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2512_15187_b200 as pb
from conftest import TRIO


def test_error_hierarchy():
    for cls in (pb.ValidationError, pb.GridMismatchError, pb.DegenerateEnsembleError,
                pb.VolumeFormatError, pb.ManifestError):
        assert issubclass(cls, pb.FuzzdepthError)


def test_gridspec_and_masks_validate_like_the_reference():
    with pytest.raises(pb.ValidationError):
        pb.GridSpec((0, 3))
    with pytest.raises(pb.ValidationError):
        pb.GridSpec((3,), np.array([1.0, -1.0, 1.0]))
    g = pb.GridSpec((2, 2))
    m = pb.ProbMask(g, np.array([[0.0, 1.0 + 5e-10], [-5e-10, 0.5]]))
    assert m.values.dtype == np.float64 and m.values.max() == 1.0 and m.values.min() == 0.0
    assert pb.ProbMask(g, np.zeros(4, dtype=np.int32)).values.dtype == np.float32
    assert not m.values.flags.writeable
    assert pb.ProbMask(g, np.zeros(4)).values.dtype == np.float64
    with pytest.raises(pb.ValidationError):
        pb.ProbMask(g, np.array([0, 0, 0, 1.1]))
    with pytest.raises(pb.ValidationError):
        pb.ProbMask(g, np.array([0, 0, np.nan, 1]))
    with pytest.raises(pb.ValidationError):
        pb.BinaryMask(g, np.array([0, 2, 0, 1]))
    with pytest.raises(pb.DegenerateEnsembleError):
        pb.Ensemble(g, [])
    with pytest.raises(pb.ValidationError):
        pb.Ensemble(g, [m, m], ids=["a", "a"])
    with pytest.raises(pb.GridMismatchError):
        pb.Ensemble(g, [pb.ProbMask(pb.GridSpec((4,)), np.zeros(4))])
    e = pb.Ensemble(g, [m, lambda: m])
    assert e.is_lazy() and len(e.materialize()) == 2
    assert e.ids == ("member_0000", "member_0001")


def test_rank_and_cv_helpers():
    np.testing.assert_array_equal(pb.ranks_from_depths(np.array([0.5, 0.7, 0.5])), [1, 0, 2])
    np.testing.assert_array_equal(pb.ranks_from_depths(np.array([0.2, 0.2])), [0, 1])
    assert pb.mass_cv(np.zeros(3)) == 0.0
    assert pb.mass_cv(np.array([3.0, 2.0, 1.0])) == pytest.approx(np.sqrt(2 / 3) / 2)


def test_depth_result_is_frozen():
    r = pb.DepthResult(("a", "b"), np.zeros(2), np.zeros(2), np.array([0.1, 0.2]),
                       np.array([1, 0]), "pid", 0.0, 0.0)
    assert r.ordered_ids() == ["b", "a"]
    with pytest.raises(ValueError):
        r.depth[0] = 1.0
    with pytest.raises(pb.ValidationError):
        pb.DepthResult(("a",), np.zeros(2), np.zeros(2), np.zeros(2), np.zeros(2), "pid", 0, 0)


def test_workers_contract():
    with pytest.raises(ValueError):
        pb.resolve_workers(0)
    assert pb.resolve_workers(3) == 3


@pytest.mark.parametrize("m,world", [(10, 3), (134217728, 8), (7, 8), (65536, 2)])
def test_shard_bounds_partition(m, world):
    spans = [pb.shard_bounds(m, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == m
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c and b >= a
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    g = pb.GridSpec((4,))
    e = pb.Ensemble(g, [pb.ProbMask(g, r) for r in TRIO])
    for fn in (pb.depth_pid, pb.depth_pid_mean, pb.depth_eid):
        with pytest.raises(RuntimeError, match="no CPU fallback"):
            fn(e)


def test_unknown_method_rejected_before_any_device_work():
    with pytest.raises(pb.ValidationError):
        pb.depth_pid(np.zeros((2, 3)), algorithm="bogus")


def test_ensemble_operations_like_the_reference():
    """grid.py:159-296 behaviours (reference tests/test_grid.py TestEnsemble,
    TestPermuteCells; binarize)."""
    g = pb.GridSpec((4,))
    masks = [pb.ProbMask(g, u) for u in TRIO]
    e = pb.Ensemble(g, masks, ids=["c0", "c1", "c2"])
    np.testing.assert_array_equal(e.block_values(1, 3), TRIO[1:3])
    assert e.subset([2, 0]).ids == ("c2", "c0")
    calls = []

    def loader(i):
        def f():
            calls.append(i)
            return masks[i]
        return f

    lazy = pb.Ensemble(g, [loader(i) for i in range(3)])
    mapped = lazy.map_members(lambda m: pb.binarize(m, 0.5).to_prob())
    assert calls == [] and mapped.is_lazy()
    np.testing.assert_array_equal(mapped.member(1).values, TRIO[1])
    assert calls == [1]
    with pytest.raises(pb.GridMismatchError):  # a loader on another grid fails on access
        pb.Ensemble(g, [lambda: pb.ProbMask(pb.GridSpec((2, 2)), np.zeros(4))]).member(0)
    perm = np.array([3, 1, 0, 2])
    p = pb.permute_cells(e, perm)
    np.testing.assert_array_equal(p.member(0).values, TRIO[0][perm])
    with pytest.raises(pb.ValidationError):
        pb.permute_cells(e, np.array([0, 0, 1, 2]))
    # binarize compares in the member dtype (numpy: Python float -> float32)
    u = pb.ProbMask(g, np.full(4, np.float32(0.7)))
    assert pb.binarize(u, 0.7).bits.all()
    with pytest.raises(pb.ValidationError):
        pb.binarize(u, 0.0)
    with pytest.raises(pb.ValidationError):
        pb.binarize_ensemble(e, 1.5)


def test_gen_fuzzy_disk_matches_reference_members():
    """gen_fuzzy_disk (synth.py:30-51) on the host: the reference's disk
    members (golden gen_disks = gen_disk_ensemble(64, 12, 0)) bit for bit."""
    from conftest import golden
    from paper_2512_15187_b200.synth import disk_params

    z = golden("gen_disks")
    prm, sigma2, _ = disk_params(64, 12, 0)
    g = pb.GridSpec((64, 64))
    for i in (0, 5, 11):
        cy, cx, r = prm[i]
        assert np.array_equal(pb.gen_fuzzy_disk(g, (cy, cx), r, sigma2).values, z["U"][i])
    with pytest.raises(pb.ValidationError):
        pb.gen_fuzzy_disk(pb.GridSpec((4,)), (0, 0), 1.0, 1.0)


def test_gram_certifier_host_logic():
    """Rank certifier of the tensor-core PID (depth._clustered /
    _gram_depth_bounds): overlapping error intervals are flagged as whole
    clusters, separated members are not; the bound grows with the soft-cell
    counts and vanishes for exact (digit-free) members."""
    from paper_2512_15187_b200.depth import _clustered, _gram_depth_bounds

    d = np.array([0.5, 0.1, 0.30, 0.3000001, 0.9, 0.2999999])
    eps = np.full(6, 1e-6)
    np.testing.assert_array_equal(_clustered(d, eps), [False, False, True, True, False, True])
    assert not _clustered(d, np.full(6, 1e-8)).any()
    assert _clustered(np.array([0.2, 0.2]), np.zeros(2)).all()  # exact tie
    m = np.array([10.0, 20.0, 30.0])
    inv = 1.0 / m
    rp, ci = np.array([30.0, 60.0, 90.0]), np.array([3.0, 3.0, 3.0])
    e0 = _gram_depth_bounds(m, np.zeros(3, dtype=np.int64), inv, rp, ci, 100.0, 1.0, 1.0)
    e1 = _gram_depth_bounds(m, np.array([50, 60, 70]), inv, rp, ci, 100.0, 1.0, 1.0)
    assert (e0 < 1e-9).all() and (e1 > e0).all() and (e1 < 1e-6).all()
