"""Parity past 2^31 elements: the headline
configurations put more than 2^31 member-voxels on the device, so 64-bit
indexing, the per-CTA cell ranges and the split reductions are checked
against the CPU oracle at that size, not only at fixture sizes.

* 9 members x 2^28 cells (2.42e9 elements, 9.7 GB fp32): K5 (PID-mean), K9
  (exact PID), K6 (masses), the tensor-core Gram PID (K1x), and eID (K7 + K2
  + exact epilogue) on the binarised ensemble -- against oracle.port (the
  reference's algorithm: 65 536-cell chunks, fp64) and, for eID, the exact
  integer oracle;
* 132 fuzzy ellipsoids x 256^3 (2.21e9 elements): K5, K9, K6 against
  oracle.port (PID-mean, masses) and an fp64 numpy factorisation of exact
  PID (SURVEY.md §0 finding 2; oracle.port's PID would need the reference's
  1 x 1 member tiles at 256^3, ~20 min), plus the Gram path.

Tolerances: 1e-12 absolute on depths (fp64 paths), 1e-8 for the Gram path,
identical ranks everywhere, eID bit-identical.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import exact, port

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pb():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2512_15187_b200 as pb

    return pb


def _check(got, want, atol):
    np.testing.assert_allclose(got.in_in, want["in_in"], rtol=0, atol=atol)
    np.testing.assert_allclose(got.in_out, want["in_out"], rtol=0, atol=atol)
    np.testing.assert_allclose(got.depth, want["depth"], rtol=0, atol=atol)
    np.testing.assert_array_equal(got.rank, want["rank"])


def test_nine_members_2p28_cells(pb):
    n, m = 9, 1 << 28
    assert n * m > 2 ** 31
    g = torch.Generator(device="cuda").manual_seed(5)
    t = torch.rand((n, m), generator=g, device="cuda", dtype=torch.float32)
    de = pb.DeviceEnsemble.from_tensor(t, validate=False)
    U = t.cpu().numpy()
    workers = 16
    _check(pb.depth_pid_mean(de), port.depth_pid_mean(U, workers=workers), 1e-12)
    want = port.depth_pid(U, workers=workers)
    _check(pb.depth_pid(de), want, 1e-12)
    _check(pb.depth_pid(de, algorithm="gram"), want, 1e-8)
    np.testing.assert_allclose(pb.member_masses(de), port.masses(U, workers=workers),
                               rtol=1e-13)
    del de
    B = (t < 0.5).to(torch.float32)
    del t
    db = pb.DeviceEnsemble.from_tensor(B, validate=False)
    Bh = B.cpu().numpy()
    in_in, in_out, depth, _ = exact.eid_fast(Bh)
    r = pb.depth_eid(db)
    assert np.array_equal(r.depth, depth) and np.array_equal(r.rank, port.ranks(depth))
    assert np.array_equal(r.in_in, in_in) and np.array_equal(r.in_out, in_out)


def test_ellipsoids_132_x_256cubed(pb):
    from paper_2512_15187_b200 import synth

    de = synth.ellipsoids_device(256, 132, 0, 1)
    assert de.n * de.m > 2 ** 31
    U = de.values[:, :de.m].cpu().numpy()
    _check(pb.depth_pid_mean(de), port.depth_pid_mean(U, workers=16), 1e-12)
    mass = port.masses(U, workers=16)
    np.testing.assert_allclose(pb.member_masses(de), mass, rtol=1e-13)
    # exact PID by the fp64 factorisation (sum of u_j and of u_j / m_j per cell)
    inv = port.inverse(mass)
    S = np.zeros(de.m)
    T = np.zeros(de.m)
    for i in range(de.n):
        x = U[i].astype(np.float64)
        S += x
        T += inv[i] * x
    in_in = inv * np.array([U[i].astype(np.float64) @ S for i in range(de.n)]) / de.n
    in_out = np.array([U[i].astype(np.float64) @ T for i in range(de.n)]) / de.n
    depth = np.minimum(in_in, in_out)
    want = {"in_in": in_in, "in_out": in_out, "depth": depth, "rank": port.ranks(depth)}
    _check(pb.depth_pid(de), want, 1e-12)
    _check(pb.depth_pid(de, algorithm="gram"), want, 1e-8)
