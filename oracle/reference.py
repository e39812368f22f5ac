"""The REAL reference package as checker and CPU baseline (TEST INFRASTRUCTURE).

``load()`` imports the unmodified ``fuzzdepth`` installed in baseline/_ref by
tools/install_reference.sh (git-ignored; it travels to the GPU box with
gpurun).  The helpers build reference ``Ensemble`` objects over the same
bytes the GPU reads:

* ``lazy_from_device`` -- one zero-argument loader per member that copies
  that member's row out of HBM on access (the reference's own lazy-loader
  contract, /root/reference/pkg/src/fuzzdepth/grid.py:159-202), so a 107 GB
  device ensemble streams through ``depth_pid_mean`` with only a few members
  resident on the host;
* ``from_array`` -- a materialised ensemble from an (n, cells) host array.

Only tests/, __graft_entry__.smoke() and bench.py (parity and CPU-baseline
legs) use this module; the product never does.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


def load():
    """The installed reference module, or None when baseline/_ref is absent."""
    if not (REF / "fuzzdepth").exists():
        return None
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import fuzzdepth

    if not str(Path(fuzzdepth.__file__).resolve()).startswith(str(REF.resolve())):
        raise ImportError(f"fuzzdepth resolved to {fuzzdepth.__file__}, not baseline/_ref")
    return fuzzdepth


def _grid(fd, dims, weights):
    return fd.GridSpec(tuple(int(d) for d in dims), None if weights is None else
                       np.asarray(weights, dtype=np.float64))


def lazy_from_device(fd, de):
    """Reference Ensemble whose members are copied from ``de`` (a
    paper_2512_15187_b200 DeviceEnsemble) one at a time on access."""
    grid = _grid(fd, de.dims, de.weights_host)
    rows, m = de.values, de.m

    def loader(i):
        return lambda: fd.ProbMask(grid, rows[i, :m].cpu().numpy())

    return fd.Ensemble(grid, [loader(i) for i in range(de.n)], list(de.ids))


def from_array(fd, U, dims=None, weights=None, ids=None):
    """Materialised reference Ensemble from an (n, cells) host array."""
    U = np.asarray(U)
    grid = _grid(fd, dims if dims is not None else (U.shape[1],), weights)
    return fd.Ensemble(grid, [fd.ProbMask(grid, u) for u in U], ids)
