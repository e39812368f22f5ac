"""INTEGRATION.md §2 module swap (paper_2512_15187_b200.integration) against
the installed, unmodified reference in baseline/_ref: which bindings move and
that uninstall restores them.  CPU only (nothing is called)."""
from __future__ import annotations

import sys
from pathlib import Path

import pytest

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


@pytest.fixture
def fd():
    if not (REF / "fuzzdepth").exists():
        pytest.skip("baseline/_ref not installed (tools/install_reference.sh)")
    sys.path.insert(0, str(REF))
    try:
        import fuzzdepth
    finally:
        sys.path.remove(str(REF))
    return fuzzdepth


def test_install_rebinds_every_depth_path_binding(fd):
    import fuzzdepth.consistency
    import fuzzdepth.depth
    import fuzzdepth.inclusion
    import fuzzdepth.reduction

    import paper_2512_15187_b200 as pb
    from paper_2512_15187_b200 import integration, reduction

    orig = fd.depth.depth_pid
    done = integration.install(fd)
    assert integration.install(fd) == done  # idempotent: originals kept
    try:
        for want in ("fuzzdepth.depth.depth_pid", "fuzzdepth.depth_pid_mean",
                     "fuzzdepth.depth.depth_eid", "fuzzdepth.consistency.depth_by_method",
                     "fuzzdepth.reduction.gram_block", "fuzzdepth.depth._member_mean_terms",
                     "fuzzdepth.inclusion.prob_inclusion", "fuzzdepth.reduction.weighted_sum"):
            assert want in done
        assert fd.depth.depth_pid is pb.depth_pid
        assert fd.depth_by_method is pb.depth_by_method
        assert fd.reduction.gram_block is reduction.gram_block
    finally:
        integration.uninstall()
    assert fd.depth.depth_pid is orig
