#!/usr/bin/env python
"""Run the reference's OWN test suite with its depth path routed to the B200.

    python tools/run_reference_suite.py [--off] [pytest args...]

Imports the unmodified reference from baseline/_ref (tools/install_reference.sh),
applies ``paper_2512_15187_b200.integration.install`` (the module swap of
INTEGRATION.md §2) BEFORE pytest imports the test modules, so every
``from fuzzdepth.depth import depth_pid`` in the reference tests binds the GPU
function, then runs baseline/_ref/tests (a copy of
/root/reference/pkg/tests).  ``--off`` runs the same suite on the stock CPU
reference (control).  Needs a CUDA device unless ``--off``.
"""
from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"


def main(argv: list[str]) -> int:
    off = "--off" in argv
    argv = [a for a in argv if a != "--off"]
    if not (REF / "fuzzdepth").exists() or not (REF / "tests").exists():
        print("baseline/_ref missing: run tools/install_reference.sh first", file=sys.stderr)
        return 2
    sys.path.insert(0, str(REF))
    sys.path.insert(0, str(ROOT))
    import fuzzdepth  # noqa: F401  (the reference, unmodified)

    if not off:
        import torch

        if not torch.cuda.is_available():
            print("no CUDA device: the routed suite needs the B200", file=sys.stderr)
            return 2
        from paper_2512_15187_b200 import integration

        done = integration.install(fuzzdepth)
        print(f"routed {len(done)} reference bindings to the B200 path:")
        for d in done:
            print("  ", d)
    import pytest

    tests = REF / "tests"
    args = argv or [str(tests)]
    return pytest.main(["-p", "no:cacheprovider", "-c", str(tests / "pytest.ini"),
                        "--rootdir", str(tests), "-q", "-rfE", *args])


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
