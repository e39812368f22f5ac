"""The C-ABI library loads and exports every entry point include/pidb.h
declares, with a ctypes signature for each (CPU only: no compute calls)."""
from __future__ import annotations

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def header_functions() -> list[str]:
    text = (ROOT / "include" / "pidb.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pidb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    names = header_functions()
    for must in ("pidb_pid_mean_partials", "pidb_pid_colsums", "pidb_member_masses",
                 "pidb_gram_i8", "pidb_gram_fixed_sums", "pidb_gram_f64", "pidb_depth_epilogue",
                 "pidb_eid_exact_epilogue", "pidb_pair_sums", "pidb_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2512_15187_b200 import _native as N

    lib = N.load()
    missing = [f for f in header_functions() if not hasattr(lib, f)]
    assert not missing, f"libpidb.so lacks {missing}"
    assert lib.pidb_abi_version() == 1


def test_ctypes_signatures_cover_the_header():
    from paper_2512_15187_b200 import _native as N

    assert set(header_functions()) <= set(N.SIGNATURES), \
        set(header_functions()) - set(N.SIGNATURES)


def test_library_is_sm100a_code():
    import subprocess

    from paper_2512_15187_b200 import _native as N

    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_workspace_query_needs_no_gpu():
    from paper_2512_15187_b200 import _native as N

    lib = N.load()
    assert lib.pidb_pid_mean_workspace_bytes(200, 1 << 20, N.PIDB_F32) > 0
    assert lib.pidb_pid_mean_workspace_bytes(100000, 10, N.PIDB_F32) > 0  # wide (two-read) path
    assert lib.pidb_pid_mean_workspace_bytes(0, 10, N.PIDB_F32) == 0  # empty ensemble
