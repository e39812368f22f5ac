"""ctypes binding of the C ABI in include/pidb.h (libpidb.so, sm_100a).

This is the binding a reference maintainer would add to route fuzzdepth's
hot path to the B200 kernels.  There is deliberately no CPU
fallback: if the library or a CUDA device is missing, every entry point
raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import ValidationError

# PIDB_LIB selects another build of the same ABI (e.g. libpidb_checked.so,
# the device-bounds-checked build of tools/checked_sweep.sh)
LIB_PATH = Path(os.environ.get("PIDB_LIB") or Path(__file__).resolve().parent / "libpidb.so")

PIDB_OK = 0
PIDB_EINVAL = -1
PIDB_ECUDA = -2
PIDB_EUNSUPPORTED = -3
PIDB_EWORKSPACE = -4

PIDB_F32 = 0
PIDB_F64 = 1
PIDB_U8 = 2
PIDB_EPI_PID_MEAN = 0
PIDB_EPI_PID = 1
PIDB_EPI_DICE = 2
PIDB_EPI_IOU = 3
PIDB_OP_INCLUSION = 0
PIDB_OP_SUBSET = 1
PIDB_OP_MINMAX = 2


class NativeError(RuntimeError):
    """CUDA / launch failure inside libpidb (not an input-validation error)."""


_p = C.c_void_p
_i64 = C.c_int64
_int = C.c_int
_dbl = C.c_double
_sz = C.c_size_t

# name -> (restype, argtypes); mirrors include/pidb.h one to one.
SIGNATURES: dict[str, tuple] = {
    "pidb_abi_version": (_int, []),
    "pidb_last_error": (C.c_char_p, []),
    "pidb_pid_mean_workspace_bytes": (_sz, [_i64, _i64, _int]),
    "pidb_pid_mean_partials": (_int, [_p, _int, _i64, _i64, _i64, _p, _p, _p, _p, _p, _sz, _p]),
    "pidb_similarity_partials": (_int, [_p, _int, _i64, _i64, _i64, _p, _p, _p, _p, _p, _sz, _p]),
    "pidb_pid_colsums": (_int, [_p, _int, _i64, _i64, _i64, _p, _p, _p, _p, _sz, _p]),
    "pidb_member_masses": (_int, [_p, _int, _i64, _i64, _i64, _p, _p, _p, _p, _sz, _p]),
    "pidb_binary_pack_bytes": (_sz, [_i64, _i64]),
    "pidb_binary_pack": (_int, [_p, _int, _i64, _i64, _i64, _p, _p, _p]),
    "pidb_gram_i8_workspace_bytes": (_sz, [_i64, _i64]),
    "pidb_gram_i8": (_int, [_p, _i64, _i64, _p, _p, _sz, _p]),
    "pidb_gram_i8_bytes": (_int, [_p, _i64, _i64, _i64, _p, _p, _sz, _p]),
    "pidb_gram_reduce": (_int, [_p, _i64, _p, _p, _p, _p]),
    "pidb_fixed_bytes": (_sz, [_i64, _i64]),
    "pidb_fixed_pack_workspace_bytes": (_sz, [_i64, _i64]),
    "pidb_fixed_pack": (_int, [_p, _int, _i64, _i64, _i64, _p, _dbl, _p, _p, _p, _p, _sz, _p]),
    "pidb_gram_fixed_workspace_bytes": (_sz, [_i64, _i64, _int]),
    "pidb_gram_fixed": (_int, [_p, _i64, _i64, _dbl, _p, _p, _sz, _p]),
    "pidb_gram_fixed_sums": (_int, [_p, _i64, _i64, _dbl, _p, _p, _p, _p, _sz, _p]),
    "pidb_gram_f64_workspace_bytes": (_sz, [_i64, _i64, _i64]),
    "pidb_gram_f64": (_int, [_p, _p, _int, _i64, _i64, _i64, _i64, _i64, _p, _int, _p, _p, _sz,
                             _p]),
    "pidb_depth_epilogue": (_int, [_int, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "pidb_inverse_masses": (_int, [_i64, _p, _p, _p]),
    "pidb_eid_exact_epilogue": (_int, [_p, _i64, _p, _p, _p, _p, _p, _p]),
    "pidb_eid_factorized_epilogue": (
        _int,
        [_i64, _p, _p, _p, _dbl, _p, _p, _p, _p, _p, _p],
    ),
    "pidb_ranks": (_int, [_i64, _p, _p, _p]),
    "pidb_pair_sums": (_int, [_p, _p, _int, _i64, _p, _int, _p, _p, _sz, _p]),
    "pidb_mean_mask": (_int, [_p, _int, _i64, _i64, _i64, _p, _p]),
    "pidb_copy_rows": (_int, [_p, _i64, _p, _i64, _i64, _i64, _p]),
    "pidb_validate": (_int, [_p, _int, _i64, _i64, _i64, _int, _p, _p]),
    "pidb_sum_rows": (_int, [_p, _i64, _i64, _p, _p]),
    "pidb_synth_ellipsoids": (_int, [_p, _i64, _i64, _i64, _p, _dbl, _p]),
    "pidb_synth_disks": (_int, [_p, _i64, _i64, _i64, _p, _dbl, _p]),
    "pidb_band_envelopes": (_int, [_p, _int, _i64, _i64, _i64, _p, _i64, _dbl, _p, _int, _p, _p,
                                   _p]),
}

_lib = None
_lock = threading.Lock()


def load(path: Path | str | None = None) -> C.CDLL:
    """Load libpidb.so (once) and attach the C signatures."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise ImportError(
                f"{p} is missing: build the sm_100a kernels first "
                "(python -m paper_2512_15187_b200._build); there is no CPU fallback"
            )
        lib = C.CDLL(str(p))
        missing = []
        for name, (res, args) in SIGNATURES.items():
            try:
                fn = getattr(lib, name)
            except AttributeError:
                missing.append(name)
                continue
            fn.restype = res
            fn.argtypes = args
        if missing:
            raise ImportError(f"{p} lacks symbols {missing}")
        if lib.pidb_abi_version() != 1:
            raise ImportError("libpidb ABI version mismatch")
        _lib = lib
        return lib


def has_symbol(name: str) -> bool:
    lib = load()
    try:
        getattr(lib, name)
        return True
    except AttributeError:
        return False


def check(rc: int, what: str) -> None:
    """Map a pidb status code to the reference's exception types."""
    if rc == PIDB_OK:
        return
    msg = (load().pidb_last_error() or b"").decode(errors="replace")
    if rc in (PIDB_EINVAL, PIDB_EUNSUPPORTED):
        raise ValidationError(f"{what}: {msg}")
    raise NativeError(f"{what} failed ({rc}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
