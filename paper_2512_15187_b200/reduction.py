"""Cell reductions that produce Gram matrices on the tensor cores.

Reference seam: gram_block (/root/reference/pkg/src/fuzzdepth/reduction.py:75-97),
the chunked ``rows . diag(w) . cols^T`` (or ``. (1 - cols)^T``) that
_pairwise_sums tiles over member blocks (depth.py:122-161).  Here one kernel
launch computes the whole symmetric N x N Gram of a resident ensemble:

* K1 ``pidb_gram_tf32x3``: fuzzy members, 3xTF32 tcgen05 MMAs, fp64 result;
* K2 ``pidb_gram_i8``: 0/1 members packed to uint8 (K7), exact int64 result.

Per-shard Grams are summed across GPUs with one NCCL allreduce.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .device import DeviceEnsemble, stage, stream_ptr
from .errors import ValidationError

CHUNK_CELLS = 65536  # reduction.py:22 (API parity; the device kernels tile differently)
WORKERS_ENV_VAR = "FUZZDEPTH_WORKERS"


def _allreduce(t: torch.Tensor, de: DeviceEnsemble) -> None:
    if de.process_group is None:
        return
    import torch.distributed as dist

    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=de.process_group)


def gram_device(de: DeviceEnsemble) -> torch.Tensor:
    """G[i, j] = sum_x w(x) u_i(x) u_j(x) as an (n, n) fp64 device tensor."""
    if de.dtype_code != N.PIDB_F32:
        raise ValidationError("the tensor-core Gram takes float32 members")
    lib = N.load()
    g = torch.empty((de.n, de.n), dtype=torch.float64, device=de.device)
    wsb = lib.pidb_gram_tf32x3_workspace_bytes(de.n, de.m)
    ws = de.workspace(wsb)
    from .depth import _launch

    _launch("pidb_gram_tf32x3", de.ptr(), de.n, de.m, de.ld, de.wptr(), g.data_ptr(),
           ws.data_ptr(), ws.numel(), stream_ptr(de.device))
    _allreduce(g, de)
    return g


def pack_binary(de: DeviceEnsemble, nonbinary: torch.Tensor | None = None) -> torch.Tensor:
    """K7: 0/1 members -> uint8 rows (row stride a multiple of 128 bytes);
    optionally counts each member's values that are neither 0 nor 1
    (`nonbinary`, int64 (n,) zero-filled by the caller)."""
    ldb = (de.m + 127) // 128 * 128
    b = torch.empty((de.n, ldb), dtype=torch.uint8, device=de.device)
    from .depth import _launch

    _launch("pidb_binary_pack", de.ptr(), de.dtype_code, de.n, de.m, de.ld, b.data_ptr(), ldb,
            None if nonbinary is None else nonbinary.data_ptr(), stream_ptr(de.device))
    return b


def intersection_gram(de: DeviceEnsemble, packed: torch.Tensor | None = None) -> torch.Tensor:
    """I[i, j] = |C_i ∩ C_j| exactly (int64), via K7 + K2."""
    lib = N.load()
    b = pack_binary(de) if packed is None else packed
    g = torch.empty((de.n, de.n), dtype=torch.int64, device=de.device)
    ws = de.workspace(lib.pidb_gram_i8_workspace_bytes(de.n, de.m))
    from .depth import _launch

    _launch("pidb_gram_i8", b.data_ptr(), de.n, de.m, b.stride(0), g.data_ptr(),
           ws.data_ptr(), ws.numel(), stream_ptr(de.device))
    _allreduce(g, de)
    return g


def gram_block(rows, cols, weights=None, complement_cols: bool = False) -> np.ndarray:
    """Array-level mirror of reduction.py:75-97 on the tensor cores.

    rows (n_r, cells) and cols (n_c, cells); returns float64 (n_r, n_c).
    The Gram of the stacked [rows; cols] block is formed once and sliced.
    """
    rows = np.asarray(rows)
    cols = np.asarray(cols)
    if rows.ndim != 2 or cols.ndim != 2 or rows.shape[1] != cols.shape[1]:
        raise ValidationError("rows and cols must be (n, cells) with equal cells")
    right = (1.0 - cols.astype(np.float64)) if complement_cols else cols
    stacked = np.concatenate([rows.astype(np.float32), np.asarray(right, dtype=np.float32)])
    de = DeviceEnsemble.from_tensor(torch.from_numpy(stacked), weights=weights, validate=False)
    g = gram_device(de).cpu().numpy()
    nr = rows.shape[0]
    return g[:nr, nr:].copy()
