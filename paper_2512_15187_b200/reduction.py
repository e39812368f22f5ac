"""Cell reductions that produce Gram matrices on the tensor cores.

Reference seam: gram_block (/root/reference/pkg/src/fuzzdepth/reduction.py:75-97),
the chunked ``rows . diag(w) . cols^T`` (or ``. (1 - cols)^T``) that
_pairwise_sums tiles over member blocks (depth.py:122-161).  Here one kernel
launch computes the whole symmetric N x N Gram of a resident ensemble:

* K1x ``pidb_gram_fixed``: fuzzy members as fixed-point base-256 digits,
  tcgen05 ``kind::i8`` MMAs with exact integer accumulation, fp64 result;
* K2 ``pidb_gram_i8``: 0/1 members packed to uint8 (K7), exact int64 result;
* ``pidb_gram_f64``: the array-level ``gram_block`` seam itself, fp64 on the
  CUDA cores (the reference's rtol 1e-12 contract).

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


def _aligned_bytes(nbytes: int, dev, align: int = 1024) -> torch.Tensor:
    """Uninitialised `align`-aligned uint8 device buffer (caching allocator)."""
    buf = torch.empty(nbytes + align, dtype=torch.uint8, device=dev)
    off = (-buf.data_ptr()) % align
    return buf[off:off + nbytes]


def pack_fixed(de: DeviceEnsemble, soft: torch.Tensor | None = None,
               mass: torch.Tensor | None = None):
    """K1x pack: members -> fixed-point digit tiles for the int8 Gram
    (pidb_fixed_pack).  Returns (q, wmax); `soft` (uint64-as-int64 (n,),
    zero-filled by the caller) receives the per-member soft-cell counts of
    the certifier's error bound, `mass` (fp64 (n,)) the member masses from
    the same pass.  The digit buffer (zero-filled once: rows
    past n stay zero) is kept on the ensemble and re-packed on every call
    (the members may change in place)."""
    q = _aligned_bytes(int(N.load().pidb_fixed_bytes(de.n, de.m)), de.device)
    wmax = de._cache.get("fixed_wmax")
    if wmax is None:
        wmax = float(de.weights.max()) if de.weights is not None else 1.0
        de._cache["fixed_wmax"] = wmax
    from .depth import _launch

    ws = None
    if mass is not None:
        ws = torch.empty(int(N.load().pidb_fixed_pack_workspace_bytes(de.n, de.m)),
                         dtype=torch.uint8, device=de.device)
    _launch("pidb_fixed_pack", de.ptr(), de.dtype_code, de.n, de.m, de.ld, de.wptr(), wmax,
            q.data_ptr(), None if soft is None else soft.data_ptr(),
            None if mass is None else mass.data_ptr(), None if ws is None else ws.data_ptr(),
            0 if ws is None else ws.numel(), stream_ptr(de.device))
    return q, wmax


def gram_device(de: DeviceEnsemble) -> torch.Tensor:
    """G[i, j] = sum_x w(x) u_i(x) u_j(x) as an (n, n) fp64 device tensor, from
    the fixed-point int8 tensor-core Gram (exact integer accumulation; error
    bound in include/pidb.h)."""
    lib = N.load()
    q, wmax = pack_fixed(de)
    g = torch.empty((de.n, de.n), dtype=torch.float64, device=de.device)
    ws = de.workspace(lib.pidb_gram_fixed_workspace_bytes(de.n, de.m, 0))
    from .depth import _launch

    _launch("pidb_gram_fixed", q.data_ptr(), de.n, de.m, wmax, g.data_ptr(),
            ws.data_ptr(), ws.numel(), stream_ptr(de.device))
    _allreduce(g, de)
    return g


def pack_binary(de: DeviceEnsemble, nonbinary: torch.Tensor | None = None) -> torch.Tensor:
    """K7: 0/1 members -> u8 tiles for K2 (include/pidb.h); optionally counts
    each member's values that are neither 0 nor 1 (`nonbinary`, int64 (n,)
    zero-filled by the caller).  The tile buffer comes from the stream-aware
    caching allocator per call (the pack writes every byte, padding included;
    inside a graph capture it becomes the graph's own)."""
    b = _aligned_bytes(int(N.load().pidb_binary_pack_bytes(de.n, de.m)), de.device)
    from .depth import _launch

    _launch("pidb_binary_pack", de.ptr(), de.dtype_code, de.n, de.m, de.ld, b.data_ptr(),
            None if nonbinary is None else nonbinary.data_ptr(), stream_ptr(de.device))
    return b


def intersection_gram(de: DeviceEnsemble, packed: torch.Tensor | None = None) -> torch.Tensor:
    """I[i, j] = |C_i ∩ C_j| exactly (int64), via K7 + K2 (K2 alone on a
    byte ensemble, whose members it loads by TMA)."""
    lib = N.load()
    g = torch.empty((de.n, de.n), dtype=torch.int64, device=de.device)
    ws = de.workspace(lib.pidb_gram_i8_workspace_bytes(de.n, de.m))
    from .depth import _launch

    if de.is_bits and packed is None:
        _launch("pidb_gram_i8_bytes", de.ptr(), de.n, de.m, de.ld, g.data_ptr(), ws.data_ptr(),
                ws.numel(), stream_ptr(de.device))
    else:
        b = pack_binary(de) if packed is None else packed
        _launch("pidb_gram_i8", b.data_ptr(), de.n, de.m, g.data_ptr(), ws.data_ptr(),
                ws.numel(), stream_ptr(de.device))
    _allreduce(g, de)
    return g


_EXACT_F32 = (np.float32, np.float16, np.bool_, np.uint8, np.int8, np.uint16, np.int16)


def _block_to_device(a, dt, dev) -> torch.Tensor:
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
    return t.to(device=dev, dtype=dt).contiguous()


def gram_block(rows, cols, weights=None, complement_cols: bool = False) -> np.ndarray:
    """Array-level drop-in for gram_block (reduction.py:75-97), in fp64.

    rows (n_r, cells) and cols (n_c, cells) of any real dtype; returns the
    float64 (n_r, n_c) block ``rows . diag(w) . cols^T`` (or ``. (1 - cols)^T``)
    with fp64 products and sums on the CUDA cores (``pidb_gram_f64``), the
    reference's accuracy contract (rtol 1e-12 in its tests).  Float32-exact
    inputs are read as float32 and widened in the kernel; anything else goes
    over as float64.  The depth methods never call this: their Grams are the
    tensor-core kernels (``fixed_gram`` / ``intersection_gram``) or the
    factorised sums."""
    from .device import require_cuda
    from .depth import _launch

    rows = rows if isinstance(rows, torch.Tensor) else np.asarray(rows)
    cols = cols if isinstance(cols, torch.Tensor) else np.asarray(cols)
    if rows.ndim != 2 or cols.ndim != 2 or rows.shape[1] != cols.shape[1]:
        raise ValidationError("rows and cols must be (n, cells) with equal cells")
    nr, m = int(rows.shape[0]), int(rows.shape[1])
    nc = int(cols.shape[0])
    if nr == 0 or nc == 0 or m == 0:
        return np.zeros((nr, nc), dtype=np.float64)
    dev = require_cuda()

    def exact32(a):  # values exactly representable in float32
        if isinstance(a, torch.Tensor):
            return a.dtype in (torch.float32, torch.float16, torch.bfloat16, torch.bool,
                               torch.uint8, torch.int8, torch.int16)
        return any(a.dtype == np.dtype(t) for t in _EXACT_F32)

    f32 = exact32(rows) and exact32(cols)
    dt = torch.float32 if f32 else torch.float64
    r = _block_to_device(rows, dt, dev)
    c = _block_to_device(cols, dt, dev)
    w = None
    if weights is not None:
        wh = np.ascontiguousarray(weights, dtype=np.float64).reshape(-1)
        if wh.shape[0] != m:
            raise ValidationError(f"weights shape {wh.shape} does not match cell count {m}")
        w = torch.from_numpy(wh).to(dev)
    out = torch.empty((nr, nc), dtype=torch.float64, device=dev)
    lib = N.load()
    ws = torch.empty(max(1, lib.pidb_gram_f64_workspace_bytes(nr, nc, m)), dtype=torch.uint8,
                     device=dev)
    _launch("pidb_gram_f64", r.data_ptr(), c.data_ptr(), N.PIDB_F32 if f32 else N.PIDB_F64,
            nr, nc, m, m, m, None if w is None else w.data_ptr(), int(bool(complement_cols)),
            out.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr(dev))
    return out.cpu().numpy()


# ------------------------------------------------- reduction-module seams
# reduction.py:30-72, 100-127: the chunked host reductions the reference's
# depth code is built from.  Here they run on the device through the K8 pair
# kernel (one fused pass, fp64 accumulation); chunk_bounds / run_tasks keep
# the reference's host contract for callers that iterate themselves.


def chunk_bounds(n_cells: int):
    """(start, stop) spans of CHUNK_CELLS cells covering [0, n_cells) in
    ascending order (reduction.py:30-33)."""
    start = 0
    while start < n_cells:
        stop = min(n_cells, start + CHUNK_CELLS)
        yield start, stop
        start = stop


def _pair_sums(a, b, weights, op):
    from .inclusion import _pair

    return _pair(a, a if b is None else b, weights, op)


def weighted_sum(values, weights=None) -> float:
    """sum_x w(x) v(x) in fp64 (reduction.py:36-44), one device pass."""
    from . import _native as _N

    return _pair_sums(values, None, weights, _N.PIDB_OP_INCLUSION)[1]


def weighted_inner(a, b, weights=None) -> float:
    """sum_x w a b in fp64 (reduction.py:47-57), one device pass."""
    from . import _native as _N

    return _pair_sums(a, b, weights, _N.PIDB_OP_INCLUSION)[0]


def weighted_excess(a, b, weights=None) -> float:
    """sum_x w a (1 - b) = sum w a - sum w a b (reduction.py:60-72)."""
    from . import _native as _N

    inner, mass = _pair_sums(a, b, weights, _N.PIDB_OP_INCLUSION)
    return mass - inner


def run_tasks(fn, items, workers: int) -> list:
    """Results of fn over items in input order (reduction.py:115-127); a
    thread pool when workers > 1 (the device calls release the GIL)."""
    todo = list(items)
    if workers > 1 and len(todo) > 1:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=workers) as ex:
            return list(ex.map(fn, todo))
    return [fn(x) for x in todo]


def resolve_workers(workers: int | None = None) -> int:
    """reduction.py:100-112 (the device kernels ignore the count)."""
    from .depth import resolve_workers as _rw

    return _rw(workers)
