"""Device residency: ensembles as one row-major (n, ld) matrix in HBM.

Replaces the reference's per-member access (Ensemble.member / block_values,
/root/reference/pkg/src/fuzzdepth/grid.py:196-213) on the hot path: members
are uploaded once through pinned, double-buffered host staging and every
depth kernel then streams the resident matrix.

Layout: row i = member i, ``ld`` = cells rounded up to 32 elements (128-byte
rows, TMA-aligned), zero padding.  float32 storage unless a member is float64
(the reference's dtype policy, grid.py:103-104), in which case the whole matrix
is float64.  A bool / uint8 tensor is staged as a byte ensemble (0/1 members,
one byte per cell, checked once here like BinaryMask, grid.py:145-148): eID
reads it directly (no pack pass, a quarter of the fp32 bytes); every other
method sees its cached float32 view (``prob()``, binarize(...).to_prob()).  A sharded ensemble holds a contiguous cell slab [lo, hi) of every
member on each rank (multi-GPU voxel sharding).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from . import _native as N
from .errors import DegenerateEnsembleError, GridMismatchError, ValidationError
from .grid import VALUE_TOLERANCE, GridSpec

_ROW_ALIGN = 32  # elements; 128-byte rows for fp32
_STAGE_BYTES = 64 << 20


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "no CUDA device: the B200 depth path has no CPU fallback"
        )
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if dev.type != "cuda":
        raise ValidationError(f"device must be a CUDA device, got {dev}")
    return dev


def padded_ld(m: int) -> int:
    return (m + _ROW_ALIGN - 1) // _ROW_ALIGN * _ROW_ALIGN


def shard_bounds(m: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced cell slab of rank `rank` out of `world`."""
    base, extra = divmod(m, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclass
class DeviceEnsemble:
    values: torch.Tensor                 # (n, ld) float32/float64 (or 0/1 uint8) on a CUDA device
    m: int                               # cells held here (shard-local)
    dims: tuple[int, ...]
    ids: tuple[str, ...]
    weights: torch.Tensor | None = None  # (m,) float64, shard-local
    weights_host: np.ndarray | None = None  # full-grid weights (GridSpec parity)
    process_group: object | None = None  # torch.distributed group when sharded
    cell_range: tuple[int, int] | None = None
    _cache: dict = field(default_factory=dict, repr=False)

    # ------------------------------------------------------------ properties
    @property
    def n(self) -> int:
        return int(self.values.shape[0])

    @property
    def ld(self) -> int:
        return int(self.values.stride(0))

    @property
    def device(self) -> torch.device:
        return self.values.device

    @property
    def dtype_code(self) -> int:
        if self.values.dtype == torch.uint8:
            return N.PIDB_U8
        return N.PIDB_F64 if self.values.dtype == torch.float64 else N.PIDB_F32

    @property
    def is_bits(self) -> bool:
        """0/1 members stored one byte per cell (a binary ensemble)."""
        return self.values.dtype == torch.uint8

    def prob(self) -> "DeviceEnsemble":
        """The float32 ensemble of a byte ensemble (binarize(...).to_prob(),
        grid.py:152-153, 271-277), widened on the device once and cached
        (4 bytes per cell next to the 1-byte matrix; in-place edits of the
        bytes after the first call are not seen by it: restage instead);
        ``self`` for a float ensemble."""
        if not self.is_bits:
            return self
        p = self._cache.get("prob")
        if p is None:
            p = DeviceEnsemble(self.values.to(torch.float32), self.m, self.dims, self.ids,
                               self.weights, self.weights_host, self.process_group,
                               self.cell_range)
            self._cache["prob"] = p
        return p

    @property
    def grid(self) -> GridSpec:
        return GridSpec(self.dims, self.weights_host)

    @property
    def sharded(self) -> bool:
        return self.process_group is not None

    def __len__(self) -> int:
        return self.n

    def ptr(self) -> int:
        return self.values.data_ptr()

    def wptr(self) -> int | None:
        return None if self.weights is None else self.weights.data_ptr()

    # ---------------------------------------------------------- construction
    @classmethod
    def from_tensor(
        cls,
        values: torch.Tensor,
        weights=None,
        ids: Sequence[str] | None = None,
        dims: Sequence[int] | None = None,
        validate: bool = True,
        device=None,
        process_group=None,
        cell_range: tuple[int, int] | None = None,
    ) -> "DeviceEnsemble":
        """Stage an (n, *dims) tensor or array (host or device).

        For a multi-GPU job pass this rank's cell slab (n, hi - lo) together
        with ``process_group`` and ``cell_range=(lo, hi)``; ``dims`` then names
        the full grid and ``weights`` the slab's weights."""
        if isinstance(values, np.ndarray):
            values = torch.from_numpy(values)
        if values.dim() < 2:
            raise ValidationError("member tensor must be (n, *dims)")
        n = int(values.shape[0])
        if n == 0:
            raise DegenerateEnsembleError("ensemble needs at least one member")
        dims = tuple(int(d) for d in (dims if dims is not None else values.shape[1:]))
        m = int(np.prod(dims)) if cell_range is None else cell_range[1] - cell_range[0]
        if int(np.prod(values.shape[1:])) != m:
            raise ValidationError(f"member tensor has {values[0].numel()} cells, grid expects {m}")
        cr = (0, m) if cell_range is None else tuple(cell_range)
        dev = require_cuda(device if device is not None else
                           (values.device if values.is_cuda else None))
        dt = torch.float64 if values.dtype == torch.float64 else torch.float32
        ids = _make_ids(ids, n)
        w_host, w_dev = _weights(weights, m, dev)
        flat = values.reshape(n, m)
        if flat.dtype in (torch.bool, torch.uint8):  # byte ensemble
            src = flat if flat.dtype == torch.uint8 else flat.view(torch.uint8)
            de = cls(_copy_padded(src, torch.uint8, dev), m, dims, ids, w_dev, w_host,
                     process_group, cr)
            if validate and flat.dtype == torch.uint8:
                _check_bits(de)
            return de
        es = 8 if dt == torch.float64 else 4
        if (flat.is_cuda and flat.device == dev and flat.dtype == dt and flat.stride(1) == 1
                and (flat.stride(0) * es) % 16 == 0 and flat.data_ptr() % 16 == 0):
            # zero-copy: the caller's device tensor already has a TMA-legal layout
            de = cls(flat.as_strided((n, flat.stride(0)), (flat.stride(0), 1)), m, dims, ids,
                     w_dev, w_host, process_group, cr)
            if validate and _validate(de, clamp=False):
                de = cls(_copy_padded(flat, dt, dev), m, dims, ids, w_dev, w_host, process_group, cr)
                _validate(de, clamp=True)
            return de
        if flat.dtype != dt:
            flat = flat.to(dt)
        de = cls(_copy_padded(flat, dt, dev), m, dims, ids, w_dev, w_host, process_group, cr)
        if validate:
            _validate(de, clamp=True)
        return de

    @classmethod
    def from_masks(cls, masks: Sequence, ids=None, device=None) -> "DeviceEnsemble":
        grid = masks[0].grid
        for mk in masks[1:]:
            grid.require_same(mk.grid)
        arr = np.stack([np.asarray(mk.values) for mk in masks])
        arr = arr if arr.dtype == np.float64 else arr.astype(np.float32, copy=False)
        return cls.from_tensor(torch.from_numpy(arr), grid.weights, ids,
                               tuple(grid.dims), validate=False, device=device)

    # reference Ensemble duck-typing (grid.py:194-212): host copies of members
    def member(self, i: int):
        from .grid import ProbMask

        if self.sharded:
            raise ValidationError("a sharded ensemble holds only this rank's cells")
        return ProbMask(self.grid, self._host_rows(i, i + 1)[0])

    def __iter__(self):
        return (self.member(i) for i in range(self.n))

    def block_values(self, lo: int, hi: int) -> np.ndarray:
        return self._host_rows(lo, hi)

    def _host_rows(self, lo: int, hi: int) -> np.ndarray:
        rows = self.values[lo:hi, :self.m]
        # a byte ensemble widens just these rows (not the cached full view)
        return (rows.to(torch.float32) if self.is_bits else rows).cpu().numpy()

    def subset(self, indices: Sequence[int]) -> "DeviceEnsemble":
        """Members ``indices`` in the given order (grid.py Ensemble.subset);
        one device-side row gather, same grid and weights."""
        idx = torch.as_tensor(list(indices), dtype=torch.int64, device=self.device)
        if idx.numel() == 0:
            raise DegenerateEnsembleError("ensemble needs at least one member")
        return DeviceEnsemble(self.values.index_select(0, idx).contiguous(), self.m, self.dims,
                              tuple(self.ids[int(i)] for i in indices), self.weights,
                              self.weights_host, process_group=self.process_group,
                              cell_range=self.cell_range)

    # ------------------------------------------------------------- helpers
    def workspace(self, nbytes: int) -> torch.Tensor:
        """Zero-initialised per-device workspace (the kernels leave their
        completion counters at zero on exit, so it is reused as is)."""
        if torch.cuda.is_current_stream_capturing():
            # a graph gets its own workspace (alive as long as this ensemble's
            # graphs): capture streams come from a pool, so a stream-keyed
            # one could end up shared by graphs replayed on different streams.
            # Zeroed once after the capture (depth._graphed), not per replay.
            ws = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=self.device)
            self._cache.setdefault("graph_ws_pending", []).append(ws)
            return ws
        key = ("ws", self.device, torch.cuda.current_stream(self.device).cuda_stream)
        ws = _WS.get(key)
        if ws is None or ws.numel() < nbytes:
            ws = torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device=self.device)
            _WS[key] = ws
        return ws

    def mean_values(self) -> torch.Tensor:
        de = self.prob()
        out = torch.empty(de.m, dtype=torch.float64, device=de.device)
        N.call("pidb_mean_mask", de.ptr(), de.dtype_code, de.n, de.m, de.ld,
               out.data_ptr(), stream_ptr(de.device))
        return out


_WS: dict = {}


def stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _make_ids(ids, n):
    ids = tuple(str(s) for s in (ids if ids is not None else (f"member_{i:04d}" for i in range(n))))
    if len(ids) != n:
        raise ValidationError(f"{len(ids)} ids for {n} members")
    if len(set(ids)) != n:
        raise ValidationError("member ids must be unique")
    return ids


def _weights(weights, m, dev, lo: int = 0, hi: int | None = None):
    if weights is None:
        return None, None
    if isinstance(weights, torch.Tensor):
        w_host = weights.detach().cpu().numpy().astype(np.float64)
    else:
        w_host = np.ascontiguousarray(weights, dtype=np.float64)
    hi = w_host.shape[0] if hi is None else hi
    if w_host.ndim != 1 or hi - lo != m:
        raise ValidationError(f"weights shape {w_host.shape} does not match cell count {m}")
    if not np.isfinite(w_host).all() or (w_host <= 0).any():
        raise ValidationError("cell weights must be finite and positive")
    w_dev = torch.tensor(w_host[lo:hi], dtype=torch.float64, device=dev)
    return w_host, w_dev


def _copy_padded(flat: torch.Tensor, dt, dev) -> torch.Tensor:
    """(n, m) tensor (host or device) -> zero-padded (n, ld) device matrix,
    one pitched copy (pidb_copy_rows)."""
    n, m = flat.shape
    ld = padded_ld(m)
    out = torch.empty((n, ld), dtype=dt, device=dev)
    if ld > m:
        out[:, m:].zero_()
    src = flat if flat.stride(1) == 1 else flat.contiguous()
    es = out.element_size()
    N.call("pidb_copy_rows", out.data_ptr(), ld * es, src.data_ptr(), src.stride(0) * es,
           m * es, n, stream_ptr(dev))
    if not src.is_cuda and not src.is_pinned():
        torch.cuda.current_stream(dev).synchronize()  # pageable source must outlive the copy
    return out


def _nonbinary_counts(de: "DeviceEnsemble") -> np.ndarray:
    """Per-member count of bytes other than 0/1 in a byte ensemble (K7 in
    count-only mode)."""
    bad = torch.zeros(de.n, dtype=torch.int64, device=de.device)
    N.call("pidb_binary_pack", de.ptr(), N.PIDB_U8, de.n, de.m, de.ld, None, bad.data_ptr(),
           stream_ptr(de.device))
    return bad.cpu().numpy()


def _check_bits(de: "DeviceEnsemble") -> None:
    """BinaryMask's value check (grid.py:145-148) on a byte ensemble."""
    if _nonbinary_counts(de).any():
        raise ValidationError("binary mask values must be 0 or 1")


def _key_to_double(k: int) -> float:
    import struct

    b = k if k >= 0 else k ^ 0x7FFFFFFFFFFFFFFF
    return struct.unpack("<d", struct.pack("<q", b))[0]


def _validate(de: "DeviceEnsemble", clamp: bool) -> bool:
    """ProbMask value policy (grid.py:105-116) on the device.  Raises for
    non-finite or out-of-tolerance values; returns True when values needed
    clipping (done in place when ``clamp``)."""
    stats = torch.empty(3, dtype=torch.int64, device=de.device)
    N.call("pidb_validate", de.ptr(), de.dtype_code, de.n, de.m, de.ld, int(clamp),
           stats.data_ptr(), stream_ptr(de.device))
    nf, kmin, kmax = (int(v) for v in stats.cpu().tolist())
    if nf:
        raise ValidationError("mask values must be finite")
    lo, hi = _key_to_double(kmin), _key_to_double(kmax)
    if lo < -VALUE_TOLERANCE or hi > 1.0 + VALUE_TOLERANCE:
        raise ValidationError(f"mask values outside [0, 1]: min={lo!r} max={hi!r}")
    return lo < 0.0 or hi > 1.0


class _PinnedRing:
    """Two pinned host slots; H2D copies overlap the host-side member loads."""

    def __init__(self, slot_elems: int, dtype: torch.dtype):
        self.slots = [torch.empty(slot_elems, dtype=dtype, pin_memory=True) for _ in range(2)]
        self.events: list[torch.cuda.Event | None] = [None, None]
        self.k = 0

    def next(self) -> tuple[torch.Tensor, int]:
        k = self.k
        self.k ^= 1
        ev = self.events[k]
        if ev is not None:
            ev.synchronize()
        return self.slots[k], k

    def mark(self, k: int, stream) -> None:
        ev = torch.cuda.Event()
        ev.record(stream)
        self.events[k] = ev


def stage(ensemble, device=None, shard: tuple[int, int] | None = None,
          process_group=None) -> DeviceEnsemble:
    """Bring an ensemble into HBM (no-op for an already staged one).

    Accepts a DeviceEnsemble, an (n, *dims) torch tensor / numpy array, or any
    reference-style Ensemble (``grid``, ``ids``, ``len``, ``member(i)``;
    lazy loaders are resolved one member at a time, grid.py:196-202).
    ``shard=(rank, world)`` keeps only this rank's contiguous cell slab.
    A bool / uint8 tensor becomes a byte ensemble; the methods other than
    depth_eid read its float32 view (``stage(x).prob()``).
    """
    if isinstance(ensemble, DeviceEnsemble):
        return ensemble
    if isinstance(ensemble, (torch.Tensor, np.ndarray)):
        return DeviceEnsemble.from_tensor(ensemble, device=device)
    dev = require_cuda(device)
    n = len(ensemble)
    if n == 0:
        raise DegenerateEnsembleError("ensemble needs at least one member")
    grid = ensemble.grid
    dims = tuple(int(d) for d in grid.dims)
    m_full = int(np.prod(dims))
    lo, hi = (0, m_full) if shard is None else shard_bounds(m_full, *shard)
    m = hi - lo
    ld = padded_ld(m)
    first = np.asarray(ensemble.member(0).values)
    dt = torch.float64 if first.dtype == np.float64 else torch.float32
    out = torch.zeros((n, ld), dtype=dt, device=dev)
    s = torch.cuda.current_stream(dev)
    per_slot = max(1, _STAGE_BYTES // max(1, m * out.element_size()))
    ring = _PinnedRing(per_slot * m, dt)
    i = 0
    vals0 = first
    while i < n:
        slot, k = ring.next()
        cnt = min(per_slot, n - i)
        host = slot.numpy()
        promote = False
        for j in range(cnt):
            v = vals0 if i + j == 0 else np.asarray(ensemble.member(i + j).values)
            if v.shape != (m_full,):
                v = v.reshape(-1)
                if v.shape != (m_full,):
                    raise GridMismatchError(f"member {i + j} has {v.size} cells, grid expects {m_full}")
            if v.dtype == np.float64 and dt == torch.float32:
                promote = True
                cnt = j
                break
            host[j * m:(j + 1) * m] = v[lo:hi]
        if cnt:
            out[i:i + cnt, :m].copy_(slot[:cnt * m].view(cnt, m), non_blocking=True)
            ring.mark(k, s)
        i += cnt
        if promote:  # a float64 member appeared: keep full precision from here on
            torch.cuda.current_stream(dev).synchronize()
            out = out.double()
            dt = torch.float64
            ring = _PinnedRing(per_slot * m, dt)
    w_host, w_dev = _weights(grid.weights, m, dev, lo, hi)
    de = DeviceEnsemble(out, m, dims, tuple(str(x) for x in ensemble.ids), w_dev, w_host,
                        process_group=process_group if shard is not None else None,
                        cell_range=(lo, hi))
    return de
