"""Drop-in depth methods (eID, exact PID, PID-mean) on the B200 kernels.

Same names, signatures, results and errors as the reference module
/root/reference/pkg/src/fuzzdepth/depth.py; the arithmetic runs in libpidb:

  depth_pid_mean  (depth.py:246-287) -> K5 single HBM pass + K4 epilogue
  depth_pid       (depth.py:213-228) -> K1x fixed-point tcgen05 Gram + K4, or the
                                        exact O(N*M) factorisation K5 + K9
  depth_eid       (depth.py:192-210) -> K6/K7 binary check + pack, K2 exact
                                        integer Gram (tcgen05 kind::i8) + exact
                                        epilogue (bit-identical to ref_eid)

Every function accepts a reference-style Ensemble (host members, staged into
HBM once), a ``DeviceEnsemble`` (already resident; optionally a cell shard of
a multi-GPU job, combined with one NCCL allreduce), or an (n, *dims) tensor.
``workers`` is accepted and validated for signature compatibility; device
results do not depend on it (the reference guarantees worker-count
invariance, reduction.py:115-127).
"""
from __future__ import annotations

import os
import threading
import time
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .device import DeviceEnsemble, stage, stream_ptr
from .errors import DegenerateEnsembleError, ValidationError

CV_WARN_THRESHOLD = 0.5          # depth.py:40
METHOD_NAMES = ("eid", "pid", "pid-mean", "dice", "iou")  # depth.py:42
PID_ALGORITHMS = ("auto", "gram", "factorized")


@dataclass(frozen=True)
class DepthResult:
    """Per-member depths and ranks (depth.py:45-77); arrays are read-only."""

    ids: tuple[str, ...]
    in_in: np.ndarray
    in_out: np.ndarray
    depth: np.ndarray
    rank: np.ndarray
    method: str
    cv_mass: float
    elapsed_seconds: float

    def __post_init__(self) -> None:
        n = len(self.ids)
        for name in ("in_in", "in_out", "depth", "rank"):
            a = getattr(self, name)
            if a.shape != (n,):
                raise ValidationError(f"{name} must have one entry per member")
            a.flags.writeable = False

    def __len__(self) -> int:
        return len(self.ids)

    def ordered_ids(self) -> list[str]:
        order = np.empty(len(self), dtype=np.int64)
        order[self.rank] = np.arange(len(self))
        return [self.ids[i] for i in order]


def ranks_from_depths(depth: np.ndarray) -> np.ndarray:
    """Ranks, 0 = deepest, ties by ascending index (depth.py:80-85).  Host
    helper for API parity; the depth functions rank on the device (K4)."""
    order = np.argsort(-np.asarray(depth), kind="stable")
    rank = np.empty(order.shape[0], dtype=np.int64)
    rank[order] = np.arange(order.shape[0])
    return rank


def mass_cv(masses: np.ndarray) -> float:
    """Population std / mean of member masses (depth.py:105-110).  The same
    two-pass arithmetic as np.std (pairwise mean, then the mean square
    deviation) without its per-call overhead (~20 us on small ensembles)."""
    m = np.asarray(masses, dtype=np.float64)
    n = m.shape[0]
    mean = float(m.sum()) / n
    if mean == 0.0:
        return 0.0
    d = m - mean
    return float(np.sqrt(float(np.dot(d, d)) / n) / mean)


def resolve_workers(workers: int | None = None) -> int:
    """Same contract as reduction.py:100-112 (kept for signature parity)."""
    if workers is not None:
        if workers < 1:
            raise ValueError("workers must be >= 1")
        return int(workers)
    env = os.environ.get("FUZZDEPTH_WORKERS")
    if env:
        try:
            return max(1, int(env))
        except ValueError:
            pass
    return _CPU_COUNT


_CPU_COUNT = os.cpu_count() or 1


# --------------------------------------------------------------- primitives

# Optional per-kernel CUDA-event log used by bench.py: when a list, every
# hot-kernel launch appends (name, start_event, end_event) recorded on the
# launching stream.
KERNEL_EVENTS: list | None = None


def _launch(name: str, *args) -> None:
    if KERNEL_EVENTS is None:
        N.call(name, *args)
        return
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    N.call(name, *args)
    b.record()
    KERNEL_EVENTS.append((name, a, b))



# CUDA graphs for repeated calls on one DeviceEnsemble (PIDB_GRAPHS=0: off)
_GRAPHS = os.environ.get("PIDB_GRAPHS", "1") != "0"
# Callers may come from any thread (the reference's contract): captures are
# serialised and run in thread-local capture mode, so other threads keep
# launching (and allocating) while one thread records a graph.
_GRAPH_LOCK = threading.RLock()


def _graphed(de: DeviceEnsemble, key: str, enqueue) -> "_Out":
    """Queue the device work of one call and return its result block, already
    copied to the host.  ``enqueue()`` returns the call's ``_Out``.

    A DeviceEnsemble reused for the same method runs eagerly once (plans,
    workspaces), is captured into a CUDA graph on its second call and
    replayed afterwards: one graph launch instead of the ctypes launches and
    allocations of the eager path (the small configurations are
    launch-bound).  Graphs are cached per (method, stream): a graph owns its
    workspace (completion counters), so two threads replaying on different
    streams never share one.  Replay and the D2H of the graph's result block
    run under the graph's own lock, so a caller always reads the block its
    own replay wrote.  Sharded ensembles (NCCL in the sequence) and timed
    runs (KERNEL_EVENTS) stay eager."""
    if not _GRAPHS or de.sharded or KERNEL_EVENTS is not None:
        out = enqueue()
        out.host()
        return out
    skey = (key, torch.cuda.current_stream(de.device).cuda_stream)
    with _GRAPH_LOCK:
        cache = de._cache.setdefault("graphs", {})
        ent = cache.get(skey)
        if ent is None:
            cache[skey] = False
        elif ent is False:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                outs = enqueue()
            for ws in de._cache.pop("graph_ws_pending", []):
                ws.zero_()  # the kernels leave their counters at zero after each replay
                de._cache.setdefault("graph_ws", []).append(ws)
            outs._pinned = torch.empty(outs.block.shape, dtype=outs.block.dtype, pin_memory=True)
            ent = cache[skey] = (g, outs, threading.Lock())
    if ent is None:
        out = enqueue()
        out.host()
        return out
    g, outs, lock = ent
    with lock:
        g.replay()
        out = outs.fresh()
        out.host()  # D2H (synchronises the stream) before the next replay
    return out


def _f64(n: int, dev) -> torch.Tensor:
    return torch.empty(n, dtype=torch.float64, device=dev)


def _allreduce(t: torch.Tensor, de: DeviceEnsemble) -> None:
    """Combine per-shard partial sums across GPUs: one NCCL allreduce."""
    if de.process_group is None:
        return
    import torch.distributed as dist

    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=de.process_group)


def _masses_device(de: DeviceEnsemble, with_nonbinary: bool = False):
    """K6 (+K7 check): member masses (depth.py:88-102) on the device."""
    dev = de.device
    mass = _f64(de.n, dev)
    nb = torch.zeros(de.n, dtype=torch.int64, device=dev) if with_nonbinary else None
    wsb = N.load().pidb_pid_mean_workspace_bytes(de.n, de.m, de.dtype_code)
    if wsb == 0:
        raise ValidationError(f"ensemble of {de.n} members is not supported by the tile layout")
    ws = de.workspace(wsb)
    _launch("pidb_member_masses", de.ptr(), de.dtype_code, de.n, de.m, de.ld, de.wptr(),
           mass.data_ptr(), None if nb is None else nb.data_ptr(), ws.data_ptr(), ws.numel(),
           stream_ptr(dev))
    if de.process_group is not None:
        _allreduce(mass, de)
        if nb is not None:
            _allreduce(nb, de)
    return (mass, nb) if with_nonbinary else mass


def _mean_partials(de: DeviceEnsemble, buf: torch.Tensor | None = None) -> torch.Tensor:
    """K5: packed [row_plain (n) | mass (n) | col_mean (1)], allreduced."""
    dev = de.device
    if buf is None:
        buf = _f64(2 * de.n + 1, dev)
    wsb = N.load().pidb_pid_mean_workspace_bytes(de.n, de.m, de.dtype_code)
    if wsb == 0:
        raise ValidationError(f"ensemble of {de.n} members is not supported by the tile layout")
    ws = de.workspace(wsb)
    p = buf.data_ptr()
    _launch("pidb_pid_mean_partials", de.ptr(), de.dtype_code, de.n, de.m, de.ld, de.wptr(),
           p, p + 8 * de.n, p + 16 * de.n, ws.data_ptr(), ws.numel(), stream_ptr(dev))
    _allreduce(buf, de)
    return buf


def _col_sums(de: DeviceEnsemble, inv: torch.Tensor) -> torch.Tensor:
    """K9-B: col_inv[j] = sum_i inv_i G[i,j] without forming G."""
    dev = de.device
    col = _f64(de.n, dev)
    ws = de.workspace(N.load().pidb_pid_mean_workspace_bytes(de.n, de.m, de.dtype_code))
    _launch("pidb_pid_colsums", de.ptr(), de.dtype_code, de.n, de.m, de.ld, de.wptr(),
           inv.data_ptr(), col.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr(dev))
    _allreduce(col, de)
    return col


class _Out:
    """Device result block [inv | in_in | in_out | depth] + ranks, one D2H."""

    def __init__(self, n: int, dev, extra: int = 0):
        self.n = n
        # one allocation -> one D2H; `extra` fp64 slots after the results carry
        # the method's partial sums (masses, mean mass) in the same copy
        self.block = _f64(5 * n + extra, dev)
        self.vals = self.block[:4 * n]
        self.rank = self.block[4 * n:5 * n].view(torch.int64)
        self.extra = self.block[5 * n:]
        self._host = None
        self._pinned = None  # pinned staging for the D2H (graph-replayed blocks)

    def ptrs(self):
        p, n = self.vals.data_ptr(), self.n
        return p, p + 8 * n, p + 16 * n, p + 24 * n

    def host(self) -> np.ndarray:
        h = self._host
        if h is None:
            pin = self._pinned
            if pin is None:
                h = self._host = self.block.cpu().numpy()
            else:  # async D2H into pinned memory, then a private host copy
                pin.copy_(self.block, non_blocking=True)
                torch.cuda.current_stream(self.block.device).synchronize()
                h = self._host = pin.numpy().copy()
        return h

    def fresh(self) -> "_Out":
        """Per-call view of a replayed graph's result block with its own
        host copy (the block itself is shared by every replay, and callers
        may come from several threads)."""
        o = object.__new__(_Out)
        o.__dict__.update(self.__dict__)
        o._host = None
        return o

    def host_extra(self) -> np.ndarray:
        return self.host()[5 * self.n:]

    def fetch(self):
        h, n = self.host(), self.n
        v = h[:4 * n].reshape(4, n)
        r = h[4 * n:5 * n].view(np.int64)
        return v[1].copy(), v[2].copy(), v[3].copy(), r.copy()


def _finish(de, out: _Out, method: str, masses: np.ndarray, t0: float) -> DepthResult:
    in_in, in_out, depth, rank = out.fetch()
    return DepthResult(ids=de.ids, in_in=in_in, in_out=in_out, depth=depth, rank=rank,
                       method=method, cv_mass=mass_cv(masses),
                       elapsed_seconds=time.perf_counter() - t0)


# ------------------------------------------------------------------ methods


def member_masses(ensemble, workers: int | None = None, require_binary: bool = False) -> np.ndarray:
    """Weighted mass of every member (depth.py:88-102), one device pass."""
    resolve_workers(workers)
    de = stage(ensemble).prob()
    if require_binary:
        mass, nb = _masses_device(de, with_nonbinary=True)
        _raise_first_nonbinary(de, nb)
    else:
        mass = _masses_device(de)
    return mass.cpu().numpy()


def _raise_first_nonbinary(de: DeviceEnsemble, nb) -> None:
    bad = np.flatnonzero(nb.cpu().numpy() if isinstance(nb, torch.Tensor) else nb)
    if bad.size:
        i = int(bad[0])
        raise ValidationError(f"member {de.ids[i]!r} is not binary (0/1) valued")


def _member_mean_terms(values, mean_values, weights) -> tuple[float, float]:
    """Seam of depth.py:231-243: fused (sum w u mean, sum w u) for one member
    against the mean mask, one device pass with fp64 accumulation (K8).  The
    depth methods themselves never call it: K5 forms these sums for every
    member in the same pass that forms the mean."""
    from .inclusion import _pair

    num, mass = _pair(values, mean_values, weights, N.PIDB_OP_INCLUSION)
    return num, mass


def depth_pid_mean(ensemble, workers: int | None = None,
                   cv_warn_threshold: float = CV_WARN_THRESHOLD) -> DepthResult:
    """Linear-time inclusion depth against the ensemble mean (depth.py:246-287).

    One HBM pass (K5) yields every member's sum against the mean, its mass
    and the mean's mass; K4 forms in_in, in_out, depth and ranks on device.
    """
    t0 = time.perf_counter()
    resolve_workers(workers)
    if _streamable(ensemble):
        return _pid_mean_streamed(ensemble, t0, cv_warn_threshold)
    de = stage(ensemble).prob()
    n, dev = de.n, de.device

    def enqueue():
        out = _Out(n, dev, extra=2 * n + 1)
        buf = _mean_partials(de, out.extra)
        p = buf.data_ptr()
        inv, ii, io, d = out.ptrs()
        N.call("pidb_depth_epilogue", N.PIDB_EPI_PID_MEAN, n, p, p + 8 * n, p + 16 * n,
               inv, ii, io, d, out.rank.data_ptr(), stream_ptr(dev))
        return out

    out = _graphed(de, "pid-mean", enqueue)
    host = out.host_extra()[n:]
    masses, col_mean = host[:n], float(host[n])
    if col_mean == 0.0:
        raise DegenerateEnsembleError("ensemble mean mask is identically zero")
    res = _finish(de, out, "pid-mean", masses, t0)
    if res.cv_mass > cv_warn_threshold:
        warnings.warn(
            f"member mass CV {res.cv_mass:.3g} exceeds {cv_warn_threshold:g}; "
            "pid-mean ranks may diverge from exact pid",
            RuntimeWarning,
            stacklevel=2,
        )
    return res


# Host-resident inputs larger than this stream through HBM in cell slabs.
STREAM_SLAB_BYTES = int(os.environ.get("PIDB_STREAM_SLAB_BYTES", str(2 << 30)))


def _streamable(x) -> bool:
    return (isinstance(x, torch.Tensor) and not x.is_cuda and x.is_pinned() and x.dim() >= 2
            and x.is_contiguous() and x.dtype in (torch.float32, torch.float64) and x.shape[0] >= 1
            and x.numel() * x.element_size() > 2 * STREAM_SLAB_BYTES)


def _pid_mean_streamed(host: torch.Tensor, t0: float, cv_warn_threshold: float) -> DepthResult:
    """PID-mean of a pinned host ensemble without staging it whole: cell slabs
    (every member, a range of cells) are copied on a side stream into two
    HBM slab buffers while the previous slab is validated in place
    (ProbMask policy, grid.py:105-116) and swept by K5 on the compute
    stream; the per-slab partial sums are additive over cells (the same
    decomposition as the multi-GPU voxel shards) and are combined in slab
    order, then the K4 epilogue runs once.  HBM holds two slabs, not the
    ensemble; copies, validation and K5 overlap."""
    from .device import _key_to_double, require_cuda
    from .grid import VALUE_TOLERANCE

    dev = require_cuda()
    n = int(host.shape[0])
    flat = host.reshape(n, -1)
    if flat.stride(1) != 1:
        raise ValidationError("host member tensor must have contiguous rows")
    m = int(flat.shape[1])
    es = flat.element_size()
    dt = flat.dtype
    code = N.PIDB_F64 if dt == torch.float64 else N.PIDB_F32
    S = max(32, (STREAM_SLAB_BYTES // (n * es)) // 32 * 32)
    S = min(S, (m + 31) // 32 * 32)
    slabs = [(c0, min(m, c0 + S)) for c0 in range(0, m, S)]
    K = torch.cuda.current_stream(dev)
    C = torch.cuda.Stream(dev)
    bufs = [torch.empty((n, S), dtype=dt, device=dev) for _ in range(2)]
    part = torch.empty((len(slabs), 2 * n + 1), dtype=torch.float64, device=dev)
    stats = torch.empty((len(slabs), 3), dtype=torch.int64, device=dev)
    lib = N.load()
    ws = torch.zeros(max(1, lib.pidb_pid_mean_workspace_bytes(n, S, code)), dtype=torch.uint8,
                     device=dev)
    free = [None, None]
    src0 = flat.data_ptr()
    for k, (c0, c1) in enumerate(slabs):
        b = k & 1
        buf = bufs[b]
        if free[b] is not None:
            C.wait_event(free[b])
        N.call("pidb_copy_rows", buf.data_ptr(), S * es, src0 + c0 * es, flat.stride(0) * es,
               (c1 - c0) * es, n, C.cuda_stream)
        landed = torch.cuda.Event()
        landed.record(C)
        K.wait_event(landed)
        mk = c1 - c0
        N.call("pidb_validate", buf.data_ptr(), code, n, mk, S, 1, stats[k].data_ptr(),
               K.cuda_stream)
        p = part[k].data_ptr()
        _launch("pidb_pid_mean_partials", buf.data_ptr(), code, n, mk, S, None, p, p + 8 * n,
                p + 16 * n, ws.data_ptr(), ws.numel(), K.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(K)
        free[b] = ev
    out = _Out(n, dev, extra=2 * n + 1)
    N.call("pidb_sum_rows", part.data_ptr(), len(slabs), 2 * n + 1, out.extra.data_ptr(),
           K.cuda_stream)
    pe = out.extra.data_ptr()
    inv, ii, io, d = out.ptrs()
    N.call("pidb_depth_epilogue", N.PIDB_EPI_PID_MEAN, n, pe, pe + 8 * n, pe + 16 * n,
           inv, ii, io, d, out.rank.data_ptr(), K.cuda_stream)
    st = stats.cpu().numpy()
    out.host()
    if st[:, 0].any():
        raise ValidationError("mask values must be finite")
    lo, hi = _key_to_double(int(st[:, 1].min())), _key_to_double(int(st[:, 2].max()))
    if lo < -VALUE_TOLERANCE or hi > 1.0 + VALUE_TOLERANCE:
        raise ValidationError(f"mask values outside [0, 1]: min={lo!r} max={hi!r}")
    host_ex = out.host_extra()[n:]
    masses, col_mean = host_ex[:n], float(host_ex[n])
    if col_mean == 0.0:
        raise DegenerateEnsembleError("ensemble mean mask is identically zero")
    in_in, in_out, depth, rank = out.fetch()
    from .device import _make_ids

    res = DepthResult(ids=_make_ids(None, n), in_in=in_in, in_out=in_out, depth=depth,
                      rank=rank, method="pid-mean", cv_mass=mass_cv(masses),
                      elapsed_seconds=time.perf_counter() - t0)
    if res.cv_mass > cv_warn_threshold:
        warnings.warn(
            f"member mass CV {res.cv_mass:.3g} exceeds {cv_warn_threshold:g}; "
            "pid-mean ranks may diverge from exact pid",
            RuntimeWarning,
            stacklevel=3,
        )
    return res


def _pid_factorized(de: DeviceEnsemble, out: _Out) -> torch.Tensor:
    """Exact PID in two HBM passes: K5 gives row_plain and masses, K9-B the
    inverse-mass-weighted column sums (SURVEY.md §0 finding 2).  Queues the
    work and returns the K5 block [row_plain | mass | col]."""
    n, dev = de.n, de.device
    buf = _mean_partials(de, out.extra if out.extra.numel() >= 2 * n + 1 else None)
    p = buf.data_ptr()
    inv = out.ptrs()[0]
    N.call("pidb_inverse_masses", n, p + 8 * n, inv, stream_ptr(dev))
    col = _col_sums(de, out.vals[:n])
    _, ii, io, d = out.ptrs()
    N.call("pidb_depth_epilogue", N.PIDB_EPI_PID, n, p, p + 8 * n, col.data_ptr(),
           inv, ii, io, d, out.rank.data_ptr(), stream_ptr(dev))
    return buf


# Error bound of the fixed-point Gram (gram_fixed.cu header): per cell
# product, quantisation 2^-32 (a_i + a_j) + 2^-64 and the dropped digit
# levels 4..6, at most 255^2 (3 * 2^16 + 2 * 2^8 + 1) * 2^-62, wherever both
# values have non-zero low digits; fp64 folding adds < 1e-13 relative.
_FX_TAIL = 255.0 ** 2 * (3 * 2 ** 16 + 2 * 2 ** 8 + 1) * 2.0 ** -62
_FX_REL = 1e-13
# Certified accuracy of depth_pid(algorithm="gram"): members whose bound
# exceeds it (members with tiny mass next to heavy ones, e.g. one-cell grids)
# are resolved with the exact path like uncertified ranks.
GRAM_DEPTH_TOL = 1e-8

# Diagnostics of the last tensor-core PID on this process (read by bench.py):
# certified bound, members resolved exactly.
LAST_GRAM_CERT: dict = {}


def _gram_depth_bounds(masses, soft, inv, row_plain, col_inv, m, wmax, wmin):
    """Rigorous per-member bounds on |depth_gram - depth_exact| (in_in and
    in_out errors propagated from the per-pair Gram bound)."""
    n = masses.shape[0]
    A = masses / np.sqrt(wmin * wmax)          # >= sum_x u sqrt(w / wmax)
    c = soft.astype(np.float64)
    order = np.argsort(c, kind="stable")
    cs = c[order]
    pre = np.concatenate([[0.0], np.cumsum(cs)])
    pre_inv = np.concatenate([[0.0], np.cumsum(inv[order] * cs)])
    inv_s = inv[order]
    suf_inv = np.concatenate([np.cumsum(inv_s[::-1])[::-1], [0.0]])
    k = np.searchsorted(cs, c, side="right")   # members with c_j <= c_i
    min_sum = pre[k] + c * (n - k)             # sum_j min(c_i, c_j)
    min_sum_inv = pre_inv[k] + c * suf_inv[k]  # sum_j inv_j min(c_i, c_j)
    sinv = float(inv.sum())
    row_err = wmax * (2.0 ** -32 * (n * A + A.sum()) + n * m * 2.0 ** -64
                      + _FX_TAIL * min_sum) + _FX_REL * np.abs(row_plain)
    col_err = wmax * (2.0 ** -32 * (A * sinv + float(inv @ A)) + m * sinv * 2.0 ** -64
                      + _FX_TAIL * min_sum_inv) + _FX_REL * np.abs(col_inv)
    return np.maximum(inv * row_err / n, col_err / n)


def _clustered(depth, eps):
    """Members whose interval [d - eps, d + eps] meets another member's:
    their relative order is not certified."""
    lo, hi = depth - eps, depth + eps
    order = np.argsort(lo, kind="stable")
    flag = np.zeros(depth.shape[0], dtype=bool)
    start, reach = 0, -np.inf
    for pos, i in enumerate(order):
        if lo[i] > reach:
            if pos - start > 1:
                flag[order[start:pos]] = True
            start = pos
        reach = max(reach, hi[i])
    if order.shape[0] - start > 1:
        flag[order[start:]] = True
    return flag


def _pid_gram(de: DeviceEnsemble, out: _Out) -> np.ndarray:
    """PID from the symmetric N x N Gram on the tcgen05 int8 tensor cores
    (K1x: fixed-point digits, exact integer accumulation), with the row sums
    and inverse-mass-weighted column sums of G (depth.py:156-160) fused into
    the Gram epilogue: no N x N matrix in HBM.  Then the rank certifier
    (SURVEY.md §7.3): every member whose depth interval (rigorous Gram error
    bound) meets another member's, or whose bound exceeds GRAM_DEPTH_TOL, is
    resolved with the exact fp64 path, so the ranks equal the exact ones and
    every depth is within GRAM_DEPTH_TOL of exact.  Returns the masses."""
    from .reduction import pack_fixed

    n, dev = de.n, de.device
    lib = N.load()
    # one pass: digit tiles, soft-cell counts and the member masses
    soft = torch.zeros(n, dtype=torch.int64, device=dev)
    mass = _f64(n, dev)
    q, wmax = pack_fixed(de, soft, mass)
    _allreduce(mass, de)
    inv = out.ptrs()[0]
    N.call("pidb_inverse_masses", n, mass.data_ptr(), inv, stream_ptr(dev))
    rc = _f64(2 * n, dev)
    ws = de.workspace(lib.pidb_gram_fixed_workspace_bytes(n, de.m, 1))
    _launch("pidb_gram_fixed_sums", q.data_ptr(), n, de.m, wmax, inv, rc.data_ptr(),
            rc.data_ptr() + 8 * n, ws.data_ptr(), ws.numel(), stream_ptr(dev))
    _allreduce(rc, de)
    _allreduce(soft, de)
    _, ii, io, d = out.ptrs()
    N.call("pidb_depth_epilogue", N.PIDB_EPI_PID, n, rc.data_ptr(), mass.data_ptr(),
           rc.data_ptr() + 8 * n, inv, ii, io, d, out.rank.data_ptr(), stream_ptr(dev))
    masses = mass.cpu().numpy()
    h = out.host()
    rch = rc.cpu().numpy()
    wmin = float(de.weights.min()) if de.weights is not None else 1.0
    if de.process_group is not None:
        import torch.distributed as dist

        t = torch.tensor([wmax, -wmin], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=de.process_group)
        wmax, wmin = float(t[0]), -float(t[1])
        mt = torch.tensor([float(de.m)], dtype=torch.float64, device=dev)
        dist.all_reduce(mt, group=de.process_group)
        m_cells = float(mt)
    else:
        m_cells = float(de.m)
    eps = _gram_depth_bounds(masses, soft.cpu().numpy(), h[:n], rch[:n], rch[n:], m_cells,
                             wmax, wmin)
    flag = _clustered(h[3 * n:4 * n], eps) | (eps > GRAM_DEPTH_TOL)
    LAST_GRAM_CERT.clear()
    LAST_GRAM_CERT.update(max_bound=float(eps.max()), resolved_exactly=int(flag.sum()))
    if flag.any():
        exact = _Out(n, dev, extra=2 * n + 1)
        _pid_factorized(de, exact)
        e = exact.host()
        blk = h.copy()
        for k in (1, 2, 3):
            blk[k * n:(k + 1) * n][flag] = e[k * n:(k + 1) * n][flag]
        blk[4 * n:5 * n] = ranks_from_depths(blk[3 * n:4 * n]).view(np.float64)
        out._host = blk
    return masses


def _gram_available() -> bool:
    return N.has_symbol("pidb_gram_fixed_sums")


def depth_pid(ensemble, workers: int | None = None, *, algorithm: str = "auto") -> DepthResult:
    """Exact probabilistic inclusion depth over all pairs (depth.py:213-228).

    algorithm="factorized" (default via "auto"): exact fp64 O(N*M) two-pass
    identity (row sums of G against S = sum_j u_j, column sums against
    T = sum_i u_i / m_i); agrees with the reference to ~1e-15.
    algorithm="gram": the symmetric N x N Gram on the tcgen05 int8 tensor
    cores (fixed-point digits, exact integer accumulation; depth error
    ~1e-9) followed by the row/column-sum epilogue -- the reference's own
    formulation -- and a rank certifier that resolves every member whose
    error interval meets another's with the exact path (K1).
    """
    t0 = time.perf_counter()
    resolve_workers(workers)
    if algorithm not in PID_ALGORITHMS:
        raise ValidationError(f"unknown pid algorithm {algorithm!r}; expected one of {PID_ALGORITHMS}")
    de = stage(ensemble).prob()
    n = de.n
    if algorithm == "gram":
        out = _Out(n, de.device)
        masses = _pid_gram(de, out)
    else:
        def enqueue():
            out = _Out(n, de.device, extra=2 * n + 1)
            _pid_factorized(de, out)
            return out

        out = _graphed(de, "pid", enqueue)
        masses = out.host_extra()[n:2 * n].copy()
    return _finish(de, out, "pid", masses, t0)


def depth_eid(ensemble, workers: int | None = None) -> DepthResult:
    """Inclusion depth of binary ensembles (depth.py:192-210).

    Unit weights: exact integer intersection Gram (K7 pack + K2 tcgen05
    kind::i8; a byte ensemble goes to K2 directly) and an exactly rounded
    epilogue, bit-identical to the exact-summation oracle ref_eid.
    Weighted grids: factorised Gram sums.
    """
    t0 = time.perf_counter()
    resolve_workers(workers)
    de = stage(ensemble)
    if de.weights is not None:
        de = de.prob()
    n, dev = de.n, de.device
    if de.weights is None:
        from .reduction import intersection_gram, pack_binary

        def enqueue():
            # K7 packs and counts non-binary values in the same pass (the
            # counts ride in the result block); the masses are the Gram
            # diagonal |C_i| (exact integers).  Byte ensembles were checked
            # when staged and need no pack.
            out = _Out(n, dev, extra=n)
            nb = out.extra.view(torch.int64)
            nb.zero_()
            if de.is_bits:
                g = intersection_gram(de)
            else:
                packed = pack_binary(de, nb)
                _allreduce(nb, de)
                g = intersection_gram(de, packed)
            mslot, ii, io, d = out.ptrs()
            N.call("pidb_eid_exact_epilogue", g.data_ptr(), n, ii, io, d, out.rank.data_ptr(),
                   mslot, stream_ptr(dev))
            return out

        out = _graphed(de, "eid", enqueue)
        # one host round trip: the non-binary check is read after the whole
        # stream has been queued (the results are discarded if it fails)
        _raise_first_nonbinary(de, out.host_extra().view(np.int64))
        masses = out.host()[:n].copy()
    else:
        out = _Out(n, dev)
        mass, nb = _masses_device(de, with_nonbinary=True)
        _raise_first_nonbinary(de, nb)
        buf = _mean_partials(de)
        p = buf.data_ptr()
        inv = out.ptrs()[0]
        N.call("pidb_inverse_masses", n, p + 8 * n, inv, stream_ptr(dev))
        col = _col_sums(de, out.vals[:n])
        masses = buf[n:2 * n].cpu().numpy()
        n_pos = float(np.count_nonzero(masses > 0.0))
        _, ii, io, d = out.ptrs()
        N.call("pidb_eid_factorized_epilogue", n, p, p + 8 * n, col.data_ptr(), n_pos,
               inv, ii, io, d, out.rank.data_ptr(), stream_ptr(dev))
    return _finish(de, out, "eid", masses, t0)


_BASELINES = {"dice": "dice", "fuzzy-dice": "dice", "iou": "iou", "prob-iou": "iou"}


def depth_similarity_baseline(ensemble, measure: str, workers: int | None = None) -> DepthResult:
    """Depth as the symmetric similarity of each member to the mean mask
    (depth.py:298-325): fuzzy Dice or probabilistic IoU.  One device pass
    forms sum w*min(u_i, mean) and the masses (sum w*max follows from
    min + max = u + mean)."""
    try:
        kind = _BASELINES[measure]
    except KeyError:
        raise ValidationError(
            f"unknown similarity measure {measure!r}; expected one of {sorted(_BASELINES)}"
        ) from None
    t0 = time.perf_counter()
    resolve_workers(workers)
    de = stage(ensemble).prob()
    n, dev = de.n, de.device

    def enqueue():
        out = _Out(n, dev, extra=2 * n + 1)
        buf = out.extra
        ws = de.workspace(N.load().pidb_pid_mean_workspace_bytes(de.n, de.m, de.dtype_code))
        p = buf.data_ptr()
        _launch("pidb_similarity_partials", de.ptr(), de.dtype_code, n, de.m, de.ld, de.wptr(),
                p, p + 8 * n, p + 16 * n, ws.data_ptr(), ws.numel(), stream_ptr(dev))
        _allreduce(buf, de)
        inv, ii, io, d = out.ptrs()
        N.call("pidb_depth_epilogue", N.PIDB_EPI_DICE if kind == "dice" else N.PIDB_EPI_IOU,
               n, p, p + 8 * n, p + 16 * n, inv, ii, io, d, out.rank.data_ptr(),
               stream_ptr(dev))
        return out

    out = _graphed(de, kind, enqueue)
    host = out.host_extra()[n:]
    if float(host[n]) == 0.0:
        raise DegenerateEnsembleError("ensemble mean mask is identically zero")
    return _finish(de, out, kind, host[:n], t0)


def compare_pid_vs_mean(ensemble, workers: int | None = None) -> dict:
    """Exact PID vs PID-mean: depth error and rank agreement (depth.py:328-346)."""
    from .consistency import kendall_tau, pearson

    de = stage(ensemble).prob()
    if de.n < 2:
        raise ValidationError("comparison needs at least two members")
    exact = depth_pid(de, workers)
    approx = depth_pid_mean(de, workers)
    err = np.abs(exact.depth - approx.depth)
    return {
        "max_abs_error": float(err.max()),
        "mean_abs_error": float(err.mean()),
        "rank_pearson": pearson(exact.rank, approx.rank),
        "rank_kendall": kendall_tau(exact.rank, approx.rank),
        "cv_mass": approx.cv_mass,
    }


def depth_by_method(ensemble, method: str, workers: int | None = None) -> DepthResult:
    """Dispatch on a method name (depth.py:349-363)."""
    if method == "eid":
        return depth_eid(ensemble, workers)
    if method == "pid":
        return depth_pid(ensemble, workers)
    if method == "pid-mean":
        return depth_pid_mean(ensemble, workers)
    if method in _BASELINES:
        return depth_similarity_baseline(ensemble, method, workers)
    raise ValidationError(f"unknown depth method {method!r}; expected one of {METHOD_NAMES}")
