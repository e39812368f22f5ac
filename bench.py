#!/usr/bin/env python
"""Benchmark of the B200 depth hot path (contract: one JSON line on rank 0).

Workload (BASELINE.json configs[4], the largest single-GPU PID-mean config):
PID-mean on a 200-member 512^3 fp32 fuzzy-ellipsoid ensemble (107.4 GB), the
reference generator's recipe evaluated on the device.  A "step" is one full
depth_pid_mean call (K5 single HBM pass + allreduce when N>1 + K4 epilogue +
result D2H).  ``value`` = member-voxels/s with the ensemble resident in HBM;
``e2e`` = the same call on a pinned HOST tensor (H2D staging, validation,
kernels and result D2H inside the timed region).  The secondary ``pid``
object reports exact PID on BASELINE configs[3] (1000 x 256^3).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (voxel-sharded, NCCL)

``--impl reference`` times the reference algorithm's CPU restatement
(oracle.port, numpy/OpenBLAS, all host threads) on a bounded sample of the
same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (method, res, members, description)
    "cfg1": ("pid-mean", 256, 100, "cfg1: 2D fuzzy disks, 100 members 256^2"),
    "cfg3": ("pid-mean", 128, 200, "cfg3: PID-mean, 200 fuzzy ellipsoids 128^3 fp32"),
    "cfg4": ("pid", 256, 1000, "cfg4: PID, 1000 fuzzy ellipsoids 256^3 fp32"),
    "cfg5": ("pid-mean", 512, 200, "cfg5: PID-mean, 200 fuzzy ellipsoids 512^3 fp32 (107.4 GB)"),
}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "src": "measured (MEASURED_PEAKS.json)",
                "bf16": d.get("bf16_tflops", 1590.0)}
    return {"hbm_gbs": 6650.0, "src": "fallback (B200_PROFILING.md)", "bf16": 1590.0}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ helpers


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if os.environ.get("PIDB_BENCH_SHARE_GPU") == "1":
            # flow check only (as tools/dist_check.py does): every rank on cuda:0, gloo
            # collectives; the timings of such a run mean nothing
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist.group.WORLD
    return rank, world, local, pg


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


_L2_FLUSH = None


def flush_l2():
    """Write 512 MB (> the 126 MB L2) so the next step starts cold."""
    import torch

    global _L2_FLUSH
    if _L2_FLUSH is None:
        _L2_FLUSH = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
    _L2_FLUSH.fill_(1.0)


def timed(step, steps, warmup, world, sampler=None, flush=False):
    """W untimed steps, then K steps between barrier+sync, device events.
    flush=True (inputs smaller than L2): each step is timed on its own with
    an L2 flush between steps, outside the timed intervals."""
    import torch

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    if sampler:
        sampler.__enter__()
        time.sleep(0.3)
    if flush:
        total = 0.0
        for _ in range(steps):
            flush_l2()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            step()
            b.record()
            b.synchronize()
            total += a.elapsed_time(b)
        ms = total / steps
    else:
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            step()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / steps
    if sampler:
        sampler.__exit__()
    barrier(world)
    return max_over_ranks(ms, world)


def kernel_ms(events, name):
    ts = [a.elapsed_time(b) for nm, a, b in events if nm == name]
    return (float(np.mean(ts)) if ts else None), len(ts)


def ellipsoid_sample_cpu(res, n, y_planes, seed=0):
    """Bounded CPU sample of the cfg ellipsoid workload: all n members on
    `y_planes` central planes (generated with torch on the host cores)."""
    import torch

    from paper_2512_15187_b200.synth import ellipsoid_params

    prm, sigma, _ = ellipsoid_params(res, n, 0, seed)
    y0 = res // 2 - y_planes // 2
    y = torch.arange(y0, y0 + y_planes, dtype=torch.float64).view(-1, 1, 1)
    x = torch.arange(res, dtype=torch.float64).view(1, -1, 1)
    z = torch.arange(res, dtype=torch.float64).view(1, 1, -1)
    out = np.empty((n, y_planes * res * res), dtype=np.float32)
    for i in range(n):
        cy, cx, cz, ay, ax, az = prm[i]
        dy, dx, dz = y - cy, x - cx, z - cz
        rho = torch.sqrt((dy / ay) ** 2 + (dx / ax) ** 2 + (dz / az) ** 2)
        r = torch.sqrt(dy ** 2 + dx ** 2 + dz ** 2)
        d = r * (1.0 - 1.0 / rho)
        u = torch.where(rho > 1.0, torch.exp(-(d ** 2) / (2.0 * sigma * sigma)), torch.ones_like(rho))
        out[i] = u.to(torch.float32).reshape(-1).numpy()
    return out


def disk_sample_cpu(res, n, seed=0):
    """cfg1 members on the host (gen_disk_ensemble recipe, numpy)."""
    from paper_2512_15187_b200.synth import disk_params

    prm, sigma2, _ = disk_params(res, n, seed)
    y, x = np.mgrid[0:res, 0:res].astype(np.float64)
    out = np.empty((n, res * res), dtype=np.float32)
    for i in range(n):
        cy, cx, radius = prm[i]
        dist = np.sqrt((y - cy) ** 2 + (x - cx) ** 2)
        out[i] = np.where(dist <= radius, 1.0,
                          np.exp(-((dist - radius) ** 2) / (2.0 * sigma2))).reshape(-1)
    return out


def reference_module():
    """The unmodified reference (baseline/_ref, tools/install_reference.sh) or None."""
    from oracle import reference

    try:
        return reference.load()
    except ImportError:
        return None


def cpu_reference(U, method, workers, dims=None):
    """Seconds for one depth call of the CPU reference on host array U: the
    real fuzzdepth (baseline/_ref) when installed, else oracle.port.  The
    Ensemble (ProbMask validation) is built outside the timed call."""
    fd = reference_module()
    if fd is not None:
        from oracle import reference

        ens = reference.from_array(fd, U, dims)
        fn = {"pid-mean": fd.depth_pid_mean, "eid": fd.depth_eid, "pid": fd.depth_pid}[method]
        t0 = time.perf_counter()
        fn(ens, workers=workers)
        return time.perf_counter() - t0
    from oracle import port

    t0 = time.perf_counter()
    if method == "pid-mean":
        port.depth_pid_mean(U, None, workers=workers)
    elif method == "eid":
        port.depth_eid(U, None, workers=workers)
    else:
        port.depth_pid(U, None, workers=workers)
    return time.perf_counter() - t0


def cpu_kind():
    return "reference" if reference_module() is not None else "port"


def cpu_what():
    fd = reference_module()
    if fd is not None:
        return (f"fuzzdepth {fd.__version__} (the unmodified reference, baseline/_ref; "
                f"numpy {np.__version__}, OPENBLAS_NUM_THREADS="
                f"{os.environ.get('OPENBLAS_NUM_THREADS', 'unset')})")
    return "oracle.port (numpy/OpenBLAS restatement of fuzzdepth; baseline/_ref not installed)"


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_pair_baseline(U, method, n_full, m_full, what):
    """oracle.port on a bounded sample of an O(N^2 M) workload: measured
    pair-voxels/s plus the full-size time extrapolated from it (labelled)."""
    workers = os.cpu_count() or 1
    sec = cpu_reference(U, method, workers)
    pv = U.shape[0] ** 2 * U.shape[1] / sec
    return {"value": U.shape[0] * U.shape[1] / sec, "unit": "member-voxels/s",
            "pair_voxels_per_s": pv, "cores": workers, "kind": cpu_kind(),
            "sample": f"{U.shape[0]} members x {U.shape[1]} cells of {what}; {cpu_what()} "
                      f"{method}, workers={workers}", "cpu_model": cpu_model(),
            "seconds": sec,
            "extrapolated_full_seconds": n_full ** 2 * m_full / pv,
            "extrapolation": "full-size time = N^2 M / measured pair-voxels/s (not measured)"}


# ------------------------------------------------------------ reference arm


def run_reference(args, rank, world):
    """The reference's own CPU implementation on this box's host cores: the
    unmodified fuzzdepth from baseline/_ref (oracle.port only when it is not
    installed), each step one depth call on a bounded sample of the
    workload (all members, the central planes), rank 0 only."""
    if rank != 0:
        return
    method, res, n, desc = WORKLOADS[args.workload]
    workers = os.cpu_count() or 1
    planes = args.ref_planes or (REF_PLANES if res >= 512 else max(1, res // 16))
    if args.workload == "cfg1":  # the whole 2D ensemble (26 MB)
        U, planes = disk_sample_cpu(res, n), res
    else:
        U = ellipsoid_sample_cpu(res, n, planes)
    if method == "pid":
        U = U[: min(n, args.ref_pid_members)]
    mv = U.shape[0] * U.shape[1]
    for _ in range(args.warmup):
        cpu_reference(U, method, workers)
    ts = [cpu_reference(U, method, workers) for _ in range(args.steps)]
    sec = float(np.mean(ts))
    value = mv / sec
    sample = (f"{U.shape[0]} members x {planes} central planes of {res}^3 "
              f"({U.shape[1]} cells/member) of the {args.workload} workload; {cpu_what()} "
              f"depth_{method.replace('-', '_')}(Ensemble of host ProbMasks), workers={workers}")
    line = {
        "impl": "reference", "metric": metric_name(method), "value": value,
        "unit": "member-voxels/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "sample": sample},
        "cpu_baseline": {"value": value, "unit": "member-voxels/s", "cores": workers,
                         "kind": cpu_kind(), "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "member-voxels/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# central planes of 512^3 in the CPU samples (reference arm, cpu_baseline)
REF_PLANES = 16
# end-to-end steps (each moves the whole ensemble over PCIe: ~2 s at cfg5)
E2E_STEPS = 10


def ncu_traffic(workload, world):
    """DRAM bytes (read + write) per K5 launch from the committed ncu capture of
    the same workload (profiles/r02_traffic.json), or None."""
    if world != 1:
        return None
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                               "r02_traffic.json")) as fh:
            t = json.load(fh).get(workload)
        return None if t is None else t["dram_read_bytes"] + t["dram_write_bytes"]
    except (OSError, ValueError, KeyError):
        return None


def metric_name(method):
    return "member-voxels/sec for PID-mean" if method == "pid-mean" else "member-voxels/sec for PID"


# ------------------------------------------------------------------ our arm


def run_ours(args, rank, world, local, pg):
    import torch

    import paper_2512_15187_b200 as pb
    from paper_2512_15187_b200 import depth as D
    from paper_2512_15187_b200 import synth

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    method, res, n, desc = WORKLOADS[args.workload]
    two_d = args.workload == "cfg1"
    m_full = res ** 2 if two_d else res ** 3
    shard = (rank, world) if world > 1 else None
    fn = pb.depth_pid_mean if method == "pid-mean" else pb.depth_pid
    pk = peaks()

    if two_d:  # reference gen_disk_ensemble recipe (SURVEY.md §8 d: no 2D ellipse generator)
        if shard is not None:
            raise SystemExit("cfg1 (26 MB) is a single-GPU workload")
        de = synth.disks_device(res, n, 0, device=dev)
    else:
        de = synth.ellipsoids_device(res, n, 0, 0, device=dev, shard=shard, process_group=pg)
    torch.cuda.synchronize()
    m_local = de.m

    def step():
        return fn(de)

    D.KERNEL_EVENTS = []
    sampler = ClockSampler(local) if rank == 0 else None
    fn(de)  # first call outside the event log (plans, workspace)
    D.KERNEL_EVENTS = []
    small = n * m_local * 4 < 2 * 126e6  # inputs not much larger than L2: flush between steps
    ms = timed(step, args.steps, args.warmup, world, sampler, flush=small)
    kname = "pidb_pid_mean_partials"
    kms, klaunch = kernel_ms(D.KERNEL_EVENTS, kname)
    launches_per_step = 3 if method == "pid-mean" else 6
    D.KERNEL_EVENTS = None
    total_mv = n * m_full
    value = total_mv / (ms * 1e-3)
    alg_bytes = n * m_local * 4
    achieved = alg_bytes / (kms * 1e-3) / 1e9 if kms else None

    res_chk = fn(de)
    line = {
        "metric": metric_name(method), "value": value, "unit": "member-voxels/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference gen_ellipsoid_ensemble recipe: per-member Philox "
                "parameters on the host, voxels evaluated on the device)",
        "config": {"workload": desc, "members": n, "cells": m_full, "cells_per_gpu": m_local,
                   "bytes_per_gpu": alg_bytes, "l2": ("L2 flushed (512 MB write) between individually timed steps: inputs "
                          "(%.3f GB) < 2 x 126 MB L2" if small else
                          "no flush: inputs (%.1f GB/GPU) >> 126 MB L2") % (alg_bytes / 1e9),
                   "parallelism": f"voxel-sharded x{world}, one NCCL allreduce of 2N+1 fp64"
                   if world > 1 else "single GPU"},
        "roofline": {"bound": "hbm", "kernel": "stream_pass_kernel (K5, pidb_pid_mean_partials)",
                     "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / pk["hbm_gbs"] if achieved else None,
                     "traffic": ncu_traffic(args.workload, world),
                     "algorithmic_bytes_per_launch": alg_bytes,
                     # the peak above is a copy (read + write) benchmark; a pure
                     # read stream goes faster: our TMA streaming microbenchmark
                     # (tools/ubench_tma.cu, profiles/r01_ubench_tma.log) reached
                     # 7227 GB/s with 512-byte box rows
                     "read_stream_peak": READ_STREAM_PEAK_GBS,
                     "frac_read_stream": achieved / READ_STREAM_PEAK_GBS if achieved else None,
                     "kernel_ms": kms, "launches_timed": klaunch, "peak_src": pk["src"]},
        "gpu_launches": launches_per_step * args.steps,
        "min_depth_gap": float(np.min(np.diff(np.sort(res_chk.depth)))) if n > 1 else None,
    }
    if sampler is not None:
        line["clocks"] = sampler.summary()

    # ---------------- CPU baseline (rank 0, N=1): the reference on a sample
    if rank == 0 and world == 1 and not args.no_cpu:
        planes = args.ref_planes or (REF_PLANES if res >= 512 else max(1, res // 16))
        y0 = res // 2 - planes // 2
        lo, hi = y0 * res * res, (y0 + planes) * res * res
        if two_d:  # all of cfg1
            lo, hi, planes = 0, res * res, res
        U = de.values[:, lo:hi].cpu().numpy()
        if method == "pid":
            U = U[: args.ref_pid_members]
        workers = os.cpu_count() or 1
        sec = cpu_reference(U, method, workers)
        line["cpu_baseline"] = {
            "value": U.shape[0] * U.shape[1] / sec, "unit": "member-voxels/s", "cores": workers,
            "kind": cpu_kind(), "cpu_model": cpu_model(),
            "sample": f"{U.shape[0]} members x {planes} central planes ({U.shape[1]} cells) "
                      f"of the same ensemble (the same sample as the --impl reference arm); "
                      f"{cpu_what()} depth_{method.replace('-', '_')}, workers={workers}; "
                      "PID-mean is GIL-bound (effectively 1 core) in the reference",
        }

    # ---------------- parity at full size against the CPU reference
    if rank == 0 and world == 1 and not args.no_parity and method == "pid-mean":
        line["parity"] = {f"{args.workload}_pid_mean_full": _guarded(
            f"{args.workload} parity", parity_pid_mean_full, de, res_chk)}
    elif rank == 0 and world == 1 and not args.no_parity and args.workload == "cfg4":
        line["parity"] = {"cfg4_1000x64": _guarded("cfg4 1000x64^3 parity", parity_pid_reduced,
                                                   dev)}
    if "parity" in line and args.workload == "cfg1":  # cfg1 names full PID too (CPU-sized)
        line["parity"]["cfg1_pid_full"] = _guarded("cfg1 pid parity", parity_pid_full, de,
                                                   pb.depth_pid(de))

    # ---------------- end to end from pinned host memory
    host = None
    if not args.no_e2e:
        host, e2e_meta = prepare_e2e(de, world)
    meta = (de.n, de.m, de.dims, de.cell_range)
    del de
    torch.cuda.empty_cache()
    if not args.no_e2e:
        line["e2e"] = run_e2e(args, host, e2e_meta, meta, fn, world, pg, dev,
                              res_chk if world == 1 else None) if host is not None \
            else e2e_meta
        del host

    # ---------------- secondary: exact PID on cfg4, bit-exact eID on cfg2
    if args.workload == "cfg5" and not args.no_pid:
        line["pid"] = (_guarded("cfg4 pid", run_pid_secondary, args, rank, world, pg, dev, pk)
                       if world == 1 else run_pid_secondary(args, rank, world, pg, dev, pk))
    if args.workload == "cfg5" and not args.no_eid and world == 1:
        line["eid"] = _guarded("cfg2 eid", run_eid_secondary, args, dev, pk)

    if rank == 0:
        print(json.dumps(line), flush=True)


def _guarded(what, fn, *a):
    """A secondary leg (parity, cfg4 / cfg2 lines) must not cost the
    headline: its failure is recorded in the line instead of raised."""
    try:
        return fn(*a)
    except Exception as exc:  # noqa: BLE001 -- reported, not swallowed
        import traceback

        traceback.print_exc()
        return {"error": f"{what}: {type(exc).__name__}: {exc}"}


def _agreement(got, ref):
    d = np.abs(np.asarray(got.depth) - np.asarray(ref.depth))
    gap = float(np.min(np.diff(np.sort(ref.depth)))) if len(ref.depth) > 1 else None
    return {"max_abs_depth_err": float(d.max()),
            "max_abs_in_in_err": float(np.abs(got.in_in - ref.in_in).max()),
            "max_abs_in_out_err": float(np.abs(got.in_out - ref.in_out).max()),
            "rank_identical": bool(np.array_equal(np.asarray(got.rank), np.asarray(ref.rank))),
            "rank_mismatches": int(np.sum(np.asarray(got.rank) != np.asarray(ref.rank))),
            "ref_min_adjacent_gap": gap}


def parity_pid_mean_full(de, got):
    """Full-size depth_pid_mean of the REAL reference on the same device bytes
    (lazy loaders copy one member at a time out of HBM) vs the GPU result."""
    fd = reference_module()
    if fd is None:
        return {"skipped": "baseline/_ref not installed (tools/install_reference.sh)"}
    from oracle import reference

    workers = min(16, os.cpu_count() or 1)  # bounds host residency (one member per worker)
    t0 = time.perf_counter()
    ref = fd.depth_pid_mean(reference.lazy_from_device(fd, de), workers=workers)
    out = {"reference": cpu_what(), "size": f"{de.n} x {de.m} cells (full config, "
                                             f"{de.n * de.m:.3e} member-voxels)",
           "reference_seconds": time.perf_counter() - t0, "workers": workers}
    out.update(_agreement(got, ref))
    return out


def parity_pid_full(de, got):
    """Full-size depth_pid of the REAL reference on the same device bytes."""
    fd = reference_module()
    if fd is None:
        return {"skipped": "baseline/_ref not installed (tools/install_reference.sh)"}
    from oracle import reference

    workers = min(16, os.cpu_count() or 1)
    t0 = time.perf_counter()
    ref = fd.depth_pid(reference.lazy_from_device(fd, de), workers=workers)
    out = {"reference": cpu_what(), "size": f"{de.n} x {de.m} cells (full config)",
           "reference_seconds": time.perf_counter() - t0, "workers": workers}
    out.update(_agreement(got, ref))
    return out


def parity_pid_reduced(dev):
    """cfg4 at reduced resolution (1000 x 64^3, SURVEY.md §7.3 hard part 4:
    full-size CPU PID takes ~21 h): the real reference depth_pid vs the exact
    GPU path and the tensor-core Gram path, on the same bytes."""
    import paper_2512_15187_b200 as pb
    from paper_2512_15187_b200 import depth as D
    from paper_2512_15187_b200 import synth

    fd = reference_module()
    if fd is None:
        return {"skipped": "baseline/_ref not installed (tools/install_reference.sh)"}
    from oracle import reference

    de = synth.ellipsoids_device(64, 1000, 0, 0, device=dev)
    U = de.values[:, :de.m].cpu().numpy()
    ens = reference.from_array(fd, U, de.dims, ids=list(de.ids))
    t0 = time.perf_counter()
    ref = fd.depth_pid(ens, workers=os.cpu_count() or 1)
    sec = time.perf_counter() - t0
    exact = pb.depth_pid(de, algorithm="factorized")
    gram = pb.depth_pid(de, algorithm="gram")
    cert = dict(D.LAST_GRAM_CERT)
    return {"size": "1000 x 64^3 (cfg4 members and generator at reduced resolution)",
            "reference": cpu_what(), "reference_seconds": sec,
            "factorized_vs_reference": _agreement(exact, ref),
            "gram_vs_reference": _agreement(gram, ref), "gram_certifier": cert}


def parity_eid_full(de, got):
    """cfg2 at full size: the real reference's depth_eid and the exact-
    summation oracle (the reference tests' ref_eid restated exactly,
    oracle.exact.eid_fast) on the same bytes.  The GPU path is defined to be
    bit-identical to the oracle; against depth_eid (BLAS dgemv sums) it agrees
    to a few ulps, with ranks equal except inside exact-rational ties."""
    fd = reference_module()
    from oracle import exact, port

    U = de.values[:, :de.m].cpu().numpy()
    a, b, c, _ = exact.eid_fast(U)
    out = {"size": f"{de.n} x {de.m} cells (full cfg2)",
           "oracle_bit_identical": bool(np.array_equal(got.depth, c) and np.array_equal(got.in_in, a)
                                        and np.array_equal(got.in_out, b)),
           "oracle_rank_identical": bool(np.array_equal(got.rank, port.ranks(c)))}
    if fd is not None:
        from oracle import reference

        t0 = time.perf_counter()
        ref = fd.depth_eid(reference.from_array(fd, U, de.dims, ids=list(de.ids)),
                           workers=os.cpu_count() or 1)
        out["reference_seconds"] = time.perf_counter() - t0
        out["reference"] = cpu_what()
        out.update(_agreement(got, ref))
    return out


def prepare_e2e(de, world):
    """Copy the resident ensemble (this rank's slab) into pinned host memory."""
    import psutil
    import torch

    need = de.n * de.m * 4
    avail = psutil.virtual_memory().available
    if need * world > 0.8 * avail:
        return None, {"value": None, "unit": "member-voxels/s",
                      "skipped": f"needs {need * world / 1e9:.1f} GB pinned host memory, "
                                 f"{avail / 1e9:.1f} GB available"}
    host = torch.empty((de.n, de.m), dtype=torch.float32, pin_memory=True)
    host.copy_(de.values[:, :de.m])
    torch.cuda.synchronize()
    return host, None


def run_e2e(args, host, _, meta, fn, world, pg, dev, resident=None):
    """The public API on this rank's pinned host tensor.  Single GPU, PID-mean:
    ``depth_pid_mean(host_tensor)`` streams cell slabs through HBM (H2D on a
    side stream overlapped with in-place validation and K5).  Otherwise the
    tensor is staged whole (DeviceEnsemble.from_tensor) and the method runs."""
    from paper_2512_15187_b200 import depth as D
    from paper_2512_15187_b200.device import DeviceEnsemble

    n, m, dims, cr = meta
    streamed = world == 1 and fn is D.depth_pid_mean and D._streamable(host)

    def step():
        if streamed:
            return fn(host)
        e = DeviceEnsemble.from_tensor(host, dims=dims, process_group=pg,
                                       cell_range=cr if world > 1 else None, device=dev)
        return fn(e)

    ms = timed(step, E2E_STEPS, 3, world)
    check = None
    if resident is not None:  # the host path must give the resident path's depths
        r = step()
        check = {"max_abs_depth_diff_vs_resident": float(np.abs(r.depth - resident.depth).max()),
                 "ranks_equal_resident": bool(np.array_equal(r.rank, resident.rank))}
    total = n * int(np.prod(dims))
    probe = h2d_probe(host, dev)
    path = ("depth_pid_mean(pinned host tensor): cell slabs of "
            f"{D.STREAM_SLAB_BYTES >> 20} MB, H2D on a side stream overlapped with in-place "
            "validation + K5 on two HBM slab buffers, fixed-order slab sum, K4, result D2H"
            if streamed else
            "DeviceEnsemble.from_tensor(pinned host tensor) (pitched H2D + device validation) "
            "+ the method + result D2H")
    return {"value": total / (ms * 1e-3), "unit": "member-voxels/s", "ms_per_step": ms,
            "steps": E2E_STEPS, "warmup": 3,
            "h2d_bytes_per_step": n * m * 4, "d2h_bytes_per_step": (5 * n + n + 1) * 8,
            "h2d_GBps_effective": n * m * 4 / (ms * 1e-3) / 1e9,
            "h2d_GBps_probe": probe,
            "frac_of_h2d_probe": n * m * 4 / (ms * 1e-3) / 1e9 / probe if probe else None,
            "bound": "PCIe host-to-device copy", "path": path, "check": check}


def h2d_probe(host, dev, nbytes=4 << 30):
    """Plain pinned H2D bandwidth on this box (best of 3 copies of up to
    4 GB of the e2e host buffer): the e2e roofline."""
    import torch

    flat = host.reshape(-1).view(torch.uint8)
    k = min(nbytes, flat.numel())
    dst = torch.empty(k, dtype=torch.uint8, device=dev)
    best = 0.0
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(flat[:k], non_blocking=True)
        b.record()
        b.synchronize()
        best = max(best, k / (a.elapsed_time(b) * 1e-3) / 1e9)
    del dst
    return best


# cuBLAS TF32 / INT8 dense GEMM peaks measured on this pool's B200 by
# tools/probe_box.sh (8192^3, best of 20; profiles/r01_probe_box.log).
TF32_TFLOPS_PROBE = 747.2
READ_STREAM_PEAK_GBS = 7227.4  # TMA 2D read stream, 512-B rows (profiles/r01_ubench_tma.log)
# INT8 tensor peak: the higher of cuBLAS's int8 GEMM (3004.5 TOP/s) and our
# tcgen05 kind::i8 issue-rate microbenchmark (tools/ubench_mma.cu, 128x128x32
# MMAs, profiles/r02_ubench_mma.log: 4425 TOP/s); the roofline uses the max.
INT8_TOPS_PROBE = 4425.0


def run_pid_secondary(args, rank, world, pg, dev, pk):
    import torch

    import paper_2512_15187_b200 as pb
    from paper_2512_15187_b200 import depth as D
    from paper_2512_15187_b200 import synth

    res, n = 256, 1000
    shard = (rank, world) if world > 1 else None
    de = synth.ellipsoids_device(res, n, 0, 0, device=dev, shard=shard, process_group=pg)
    torch.cuda.synchronize()
    mv = n * res ** 3
    out = {"workload": "cfg4: PID, 1000 fuzzy ellipsoids 256^3 fp32 (67.1 GB)", "unit": "member-voxels/s"}
    results = {}
    for alg in ("factorized", "gram"):
        if alg == "gram" and not D._gram_available():
            continue
        D.KERNEL_EVENTS = []
        results[alg] = pb.depth_pid(de, algorithm=alg)
        D.KERNEL_EVENTS = []
        ms = timed(lambda: pb.depth_pid(de, algorithm=alg), max(1, min(args.steps, 5)), 2, world)
        ev = D.KERNEL_EVENTS
        D.KERNEL_EVENTS = None
        o = {"ms_per_depth": ms, "value": mv / (ms * 1e-3),
             "pair_voxels_per_s": n * n * res ** 3 / (ms * 1e-3)}
        if alg == "factorized":
            k1, _ = kernel_ms(ev, "pidb_pid_mean_partials")
            k2, _ = kernel_ms(ev, "pidb_pid_colsums")
            b = n * de.m * 4
            ach = 2 * b / ((k1 + k2) * 1e-3) / 1e9
            o["roofline"] = {"bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                             "frac": ach / pk["hbm_gbs"], "kernels_ms": [k1, k2],
                             "algorithmic_bytes": 2 * b, "note": "exact fp64, two HBM passes"}
        else:
            kg, _ = kernel_ms(ev, "pidb_gram_fixed_sums")
            kp, _ = kernel_ms(ev, "pidb_fixed_pack")
            flops = n * (n + 1) * de.m  # symmetric Gram, 2 flops per MAC
            ach = flops / (kg * 1e-3) / 1e12
            nib = (n + 127) // 128
            executed = nib * (nib + 1) // 2 * ((de.m + 31) // 32) * 10 * 2 * 128 * 128 * 32
            mode_peak = INT8_TOPS_PROBE / 10  # 10 digit-pair int8 MMAs per product
            o["roofline"] = {"bound": "tensor",
                             "kernel": "gram_fx_kernel (K1x: fixed-point digits, tcgen05 kind::i8, "
                                       "exact int32 accumulation, fused PID sums)",
                             "achieved": ach, "unit": "TFLOP/s", "peak": mode_peak,
                             "frac": ach / mode_peak,
                             "peak_src": "INT8 tensor peak (tcgen05 microbenchmark, 4425 TOP/s) / 10 "
                                         "(10 digit-pair MMAs per product)",
                             "frac_vs_tf32x3": ach / (TF32_TFLOPS_PROBE / 3),
                             "executed_int8_ops": executed,
                             "executed_frac_of_int8_peak": executed / (kg * 1e-3) / 1e12 / INT8_TOPS_PROBE,
                             "kernel_ms": kg, "pack_ms": kp, "algorithmic_flops": flops,
                             "traffic": ncu_traffic("cfg4_gram", world),
                             "traffic_note": "ncu DRAM read+write bytes of one K1x launch at cfg4 "
                                             "(profiles/r02_traffic.json): 1.7x the unique digit bytes"}
            o["certifier"] = dict(D.LAST_GRAM_CERT)
        out[alg] = o
    if len(results) == 2:
        a, b = results["gram"], results["factorized"]
        out["gram_vs_exact"] = {
            "max_abs_depth_err": float(np.abs(a.depth - b.depth).max()),
            "max_rel_depth_err": float(np.abs(a.depth - b.depth).max() / np.abs(b.depth).max()),
            "rank_mismatches": int(np.sum(a.rank != b.rank)),
            "min_depth_gap": float(np.min(np.diff(np.sort(b.depth))))}
    if rank == 0 and world == 1 and not args.no_parity:
        out["parity_1000x64"] = _guarded("cfg4 1000x64^3 parity", parity_pid_reduced, dev)
    out["ms_per_depth"] = out["factorized"]["ms_per_depth"]
    out["value"] = out["factorized"]["value"]
    out["algorithm"] = "factorized (exact, default)"
    if rank == 0 and world == 1 and not args.no_cpu:
        planes = 8
        lo = (res // 2 - planes // 2) * res * res
        U = de.values[: args.ref_pid_members, lo:lo + planes * res * res].cpu().numpy()
        out["cpu_baseline"] = cpu_pair_baseline(U, "pid", n, res ** 3,
                                                f"{planes} central planes of cfg4")
    del de
    torch.cuda.empty_cache()
    return out


def run_eid_secondary(args, dev, pk):
    """cfg2: eID on 500 binary Fourier contours 512^2 (reference generator),
    bit-exact integer path: K6 binary check + K7 pack + K2 tcgen05 i8 Gram +
    exact epilogue."""
    import torch

    import paper_2512_15187_b200 as pb
    from paper_2512_15187_b200 import depth as D
    from paper_2512_15187_b200 import synth

    n, res = 500, 512
    de = synth.contours_device(n, res, 0, device=dev)
    torch.cuda.synchronize()
    D.KERNEL_EVENTS = []
    pb.depth_eid(de)
    D.KERNEL_EVENTS = []
    ms = timed(lambda: pb.depth_eid(de), max(1, min(args.steps, 10)), 3, 1)
    ev = D.KERNEL_EVENTS
    D.KERNEL_EVENTS = None
    # the same calls without the per-kernel event hooks: repeated calls on one
    # DeviceEnsemble then replay a captured CUDA graph
    ms_graph = timed(lambda: pb.depth_eid(de), max(1, min(args.steps, 10)), 3, 1)
    kg, _ = kernel_ms(ev, "pidb_gram_i8")
    kp, _ = kernel_ms(ev, "pidb_binary_pack")
    cpu = None
    if not args.no_cpu:
        U = de.values[:100, : res * res].cpu().numpy()
        cpu = cpu_pair_baseline(U, "eid", n, res * res, "cfg2 (full 512^2 grid)")
    m = res * res
    ops = float(n) * (n + 1) * m  # symmetric Gram (upper triangle), 2 ops per MAC
    out = {"workload": "cfg2: eID, 500 binary contours 512^2 (bit-exact integer path)",
           "ms_per_depth": ms, "value": n * m / (ms * 1e-3), "unit": "member-voxels/s",
           "pair_voxels_per_s": n * n * m / (ms * 1e-3),
           "gram_roofline": {"bound": "tensor", "kernel": "gram_i8_kernel (+int64 reduce)",
                             "achieved": ops / (kg * 1e-3) / 1e12, "unit": "TOP/s",
                             "peak": INT8_TOPS_PROBE, "frac": ops / (kg * 1e-3) / 1e12 / INT8_TOPS_PROBE,
                             "kernel_ms": kg, "algorithmic_ops": ops,
                             "peak_src": "INT8 tensor peak (tcgen05 microbenchmark, profiles/r02_ubench_mma.log)"},
           # eID is bound by max(int8 tensor time, HBM time to
           # read the fp32 input); the input read is the floor here
           "hbm_roofline": {"bound": "hbm", "algorithmic_bytes": n * m * 4,
                            "floor_ms": n * m * 4 / (pk["hbm_gbs"] * 1e9) * 1e3,
                            "frac_whole_call": n * m * 4 / (pk["hbm_gbs"] * 1e9) / (ms_graph * 1e-3),
                            "pack_kernel_ms": kp,
                            "pack_achieved_GBps": (n * m * 5) / (kp * 1e-3) / 1e9 if kp else None,
                            "pack_note": "K7 reads 4 B and writes 1 B per member-voxel"},
           "ms_per_depth_graph": ms_graph}
    # the same members held as bytes (a bool ensemble): K2 loads them by TMA,
    # no pack pass; the input floor drops to 1 B per member-voxel
    ref = pb.depth_eid(de)
    db = pb.stage(de.values[:, :m] != 0)
    D.KERNEL_EVENTS = []
    rb = pb.depth_eid(db)
    D.KERNEL_EVENTS = []
    ms_b = timed(lambda: pb.depth_eid(db), max(1, min(args.steps, 10)), 3, 1)
    evb = D.KERNEL_EVENTS
    D.KERNEL_EVENTS = None
    ms_bg = timed(lambda: pb.depth_eid(db), max(1, min(args.steps, 10)), 3, 1)
    kb, _ = kernel_ms(evb, "pidb_gram_i8_bytes")
    out["byte_ensemble"] = {
        "input": "the cfg2 members as a bool tensor (1 B per member-voxel), pb.stage(bool)",
        "ms_per_depth": ms_b, "ms_per_depth_graph": ms_bg,
        "value": n * m / (ms_bg * 1e-3), "unit": "member-voxels/s",
        "gram_kernel_ms": kb,
        "gram_frac_of_int8_peak": ops / (kb * 1e-3) / 1e12 / INT8_TOPS_PROBE if kb else None,
        "hbm_floor_ms": n * m / (pk["hbm_gbs"] * 1e9) * 1e3,
        "bit_identical_to_fp32_path": bool(np.array_equal(rb.depth, ref.depth)
                                           and np.array_equal(rb.in_in, ref.in_in)
                                           and np.array_equal(rb.in_out, ref.in_out)
                                           and np.array_equal(rb.rank, ref.rank))}
    del db
    if cpu is not None:
        out["cpu_baseline"] = cpu
    if not args.no_parity:
        out["parity_full"] = _guarded("cfg2 parity", parity_eid_full, de, ref)
    del de
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg5", choices=sorted(WORKLOADS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-pid", action="store_true")
    ap.add_argument("--no-eid", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--ref-planes", type=int, default=0)
    ap.add_argument("--ref-pid-members", type=int, default=64)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        run_reference(args, rank, world)
        return
    rank, world, local, pg = dist_setup()
    try:
        run_ours(args, rank, world, local, pg)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
