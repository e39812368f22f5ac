"""Multi-rank check of the voxel-sharded depth path on real kernels.

Run under torchrun; with PIDB_BENCH_SHARE_GPU=1 every rank uses cuda:0 and
gloo collectives (one-GPU environments), otherwise one GPU per rank and NCCL.
Each rank stages only its cell slab (shard_bounds) and calls the public API
with the process group; rank 0 compares with a single-process run on the
whole ensemble.
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/dist_check.py
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2512_15187_b200 as pb  # noqa: E402

share = os.environ.get("PIDB_BENCH_SHARE_GPU") == "1"
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = 0 if share else int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("gloo" if share else "nccl")
pg = dist.group.WORLD

rng = np.random.default_rng(5)
cases = [("fuzzy", 300, (24, 20, 18), True), ("fuzzy", 120, (64, 70), False),
         ("binary", 200, (40, 41), False)]
ok = True
for kind, n, dims, weighted in cases:
    m = int(np.prod(dims))
    if kind == "fuzzy":
        U = rng.uniform(size=(n, m)).astype(np.float32)
    else:
        U = (rng.uniform(size=(n, m)) < rng.uniform(0.2, 0.8, size=(n, 1))).astype(np.float32)
    w = rng.uniform(0.5, 2.0, size=m) if weighted else None
    lo, hi = pb.shard_bounds(m, rank, world)
    de = pb.DeviceEnsemble.from_tensor(torch.from_numpy(U[:, lo:hi].copy()),
                                       None if w is None else w[lo:hi], dims=dims,
                                       process_group=pg, cell_range=(lo, hi))
    methods = ["pid-mean", "pid", "dice", "iou"] + (["eid"] if kind == "binary" else [])
    got = {mth: pb.depth_by_method(de, mth) for mth in methods}
    got["pid-gram"] = pb.depth_pid(de, algorithm="gram")  # K1x per shard + allreduce
    if kind == "binary":  # the slab as a byte ensemble: K2 from the bytes + allreduce
        db = pb.DeviceEnsemble.from_tensor(torch.from_numpy(U[:, lo:hi] != 0), dims=dims,
                                           process_group=pg, cell_range=(lo, hi))
        got["eid-bytes"] = pb.depth_eid(db)
        got["pid-bytes"] = pb.depth_pid(db)
    if rank == 0:
        full = pb.DeviceEnsemble.from_tensor(torch.from_numpy(U), w, dims=dims)
        for mth in methods + [k for k in ("pid-gram", "eid-bytes", "pid-bytes") if k in got]:
            want = pb.depth_by_method(full, {"pid-gram": "pid", "eid-bytes": "eid",
                                             "pid-bytes": "pid"}.get(mth, mth))
            err = float(np.abs(got[mth].depth - want.depth).max())
            same = bool(np.array_equal(got[mth].rank, want.rank))
            exact = bool(np.array_equal(got[mth].depth, want.depth))
            tol = 1e-8 if mth == "pid-gram" else 1e-12  # tensor-core Gram bound vs exact
            good = (exact if mth in ("eid", "eid-bytes") else err <= tol) and same
            ok &= good
            print(f"{kind} n={n} m={m} w={weighted} {mth}: max|d| diff {err:.2e} "
                  f"ranks {'equal' if same else 'DIFFER'}{' bit-exact' if exact else ''}"
                  f" -> {'ok' if good else 'FAIL'}", flush=True)
dist.barrier()
if rank == 0:
    print("dist_check", "PASSED" if ok else "FAILED", f"world={world}", flush=True)
dist.destroy_process_group()
sys.exit(0 if ok else 1)
