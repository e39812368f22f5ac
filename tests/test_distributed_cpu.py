"""Multi-GPU host logic on CPU: world_size 2 over gloo.

Each rank holds a contiguous cell slab of every member (shard_bounds), forms
the additive per-shard partial sums that K5 / K9 produce on a GPU (computed
here with numpy), combines them with the package's allreduce helper and runs
the K4 epilogue arithmetic; the result must equal the single-process oracle.
This pins the sharding/partial/allreduce decomposition; the
GPU kernels themselves are pinned by tests/test_gpu_parity.py.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import make_fuzzy
from oracle import port


class _Shard:
    def __init__(self, pg):
        self.process_group = pg


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port_, U, w, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_15187_b200 import shard_bounds
        from paper_2512_15187_b200.depth import _allreduce

        n, m = U.shape
        lo, hi = shard_bounds(m, rank, world)
        Us = U[:, lo:hi].astype(np.float64)
        ws = np.ones(hi - lo) if w is None else w[lo:hi]
        de = _Shard(dist.group.WORLD)
        # --- K5 partials of this shard: [row_plain | mass | col_mean]
        S = Us.sum(0)
        buf = torch.from_numpy(np.concatenate([(Us * ws) @ S, (Us * ws).sum(1), [(ws * S).sum()]]))
        _allreduce(buf, de)
        row, mass, col = buf[:n].numpy(), buf[n:2 * n].numpy(), float(buf[2 * n])
        # PID-mean epilogue (K4, depth.py:274-278)
        inv = np.where(mass > 0, 1.0 / np.where(mass > 0, mass, 1), 0.0)
        num = row / n
        pm = np.minimum(num * inv, num / (col / n))
        # --- K9: masses are global now; per-shard T-weighted column sums
        T = (inv[:, None] * Us).sum(0)
        colinv = torch.from_numpy((Us * ws) @ T)
        _allreduce(colinv, de)
        pid = np.minimum(inv * row / n, colinv.numpy() / n)
        if rank == 0:
            out["pm"] = pm
            out["pid"] = pid
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("weighted", [False, True])
def test_two_rank_voxel_sharding_matches_oracle(weighted):
    U, w = make_fuzzy(42, 11, (13, 17), weighted)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(2, _free_port(), U, w, out), nprocs=2, join=True,
                       start_method="fork")
    ref = port.depth_pid_mean(U, w)
    np.testing.assert_allclose(out["pm"], ref["depth"], rtol=0, atol=1e-13)
    ref = port.depth_pid(U, w)
    np.testing.assert_allclose(out["pid"], ref["depth"], rtol=0, atol=1e-13)
