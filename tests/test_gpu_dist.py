"""Multi-rank path on the real kernels: tools/dist_check.py under torchrun
with two or three ranks sharing the one GPU (gloo collectives;
PIDB_BENCH_SHARE_GPU=1), and one rank with the NCCL backend (the NCCL
allreduces of the sharded path on device buffers; NCCL refuses two ranks on
one GPU).  Each rank stages only its cell slab and calls the public API with
the process group; rank 0 compares with a single-process run."""
from __future__ import annotations

import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,backend", [(1, "nccl"), (2, "gloo"), (3, "gloo")])
def test_sharded_path_matches_single_process(world, backend):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    env = dict(os.environ, OMP_NUM_THREADS="1")
    if backend == "gloo":
        env["PIDB_BENCH_SHARE_GPU"] = "1"
    else:
        env.pop("PIDB_BENCH_SHARE_GPU", None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", str(ROOT / "tools" / "dist_check.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"dist_check PASSED world={world}" in r.stdout
