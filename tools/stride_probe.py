"""Does the member row stride (ld) change K5's bandwidth?
python tools/stride_probe.py N RES PAD...   (PAD: extra fp32 elements per row)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2512_15187_b200 as pb  # noqa: E402
from paper_2512_15187_b200 import synth  # noqa: E402
from paper_2512_15187_b200.device import DeviceEnsemble  # noqa: E402

n, res = int(sys.argv[1]), int(sys.argv[2])
base = synth.ellipsoids_device(res, n, 0, 0)
m = base.m
for pad in map(int, sys.argv[3:]):
    big = torch.zeros((n, base.ld + pad), dtype=torch.float32, device="cuda")
    big[:, :base.ld] = base.values
    de = DeviceEnsemble(values=big[:, :base.ld], m=m, dims=base.dims, ids=base.ids)
    for _ in range(3):
        r = pb.depth_pid_mean(de)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    s.record()
    for _ in range(reps):
        pb.depth_pid_mean(de)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    ok = bool((r.depth == pb.depth_pid_mean(base).depth).all())
    print(f"n={n} res={res} ld={de.ld} (+{pad}): {ms:.3f} ms  {n * m * 4 / ms / 1e9:.2f} TB/s  same={ok}")
    del big, de
