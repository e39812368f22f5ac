"""Where the time between consecutive depth_pid_mean calls goes on a staged
ensemble: python tools/step_gap.py N RES  (per-call wall/GPU time with graph
replay, the K5 launch alone by CUDA events, and the GPU idle gap)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2512_15187_b200 as pb  # noqa: E402
from paper_2512_15187_b200 import depth as D  # noqa: E402
from paper_2512_15187_b200 import synth  # noqa: E402

n, res = int(sys.argv[1]), int(sys.argv[2])
de = synth.ellipsoids_device(res, n, 0, 0)
for _ in range(3):
    pb.depth_pid_mean(de)
torch.cuda.synchronize()
reps = 10
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
t0 = time.perf_counter()
for i in range(reps):
    ev[2 * i].record()
    pb.depth_pid_mean(de)
    ev[2 * i + 1].record()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / reps * 1e3
inside = sum(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(reps)) / reps
between = sum(ev[2 * i + 1].elapsed_time(ev[2 * i + 2]) for i in range(reps - 1)) / (reps - 1)
D.KERNEL_EVENTS = []
for _ in range(reps):
    pb.depth_pid_mean(de)
torch.cuda.synchronize()
k5 = sum(a.elapsed_time(b) for nm, a, b in D.KERNEL_EVENTS if nm == "pidb_pid_mean_partials") / reps
D.KERNEL_EVENTS = None
print(f"n={n} res={res}: wall {wall:.3f} ms/call, GPU inside call {inside:.3f} ms, "
      f"GPU gap between calls {between:.3f} ms, K5 alone (eager, events) {k5:.3f} ms")
