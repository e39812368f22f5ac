"""Small driver for timing / ncu captures of the streaming kernels:
python tools/prof_k5.py N RES [pid-mean|pid|pid:gram|dice|mass|eid|eid:bits] [reps]
(eid: N binary Fourier contours on a RES^2 grid, as fp32; eid:bits the same
contours as a byte ensemble)
Prints the per-call time and the per-kernel device times (CUDA events around
each native launch, depth.KERNEL_EVENTS)."""
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2512_15187_b200 as pb  # noqa: E402
from paper_2512_15187_b200 import depth as D  # noqa: E402
from paper_2512_15187_b200 import synth  # noqa: E402

n, res = int(sys.argv[1]), int(sys.argv[2])
method = sys.argv[3] if len(sys.argv) > 3 else "pid-mean"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
eid = method.startswith("eid")
de = synth.contours_device(n, res, 0) if eid else synth.ellipsoids_device(res, n, 0, 0)
if method == "eid:bits":
    de = pb.stage(de.values[:, :de.m] != 0)
if eid:
    fn = pb.depth_eid
elif method == "pid-mean":
    fn = pb.depth_pid_mean
elif method == "mass":
    fn = pb.member_masses
elif method == "dice":
    fn = lambda d: pb.depth_similarity_baseline(d, "dice")  # noqa: E731
else:
    algo = method.split(":")[1] if ":" in method else "factorized"
    fn = lambda d: pb.depth_pid(d, algorithm=algo)  # noqa: E731
for _ in range(reps):
    fn(de)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(reps):
    fn(de)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
D.KERNEL_EVENTS = []
for _ in range(reps):
    fn(de)
torch.cuda.synchronize()
per = defaultdict(float)
for name, a, b in D.KERNEL_EVENTS:
    per[name] += a.elapsed_time(b) / reps
D.KERNEL_EVENTS = None
gb = n * (res**2 if eid else res**3) * (1 if method == "eid:bits" else 4) / 1e9
kern = " ".join(f"{k}={v:.3f}ms({gb / v:.0f}TB/s)" for k, v in per.items())
print(f"n={n} res={res} {method}: {ms:.3f} ms/call | {kern}")
