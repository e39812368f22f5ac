"""Small driver for ncu captures of the streaming kernels:
python tools/prof_k5.py N RES [pid-mean|pid] [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2512_15187_b200 as pb  # noqa: E402
from paper_2512_15187_b200 import synth  # noqa: E402

n, res = int(sys.argv[1]), int(sys.argv[2])
method = sys.argv[3] if len(sys.argv) > 3 else "pid-mean"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
de = synth.ellipsoids_device(res, n, 0, 0)
fn = pb.depth_pid_mean if method == "pid-mean" else (lambda d: pb.depth_pid(d, algorithm=method.split(":")[1] if ":" in method else "factorized"))
for _ in range(reps):
    r = fn(de)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(reps):
    fn(de)
e.record()
torch.cuda.synchronize()
print(f"n={n} res={res} {method}: {s.elapsed_time(e) / reps:.3f} ms/call, "
      f"{n * res**3 * 4 / (s.elapsed_time(e) / reps * 1e-3) / 1e9:.0f} GB/s (1 pass equiv)")
