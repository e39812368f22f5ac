"""Host-side cost of one graph-replayed depth call on a small ensemble:
python tools/host_overhead.py [N RES2D calls]  (cProfile top entries + us/call)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2512_15187_b200 as pb  # noqa: E402
from paper_2512_15187_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
res = int(sys.argv[2]) if len(sys.argv) > 2 else 256
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
de = pb.DeviceEnsemble.from_tensor(torch.rand(n, res * res, device="cuda"), dims=(res, res))
for meth in ("pid-mean", "pid", "eid"):
    d = de
    if meth == "eid":
        d = pb.DeviceEnsemble.from_tensor((torch.rand(n, res * res, device="cuda") < 0.4).float(),
                                          dims=(res, res))
    for _ in range(5):
        pb.depth_by_method(d, meth)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(calls):
        pb.depth_by_method(d, meth)
    dt = (time.perf_counter() - t) / calls * 1e6
    print(f"{meth}: {dt:.1f} us per call (wall, includes the GPU work)")
pr = cProfile.Profile()
pr.enable()
for _ in range(calls):
    pb.depth_pid_mean(de)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
