"""Timing of the streaming kernels on float64 members and the masses-only
mode: python tools/prof_f64.py N M reps"""
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2512_15187_b200 as pb  # noqa: E402
from paper_2512_15187_b200 import depth as D  # noqa: E402

n, m, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
for dt in (torch.float64, torch.float32):
    u = torch.rand(n, m, dtype=dt, device="cuda")
    de = pb.DeviceEnsemble.from_tensor(u)
    for name, fn in (("pid-mean", pb.depth_pid_mean), ("masses", pb.member_masses),
                     ("pid", pb.depth_pid)):
        fn(de)
        D.KERNEL_EVENTS = []
        for _ in range(reps):
            fn(de)
        torch.cuda.synchronize()
        per = defaultdict(float)
        for k, a, b in D.KERNEL_EVENTS:
            per[k] += a.elapsed_time(b) / reps
        D.KERNEL_EVENTS = None
        gb = n * m * u.element_size() / 1e9
        print(f"{str(dt)[6:]} n={n} m={m} {name}: " +
              " ".join(f"{k}={v:.3f}ms({gb / v:.2f}TB/s)" for k, v in per.items()))
    del de, u
    torch.cuda.empty_cache()
