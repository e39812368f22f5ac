"""Crash sweep over small cases (compute-sanitizer is not available on the pool)
over every streaming-kernel variant: rows (WS and plain), cluster WS, chunked,
wide, plus eID, Gram, boxplot."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_15187_b200 as pb  # noqa: E402

rng = np.random.default_rng(0)
for n, m, w in ((40, 3000, False), (200, 2100, True), (300, 700, True), (700, 500, False),
                (2600, 130, True), (4200, 70, False)):
    U = rng.uniform(size=(n, m)).astype(np.float32)
    wt = rng.uniform(0.5, 2, size=m) if w else None
    de = pb.DeviceEnsemble.from_tensor(torch.from_numpy(U), wt)
    for meth in ("pid-mean", "pid", "dice"):
        pb.depth_by_method(de, meth)
    pb.member_masses(de)
    d64 = pb.DeviceEnsemble.from_tensor(torch.from_numpy(U.astype(np.float64)), wt)
    pb.depth_pid_mean(d64)
    print("ok", n, m, flush=True)
B = (rng.uniform(size=(130, 1000)) < 0.5).astype(np.float32)
de = pb.DeviceEnsemble.from_tensor(torch.from_numpy(B))
r = pb.depth_eid(de)
pb.depth_pid(de, algorithm="gram")
pb.boxplot.band_envelopes(de, r.rank, [13, 65, 130], 0.5)
print("ok eid/gram/boxplot", flush=True)
