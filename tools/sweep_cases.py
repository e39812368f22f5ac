"""Small cases over every kernel variant, for compute-sanitizer
(memcheck / racecheck / synccheck; tools/sanitize.sh) and as a crash sweep:
K5/K9 rows (WS and plain), cluster WS, chunked, wide/ext (n > 4096), fp64
members, K6 masses, similarity, K7 pack + K2 i8 Gram + exact epilogue, the
tensor-core PID Gram (fused sums) and the full Gram, byte-ensemble eID
(K7 count-only + K2 from the bytes), the fp64 gram_block
seam, K8 pair sums, mean mask, validation, K10 band envelopes.
``--quick`` keeps one case per variant (racecheck is slow)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_15187_b200 as pb  # noqa: E402
from paper_2512_15187_b200 import reduction  # noqa: E402

quick = "--quick" in sys.argv
rng = np.random.default_rng(0)
cases = ((40, 3000, False), (200, 2100, True), (300, 700, True), (700, 500, False),
         (2600, 130, True), (4200, 70, False))
if quick:
    cases = ((40, 3000, False), (300, 700, True), (2600, 130, True), (4200, 70, False))
for n, m, w in cases:
    U = rng.uniform(size=(n, m)).astype(np.float32)
    wt = rng.uniform(0.5, 2, size=m) if w else None
    de = pb.DeviceEnsemble.from_tensor(torch.from_numpy(U), wt)
    for meth in ("pid-mean", "pid", "dice"):
        pb.depth_by_method(de, meth)
    pb.member_masses(de)
    de.mean_values()
    d64 = pb.DeviceEnsemble.from_tensor(torch.from_numpy(U.astype(np.float64)), wt)
    pb.depth_pid_mean(d64)
    print("ok", n, m, flush=True)
B = (rng.uniform(size=(130, 1000)) < 0.5).astype(np.float32)
de = pb.DeviceEnsemble.from_tensor(torch.from_numpy(B))
r = pb.depth_eid(de)
pb.depth_pid(de, algorithm="gram")
reduction.gram_device(de)
pb.boxplot.band_envelopes(de, r.rank, [13, 65, 130], 0.5)
for nb, mb in ((130, 1000), (257, 129), (3, 17)):  # byte ensembles: K7 count-only + K2 by TMA
    Bb = rng.uniform(size=(nb, mb)) < 0.5
    pb.depth_eid(torch.from_numpy(Bb))
    pb.depth_eid(torch.from_numpy(Bb.astype(np.uint8)))
print("ok eid/gram/boxplot/bytes", flush=True)
a = rng.uniform(size=(37, 1001))
b = rng.uniform(size=(70, 1001)).astype(np.float32)
reduction.gram_block(a, b, rng.uniform(0.5, 2, size=1001), complement_cols=True)
reduction.gram_block(b, b)
g = pb.GridSpec((1001,))
pb.prob_inclusion(pb.ProbMask(g, a[0]), pb.ProbMask(g, b[0]))
pb.fuzzy_dice(pb.ProbMask(g, a[1]), pb.ProbMask(g, b[1]))
print("ok gram_block/pairs", flush=True)
torch.cuda.synchronize()
