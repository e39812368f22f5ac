"""Ingestion timing: a manifest of N float32 .npy members (RES^3) written to
a scratch directory, then staged into HBM by stage_manifest (memory-mapped
reads + pinned double buffer + async H2D + device validation) and, for
comparison, by the lazy read_manifest + stage path.
python tools/ingest_bench.py N RES DIR"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_15187_b200 as pb  # noqa: E402

n, res, d = int(sys.argv[1]), int(sys.argv[2]), Path(sys.argv[3])
(d / "members").mkdir(parents=True, exist_ok=True)
de = pb.gen_ellipsoid_ensemble(res, n, 0, 0)
vals = de.values[:, :de.m].cpu().numpy()
entries = []
for i in range(n):
    np.save(d / "members" / f"m{i:04d}.npy", vals[i].reshape(res, res, res))
    entries.append({"id": f"m{i:04d}", "path": f"members/m{i:04d}.npy"})
pb.write_manifest(d / "manifest.json", (res, res, res), entries)
del de
gb = n * res ** 3 * 4 / 1e9
for name, fn in (("stage_manifest", lambda: pb.stage_manifest(d / "manifest.json")),
                 ("read_manifest+stage", lambda: pb.stage(pb.read_manifest(d / "manifest.json")))):
    fn()  # page cache warm: time the host->HBM path, not the disk
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e = fn()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    r = pb.depth_pid_mean(e)
    print(f"{name}: {dt * 1e3:.1f} ms for {gb:.2f} GB ({gb / dt:.1f} GB/s), depth[0]={r.depth[0]:.6f}",
          flush=True)
    del e
