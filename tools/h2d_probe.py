"""H2D bandwidth from pinned host memory (the e2e bound): one stream vs two
concurrent streams, plain vs pitched (2D) copies.  python tools/h2d_probe.py [GB]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2512_15187_b200 import _native as N  # noqa: E402

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 8.0
n = int(gb * (1 << 30)) // 4
host = torch.empty(n, dtype=torch.float32, pin_memory=True)
host.fill_(0.5)
dev = torch.empty(n, dtype=torch.float32, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]


def run(k, pitched=False, reps=3):
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        part = n // k
        for i, s in enumerate(streams[:k]):
            s.wait_event(a)
            with torch.cuda.stream(s):
                if pitched:  # rows of 4096 floats, pitch 4096 (same bytes, 2D engine path)
                    rows = part // 4096
                    N.call("pidb_copy_rows", dev[i * part:].data_ptr(), 4096 * 4,
                           host[i * part:].data_ptr(), 4096 * 4, 4096 * 4, rows, s.cuda_stream)
                else:
                    dev[i * part:(i + 1) * part].copy_(host[i * part:(i + 1) * part], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s)
            torch.cuda.current_stream().wait_event(ev)
        b.record()
        b.synchronize()
        best = max(best, n * 4 / (a.elapsed_time(b) * 1e-3) / 1e9)
    return best


for k in (1, 2, 4):
    print(f"H2D {gb:.0f} GB, {k} stream(s): {run(k):.1f} GB/s; pitched: {run(k, True):.1f} GB/s",
          flush=True)
