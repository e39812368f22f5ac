"""Does the K7 pack overlap with a concurrent K2 Gram?  (cfg2 shapes)
Runs pack(A) and gram_i8(B) back to back on one stream, then concurrently on
two streams, and reports the device times.  python tools/ab_eid_overlap.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_15187_b200 import _native as N  # noqa: E402
from paper_2512_15187_b200 import synth  # noqa: E402

lib = N.load()
de = synth.contours_device(500, 512, 0)
n, m = de.n, de.m
nb_ = int(lib.pidb_binary_pack_bytes(n, m))
tiles = [torch.zeros(nb_ + 1024, dtype=torch.uint8, device="cuda") for _ in range(2)]
tp = [t.data_ptr() + ((-t.data_ptr()) % 1024) for t in tiles]
nb = torch.zeros(n, dtype=torch.int64, device="cuda")
g = torch.empty((n, n), dtype=torch.int64, device="cuda")
ws = torch.zeros(lib.pidb_gram_i8_workspace_bytes(n, m), dtype=torch.uint8, device="cuda")
S1, S2 = torch.cuda.Stream(), torch.cuda.Stream()


def pack(t, s):
    N.call("pidb_binary_pack", de.ptr(), de.dtype_code, n, m, de.ld, tp[t], nb.data_ptr(), s.cuda_stream)


def gram(t, s):
    N.call("pidb_gram_i8", tp[t], n, m, g.data_ptr(), ws.data_ptr(), ws.numel(), s.cuda_stream)


pack(0, S1), pack(1, S1)
torch.cuda.synchronize()


def timeit(fn, reps=50):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)) * 1e3


cur = torch.cuda.current_stream()


def seq():
    pack(0, cur)
    gram(1, cur)


def par():
    e = torch.cuda.Event()
    e.record(cur)
    S1.wait_event(e)
    S2.wait_event(e)
    pack(0, S1)
    gram(1, S2)
    for s in (S1, S2):
        x = torch.cuda.Event()
        x.record(s)
        cur.wait_event(x)


print(f"pack alone {timeit(lambda: pack(0, cur)):.1f} us, gram alone {timeit(lambda: gram(1, cur)):.1f} us")
print(f"sequential {timeit(seq):.1f} us, concurrent {timeit(par):.1f} us")
