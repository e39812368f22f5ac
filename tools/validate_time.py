"""Times pidb_validate (the ProbMask value policy on the device) on 200 x 2^24
fp32 cells: python tools/validate_time.py"""
import torch, sys
sys.path.insert(0, '.')
from paper_2512_15187_b200 import _native as N
n, m = 200, 1 << 24
t = torch.rand(n, m, device='cuda')
stats = torch.empty(3, dtype=torch.int64, device='cuda')
s = torch.cuda.current_stream().cuda_stream
for clamp in (0, 1):
    for _ in range(2):
        N.call("pidb_validate", t.data_ptr(), N.PIDB_F32, n, m, m, clamp, stats.data_ptr(), s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(5):
        N.call("pidb_validate", t.data_ptr(), N.PIDB_F32, n, m, m, clamp, stats.data_ptr(), s)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"validate clamp={clamp} {n}x{m}: {ms:.3f} ms, {n*m*4/ms/1e6:.0f} GB/s")
