"""A/B of the result-block D2H of graph-replayed calls: pinned staging owned
by the graph vs a plain .cpu() (cfg1: 100 disks 256^2; device-event and wall
time per call).  python tools/ab_pinned_d2h.py"""
import sys, time
sys.path.insert(0, '.')
import torch, numpy as np
import paper_2512_15187_b200 as pb
from paper_2512_15187_b200 import synth, depth as D
de = synth.disks_device(256, 100, 0)
for _ in range(5): pb.depth_pid_mean(de)
torch.cuda.synchronize()
def bench(label):
    ts=[]
    for _ in range(300):
        a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
        a.record(); pb.depth_pid_mean(de); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    t0=time.perf_counter()
    for _ in range(300): pb.depth_pid_mean(de)
    wall=(time.perf_counter()-t0)/300*1e3
    print(label, "event ms median %.4f  wall ms %.4f" % (np.median(ts), wall))
bench("pinned")
for k,(g,outs,lock) in de._cache["graphs"].items(): outs._pinned=None
bench("cpu()")
