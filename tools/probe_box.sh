#!/bin/bash
# One-off GPU-box probe: host resources + measured TF32/INT8 GEMM peaks (cuBLAS via torch).
nvidia-smi
free -g
nproc
lscpu | head -20
df -h /tmp /dev/shm
cat /sys/fs/cgroup/memory.max 2>/dev/null
python - <<'PY'
import torch, time, os
print(torch.cuda.get_device_properties(0), os.cpu_count())
def bench(fn, flops, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    best=1e9
    for _ in range(n):
        s.record(); fn(); e.record(); torch.cuda.synchronize(); best=min(best,s.elapsed_time(e))
    return flops/(best*1e-3)/1e12
n=8192
a=torch.randn(n,n,device='cuda'); b=torch.randn(n,n,device='cuda')
torch.backends.cuda.matmul.allow_tf32=True
print("tf32 TFLOP/s", bench(lambda: a@b, 2*n**3))
torch.backends.cuda.matmul.allow_tf32=False
print("fp32 TFLOP/s", bench(lambda: a@b, 2*n**3, 5))
ai=torch.randint(-128,127,(n,n),device='cuda',dtype=torch.int8); bi=torch.randint(-128,127,(n,n),device='cuda',dtype=torch.int8).t()
try:
    print("int8 TOP/s", bench(lambda: torch._int_mm(ai,bi), 2*n**3))
except Exception as ex: print("int8 fail", ex)
ah=a.half(); bh=b.half()
print("fp16 TFLOP/s", bench(lambda: ah@bh, 2*n**3))
x=torch.empty(2**30, dtype=torch.float32, device='cuda')
print("read GB/s (sum)", bench(lambda: x.sum(), 4*2**30)/1e-3/1e3)
PY
