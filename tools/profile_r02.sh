#!/usr/bin/env bash
# Round-2 ncu evidence (run on the B200 through gpurun; each ncu command only
# after the same command ran clean without ncu).  Outputs in gpurun_out/.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum
# 1. launch list of the bench command (timing legs only; CPU legs launch nothing)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02_launches_cfg5.csv \
    python bench.py --steps 2 --warmup 3 --no-parity --no-cpu --no-e2e \
    > gpurun_out/r02_ncu_launch_bench.log 2>&1
echo "launch list rc=$?"
# 2. DRAM bytes per launch, whole-application replay (no memory save/restore)
ncu --replay-mode application --metrics $M -k regex:rows_ws_kernel -c 1 --csv \
    --log-file gpurun_out/r02_ncu_k5_cfg5_dram.csv python tools/prof_k5.py 200 512 pid-mean 1 \
    > /dev/null 2>&1
echo "k5 cfg5 dram rc=$?"
ncu --replay-mode application --metrics $M -k 'regex:gram_fx_kernel|fx_pack_kernel' -c 2 --csv \
    --log-file gpurun_out/r02_ncu_k1x_cfg4_dram.csv python tools/prof_k5.py 1000 256 pid:gram 1 \
    > /dev/null 2>&1
echo "k1x cfg4 dram rc=$?"
# 3. full sets (kernel replay) at 1000 x 128^3
ncu --set full --import-source on -k regex:gram_fx_kernel -c 1 -o gpurun_out/r02_ncu_k1x_full \
    python tools/prof_k5.py 1000 128 pid:gram 1 > /dev/null 2>&1
echo "k1x full rc=$?"
ncu --set full --import-source on -k regex:fx_pack_kernel -c 1 -o gpurun_out/r02_ncu_pack_full \
    python tools/prof_k5.py 1000 128 pid:gram 1 > /dev/null 2>&1
echo "pack full rc=$?"
