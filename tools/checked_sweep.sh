#!/usr/bin/env bash
# Substitute for compute-sanitizer memcheck (refused on the GPU pool,
# profiles/r02_sanitizer_refused.log): run every kernel variant at small and
# ragged shapes (tools/sweep_cases.py) and the GPU parity tests against the
# device-bounds-checked build libpidb_checked.so (PIDB_DCHECK asserts on the
# packed-tile, operand-tile and partial-slot indices; a failed check prints
# the site and traps), plus CUDA_LAUNCH_BLOCKING=1 so an async fault is
# attributed to its launch.  Build it first (in the build container):
#   python -m paper_2512_15187_b200._build --checked
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PIDB_LIB="$PWD/paper_2512_15187_b200/libpidb_checked.so" CUDA_LAUNCH_BLOCKING=1
test -f "$PIDB_LIB" || { echo "missing $PIDB_LIB"; exit 2; }
PIDB_GRAPHS=0 timeout 1200 python tools/sweep_cases.py > gpurun_out/checked_sweep.log 2>&1
echo "sweep rc=$? $(grep -c 'device check failed' gpurun_out/checked_sweep.log) failed checks"
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -q -x \
    -p no:cacheprovider > gpurun_out/checked_pytest.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/checked_pytest.log)"
grep -h "device check failed" gpurun_out/checked_*.log | head
