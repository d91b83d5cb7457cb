#!/bin/bash
# Profiling recipe (run under gpurun on ONE B200; /opt/skills/guides/B200_PROFILING.md).
#   1. the plain command must exit 0 first;
#   2. launch list of one V-cycle (cold-cache, serialised: compare shares);
#   3. full-set captures: one smoother step per level and the local corrections.
# Kernels are selected by the NVTX ranges of tools/profile_driver.py.
# Usage: bash profiles/run_ncu.sh <tag> [--workload C2]
set -u
TAG=${1:-r01}
shift || true
OUT=gpurun_out
mkdir -p $OUT
CMD="python tools/profile_driver.py $*"
if ! $CMD > $OUT/plain_$TAG.log 2>&1; then echo "plain run failed"; exit 1; fi
ncu --nvtx --nvtx-include "vcycle/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launch_$TAG.log 2>&1
echo "launch list: $?"
ncu --nvtx --nvtx-include "sweeps/" -k regex:"csr_tile_kernel|sell_kernel" --set full --clock-control none --import-source on \
    -o $OUT/prof_sweeps_$TAG $CMD > $OUT/ncu_sweeps_$TAG.log 2>&1
echo "sweeps: $?"
ncu --nvtx --nvtx-include "lc/" -k regex:patch_kernel --set full --clock-control none --import-source on \
    -o $OUT/prof_lc_$TAG $CMD > $OUT/ncu_lc_$TAG.log 2>&1
echo "lc: $?"
