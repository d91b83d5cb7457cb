#!/bin/bash
# Profiling recipe (run under gpurun on ONE B200; see /opt/skills/guides/B200_PROFILING.md).
#   1. the plain command must exit 0 first (same call, && chain);
#   2. launch list: every kernel's device time (cold-cache, serialised: compare shares);
#   3. full-set capture of the dominant kernel (fine-level Chebyshev step, Epi 4 = ChebNext).
# Usage: bash profiles/run_ncu.sh <tag> [extra bench args]
set -u
TAG=${1:-r01}
shift || true
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline $*"
$CMD > $OUT/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launch_$TAG.log 2>&1
# fine-level ChebNext launches start after the V-cycles (8 cycles x 16) in bench.py
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:Epi\)4' -s 140 -c 2 -o $OUT/prof_k3_$TAG $CMD > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu done: $?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:patch_kernel' -s 8 -c 1 -o $OUT/prof_lc_$TAG $CMD > $OUT/ncu_lc_$TAG.log 2>&1
echo "ncu lc done: $?"
