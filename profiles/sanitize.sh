#!/bin/bash
# compute-sanitizer over tools/sanitize_driver.py (one B200; run under gpurun).
#   bash profiles/sanitize.sh <tag>
# Logs: gpurun_out/sanitize_<tool>[_<variant>]_<tag>.log (copied to profiles/<round>/)
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
CS="compute-sanitizer --print-limit 50 --error-exitcode 9"
run() {  # tool, variant, env...
  local tool=$1 var=$2; shift 2
  env "$@" timeout 900 $CS --tool $tool python tools/sanitize_driver.py \
      > $OUT/sanitize_${tool}${var}_$TAG.log 2>&1
  echo "$tool$var rc=$?" >> $OUT/sanitize_rc_$TAG.txt
}
run memcheck "" SMG_LC_FOLLOW=1
run racecheck "" SMG_LC_FOLLOW=1
run synccheck "" SMG_LC_FOLLOW=1
run initcheck "" SMG_LC_FOLLOW=1
# the fused coarse solve (atomic last-CTA reduction, dense_kernels.cu)
run racecheck _coarse_fused SMG_COARSE_FUSED=1
run memcheck _coarse_fused SMG_COARSE_FUSED=1
