#!/bin/bash
# Race / bounds evidence without compute-sanitizer (closed on this pool):
#   1. the SMG_CHECKED build (device-side bounds and protocol assertions,
#      tools/build_variant.py checked -DSMG_CHECKED) over the sanitize driver,
#      in every correction mode, with the follow-mode rings and with the fused
#      (atomic last-CTA) coarse reduction;
#   2. determinism stress on the product build: every V-cycle repeated 50x
#      (graphs and eager), bit-identical or it fails.
mkdir -p gpurun_out
L=paper_2402_12947_b200/lib/libsimplexmg_b200_checked.so
SMG_LIB=$L SMG_LC_FOLLOW=1 timeout 900 python tools/sanitize_driver.py \
  > gpurun_out/checked_follow.log 2>&1; echo "checked_follow=$?" >> gpurun_out/checked_rc.txt
SMG_LIB=$L SMG_COARSE_FUSED=1 timeout 900 python tools/sanitize_driver.py --mode default \
  > gpurun_out/checked_fused.log 2>&1; echo "checked_fused=$?" >> gpurun_out/checked_rc.txt
SMG_LIB=$L SMG_PATCH_STAGES=4 timeout 900 python tools/sanitize_driver.py --mode default \
  > gpurun_out/checked_stages4.log 2>&1; echo "checked_stages4=$?" >> gpurun_out/checked_rc.txt
SMG_LC_FOLLOW=1 timeout 1200 python tools/sanitize_driver.py --stress 50 \
  > gpurun_out/stress_follow.log 2>&1; echo "stress_follow=$?" >> gpurun_out/checked_rc.txt
SMG_COARSE_FUSED=1 timeout 1200 python tools/sanitize_driver.py --stress 50 --mode default \
  > gpurun_out/stress_fused.log 2>&1; echo "stress_fused=$?" >> gpurun_out/checked_rc.txt
