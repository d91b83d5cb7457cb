#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/profile_level.py --level 2 > gpurun_out/plain_level2.log 2>&1 || exit 1
timeout 600 ncu --cache-control none --clock-control none --set full --import-source on \
  -k regex:csr_tile_kernel --launch-skip 4 --launch-count 1 -o gpurun_out/prof_level2_warm_r02h \
  python tools/profile_level.py --level 2 > gpurun_out/ncu_level2.log 2>&1
timeout 600 ncu --cache-control none --clock-control none --set full --import-source on \
  -k regex:csr_tile_kernel --launch-skip 4 --launch-count 1 -o gpurun_out/prof_level3_warm_r02h \
  python tools/profile_level.py --level 3 > gpurun_out/ncu_level3.log 2>&1
