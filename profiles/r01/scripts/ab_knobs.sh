#!/bin/bash
# GPU tests, then A/B of run-time knobs: tile size for small operators
# (SMG_TILES_PER_SM), L2 prefetch distance (SMG_PF_WAVES), and for the C5 patch
# solves the factor L2 prefetch (SMG_PATCH_L2PF) and largest-first order (SMG_PATCH_LPT).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest=$?" >> gpurun_out/rc.txt
run() {  # name workload env...
  local name=$1 w=$2; shift 2
  env "$@" timeout 900 python bench.py --workload $w --steps 500 --warmup 10 --no-cpu-baseline \
    --c5-grids 63 > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err
  echo "$name rc=$?" >> gpurun_out/rc.txt
}
run c2_base C2 X=1
run c2_t8 C2 SMG_TILES_PER_SM=8
run c2_t16 C2 SMG_TILES_PER_SM=16
run c2_pf2 C2 SMG_PF_WAVES=2
run c3_base C3 X=1
run c3_t8 C3 SMG_TILES_PER_SM=8
run c3_t16 C3 SMG_TILES_PER_SM=16
run c5_base C5 X=1
run c5_nol2pf C5 SMG_PATCH_L2PF=0
run c5_nolpt C5 SMG_PATCH_LPT=0
run c5_pf2 C5 SMG_PF_WAVES=2
