#!/bin/bash
# Whole-tile staged kernel (csr_stage_kernel, SMG_TILE_STAGE=1 default): bitwise tests, C2/C3/C1/C4 A/B against the chunked tile kernel
O=gpurun_out/x
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_layouts.py tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_multiregion.py -q -x -m gpu > $O/pytest_stage.log 2>&1
echo "pytest_stage=$?" > $O/rc.txt
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu > $O/pytest_stage_full.log 2>&1
echo "pytest_stage_full=$?" >> $O/rc.txt
for st in 0 1; do
  SMG_TILE_STAGE=$st timeout 900 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > $O/bench_C2_st$st.json 2> $O/bench_C2_st$st.err
  echo "C2_st$st=$?" >> $O/rc.txt
  SMG_TILE_STAGE=$st timeout 900 python bench.py --workload C3 --steps 300 --warmup 10 --no-cpu-baseline > $O/bench_C3_st$st.json 2> $O/bench_C3_st$st.err
  echo "C3_st$st=$?" >> $O/rc.txt
  SMG_TILE_STAGE=$st timeout 900 python bench.py --workload C1 --steps 300 --warmup 10 --no-cpu-baseline > $O/bench_C1_st$st.json 2> $O/bench_C1_st$st.err
  echo "C1_st$st=$?" >> $O/rc.txt
done
SMG_TILE_STAGE=1 timeout 600 python tools/level_costs.py > $O/level_costs_C2_st1.json 2> $O/level_costs_C2.err
echo "level_costs=$?" >> $O/rc.txt
