#!/bin/bash
# C4 level 2 on the staged kernel (streamed, 9,216-product tiles): bitwise full-size tests, bench A/B
O=gpurun_out/ah
mkdir -p $O
timeout 1500 python bench.py --workload C4 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_C4_stream_stage.json 2> $O/bench_C4_stream_stage.err
echo "C4_stream_stage=$?" >> $O/rc.txt
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu -k C4 > $O/pytest_full_C4.log 2>&1
echo "pytest_full_C4=$?" >> $O/rc.txt
SMG_STAGE_STREAM_MIN_ROW=0 timeout 1500 python bench.py --workload C4 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_C4_base.json 2> $O/bench_C4_base.err
echo "C4_base=$?" >> $O/rc.txt
