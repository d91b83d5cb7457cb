#!/bin/bash
# (1) per-operator pipelined long-row SELL loop (new default): GPU suite;
# (2) evict-first per-row vectors on streamed SELL sweeps (SMG_EVICT_VEC=1), A/B on C4/C2/C5
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_pipe.log 2>&1
echo "pytest=$?" >> gpurun_out/rc_evictvec.txt
SMG_EVICT_VEC=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_evictvec.log 2>&1
echo "pytest(evictvec)=$?" >> gpurun_out/rc_evictvec.txt
for w in C4 C2 C5; do
  for ev in 0 1; do
    SMG_EVICT_VEC=$ev timeout 900 python bench.py --workload $w --steps 200 --warmup 5 --no-cpu-baseline \
      > gpurun_out/bench_${w}_ev$ev.json 2> gpurun_out/bench_${w}_ev$ev.err
    echo "$w evict_vec=$ev rc=$?" >> gpurun_out/rc_evictvec.txt
  done
done
