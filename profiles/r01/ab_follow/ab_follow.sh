#!/bin/bash
# Follow-mode corrections (SMG_LC_FOLLOW=0 disables them): their parity tests
# first, then the whole GPU suite, then an A/B on C1/C3/C2/C4.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "follow" > gpurun_out/pytest_follow.log 2>&1
echo "pytest_follow=$?" >> gpurun_out/rc_follow.txt
[ "$1" = "quick" ] || timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_follow.log 2>&1
echo "pytest=$?" >> gpurun_out/rc_follow.txt
for w in C3 C1 C2 C4; do
  for f in 1 0; do
    SMG_LC_FOLLOW=$f timeout 900 python bench.py --workload $w --steps 500 --warmup 10 --no-cpu-baseline \
      > gpurun_out/bench_${w}_follow$f.json 2> gpurun_out/bench_${w}_follow$f.err
    echo "$w follow=$f rc=$?" >> gpurun_out/rc_follow.txt
  done
done
