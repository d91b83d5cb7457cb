#!/bin/bash
# Final binary of the round: all GPU tests, smoke, default bench + reference arm
O=gpurun_out/final4
mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1
echo "pytest=$?" > $O/rc.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke=$?" >> $O/rc.txt
timeout 900 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
echo "bench=$?" >> $O/rc.txt
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref_C2.json 2> $O/bench_ref_C2.err
echo "bench_ref=$?" >> $O/rc.txt
timeout 1500 python bench.py --workload C4 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
echo "bench_C4=$?" >> $O/rc.txt
