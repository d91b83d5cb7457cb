#!/bin/bash
# Round-end record on one B200: GPU tests, smoke, the default bench line, the
# reference arm, then the ncu launch list and full captures (after the plain
# command exited 0).  Usage: bash profiles/round_end.sh <tag>
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest=$?" >> gpurun_out/rc_$TAG.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke=$?" >> gpurun_out/rc_$TAG.txt
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench=$?" >> gpurun_out/rc_$TAG.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
echo "bench_ref=$?" >> gpurun_out/rc_$TAG.txt
timeout 1800 bash profiles/run_ncu.sh $TAG >> gpurun_out/rc_$TAG.txt 2>&1
echo "ncu=$?" >> gpurun_out/rc_$TAG.txt
