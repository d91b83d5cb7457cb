#!/bin/bash
# re-entry sanity: GPU tests, smoke, default bench after the container was re-created
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu_r02l.log 2>&1
echo "pytest=$?" > gpurun_out/rc_l.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02l.log 2>&1
echo "smoke=$?" >> gpurun_out/rc_l.txt
timeout 900 python bench.py > gpurun_out/bench_C2_r02l.json 2> gpurun_out/bench_C2_r02l.err
echo "bench=$?" >> gpurun_out/rc_l.txt
