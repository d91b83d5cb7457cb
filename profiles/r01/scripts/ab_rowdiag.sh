#!/bin/bash
# int32 tile-relative row offsets + diagonal taken from the row (no 1/a_ii
# vector stream): GPU parity, then C2/C3/C5 bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest=$?" >> gpurun_out/rc_rd.txt
timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/rd_c2.json 2> gpurun_out/rd_c2.err
echo "c2 rc=$?" >> gpurun_out/rc_rd.txt
timeout 600 python bench.py --workload C3 --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/rd_c3.json 2> gpurun_out/rd_c3.err
echo "c3 rc=$?" >> gpurun_out/rc_rd.txt
timeout 900 python bench.py --workload C5 --steps 100 --warmup 5 --no-cpu-baseline --c5-grids 63,126 > gpurun_out/rd_c5.json 2> gpurun_out/rd_c5.err
echo "c5 rc=$?" >> gpurun_out/rc_rd.txt
