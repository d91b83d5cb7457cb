#!/bin/bash
# round-2 record: GPU tests (all), smoke, default bench, reference arm, other workloads,
# and per-workload ncu captures of the dominant kernel (after plain runs exit 0)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/pytest_gpu_r02.log 2>&1
echo "pytest=$?" >> gpurun_out/rc_final.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02.log 2>&1
echo "smoke=$?" >> gpurun_out/rc_final.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_C2_r02.json 2> gpurun_out/bench_C2_r02.err
echo "bench=$?" >> gpurun_out/rc_final.txt
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_C2_r02.json 2> gpurun_out/bench_ref_C2_r02.err
echo "bench_ref=$?" >> gpurun_out/rc_final.txt
for wl in C1 C3 C4; do
  timeout 1200 python bench.py --workload $wl --steps 200 --warmup 10 > gpurun_out/bench_${wl}_r02.json 2> gpurun_out/bench_${wl}_r02.err
  echo "bench_$wl=$?" >> gpurun_out/rc_final.txt
done
timeout 900 python bench.py --workload C5 --steps 100 > gpurun_out/bench_C5_r02.json 2> gpurun_out/bench_C5_r02.err
echo "bench_C5=$?" >> gpurun_out/rc_final.txt
for wl in C1 C3 C4; do
  if timeout 900 python tools/profile_driver.py --workload $wl > gpurun_out/plain_$wl.log 2>&1; then
    timeout 1200 ncu --nvtx --nvtx-include "sweeps/" -k regex:"csr_tile_kernel|sell_kernel" --launch-count 1 \
      --set full --clock-control none -o gpurun_out/prof_sweep0_${wl}_r02 \
      python tools/profile_driver.py --workload $wl > gpurun_out/ncu_sweep0_$wl.log 2>&1
    echo "ncu_$wl=$?" >> gpurun_out/rc_final.txt
  fi
done
