#!/bin/bash
# sym path v7 (warp-private rings, no CTA barrier): tests, C5 sweep, ring depth A/B; lean kernels back for small regions: C1/C2/C3 LC check; C4
O=gpurun_out/t
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_patch_sym.py tests/test_gpu_multiregion.py tests/test_gpu_parity.py -q -x -m gpu > $O/pytest_sym.log 2>&1
echo "pytest_sym=$?" > $O/rc.txt
timeout 600 python tools/c5_patch_sweep.py > $O/c5_sweep.jsonl 2> $O/c5_sweep.err
echo "sweep=$?" >> $O/rc.txt
for st in 3 4; do
  SMG_SYM_STAGES=$st timeout 300 python tools/c5_patch_sweep.py --case C5 > $O/c5_stages$st.jsonl 2>&1
  SMG_SYM_STAGES=$st timeout 300 python tools/c5_patch_sweep.py --case "512 x1" >> $O/c5_stages$st.jsonl 2>&1
done
for wl in C2 C1 C3; do
  timeout 900 python bench.py --workload $wl --steps 300 --warmup 10 --no-cpu-baseline > $O/bench_$wl.json 2> $O/bench_$wl.err
  echo "bench_$wl=$?" >> $O/rc.txt
done
timeout 1500 python bench.py --workload C4 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
echo "bench_C4=$?" >> $O/rc.txt
