#!/bin/bash
# Round-2 closing record (session 5: carve-out, staged tile kernel, register-resident sym apply):
# all GPU tests, smoke, bench C1-C5 + reference arm, level costs, ncu launch list / sweeps / corrections (C2), C5 patch kernel
O=gpurun_out/final3
mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu --durations=10 > $O/pytest_gpu.log 2>&1
echo "pytest=$?" > $O/rc.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke=$?" >> $O/rc.txt
timeout 900 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
echo "bench=$?" >> $O/rc.txt
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref_C2.json 2> $O/bench_ref_C2.err
echo "bench_ref=$?" >> $O/rc.txt
for wl in C1 C3 C4; do
  timeout 1500 python bench.py --workload $wl --steps 200 --warmup 10 > $O/bench_$wl.json 2> $O/bench_$wl.err
  echo "bench_$wl=$?" >> $O/rc.txt
done
timeout 900 python bench.py --workload C5 --steps 100 > $O/bench_C5.json 2> $O/bench_C5.err
echo "bench_C5=$?" >> $O/rc.txt
timeout 600 python tools/level_costs.py > $O/level_costs_C2.json 2> $O/level_costs_C2.err
echo "level_costs=$?" >> $O/rc.txt
timeout 600 python tools/c5_patch_sweep.py > $O/c5_sweep.jsonl 2> $O/c5_sweep.err
echo "sweep=$?" >> $O/rc.txt
# ncu (each after its plain command exited 0)
CMD="python tools/profile_driver.py"
if $CMD > $O/plain_C2.log 2>&1; then
  ncu --nvtx --nvtx-include "vcycle/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_r02g.csv $CMD > $O/ncu_launch.log 2>&1
  echo "ncu_launches=$?" >> $O/rc.txt
  ncu --nvtx --nvtx-include "sweeps/" -k regex:"csr_tile_kernel|sell_kernel|csr_stage_kernel" --set full --clock-control none --import-source on -o $O/prof_sweeps_r02g $CMD > $O/ncu_sweeps.log 2>&1
  echo "ncu_sweeps=$?" >> $O/rc.txt
  ncu --nvtx --nvtx-include "lc/" -k regex:patch_kernel --set full --clock-control none --import-source on -o $O/prof_lc_r02g $CMD > $O/ncu_lc.log 2>&1
  echo "ncu_lc=$?" >> $O/rc.txt
fi
CMD="python tools/c5_patch_sweep.py --case C5 --reps 3"
$CMD > $O/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:patch_kernel -s 3 -c 1 -o $O/prof_patchC5_r02g $CMD > $O/ncu_c5.log 2>&1
echo "ncu_c5=$?" >> $O/rc.txt
