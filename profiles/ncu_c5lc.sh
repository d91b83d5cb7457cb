mkdir -p gpurun_out
CMD="python bench.py --workload C5 --c5-grids 63 --steps 20"
$CMD > gpurun_out/plain_c5lc.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:patch_kernel' -s 2 -c 1 -o gpurun_out/prof_c5lc $CMD > gpurun_out/ncu_c5lc.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_c5lc.log
