mkdir -p gpurun_out
for c in 10 100 300 1000; do
  CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/repro_c5lc.py $c >> gpurun_out/repro_c5lc.log 2>&1 || echo "$c FAILED" >> gpurun_out/repro_c5lc.log
done
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/repro_c5lc.py 1000 400000 >> gpurun_out/repro_c5lc.log 2>&1 || echo "1000 small FAILED" >> gpurun_out/repro_c5lc.log
