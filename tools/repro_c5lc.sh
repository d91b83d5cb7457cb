mkdir -p gpurun_out
for c in 296 297; do
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/repro_c5lc.py $c >> gpurun_out/repro_c5lc3.log 2>&1 || echo "$c seeded FAILED" >> gpurun_out/repro_c5lc3.log
done
for spec in "600x300" "200x512" "300x512" "150x512"; do
  cnt=${spec%x*}; sz=${spec#*x}
  CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/repro_lc.py $(python -c "print(','.join(['$sz']*$cnt))") >> gpurun_out/repro_c5lc3.log 2>&1 || echo "$spec FAILED" >> gpurun_out/repro_c5lc3.log
done
