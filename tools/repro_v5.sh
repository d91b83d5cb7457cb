mkdir -p gpurun_out
for op in spmv residual jacobi chebnext restrict prolong; do
  SMG_SPMV_VARIANT=5 SMG_PDL=0 CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/repro_v5.py $op c1s >> gpurun_out/repro_v5.log 2>&1 || echo "$op FAILED" >> gpurun_out/repro_v5.log
  SMG_SPMV_VARIANT=5 SMG_PDL=0 CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/repro_v5.py $op c2s >> gpurun_out/repro_v5.log 2>&1 || echo "$op c2s FAILED" >> gpurun_out/repro_v5.log
done
SMG_SPMV_VARIANT=5 SMG_PDL=0 timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/repro_v5.py spmv c1s > gpurun_out/memcheck_v5.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/repro_v5.log
