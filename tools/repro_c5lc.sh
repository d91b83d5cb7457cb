mkdir -p gpurun_out
SMG_PATCH_SMEM_PAD=40000 CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/repro_c5lc.py 300 >> gpurun_out/repro_c5lc2.log 2>&1 || echo "300 pad FAILED" >> gpurun_out/repro_c5lc2.log
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/repro_lc.py $(python -c "print(','.join(['64']*999+['512']))") >> gpurun_out/repro_c5lc2.log 2>&1 || echo "999x64 FAILED" >> gpurun_out/repro_c5lc2.log
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/repro_lc.py $(python -c "print(','.join(['300']*400))") >> gpurun_out/repro_c5lc2.log 2>&1 || echo "400x300 FAILED" >> gpurun_out/repro_c5lc2.log
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/repro_lc.py $(python -c "print(','.join(['300']*290))") >> gpurun_out/repro_c5lc2.log 2>&1 || echo "290x300 FAILED" >> gpurun_out/repro_c5lc2.log
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/repro_lc.py $(python -c "print(','.join(['300']*300))") >> gpurun_out/repro_c5lc2.log 2>&1 || echo "300x300 FAILED" >> gpurun_out/repro_c5lc2.log
