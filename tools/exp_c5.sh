mkdir -p gpurun_out
run() { echo "== $1" >> gpurun_out/exp_c5b.log; env $2 CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/repro_lc.py $3 >> gpurun_out/exp_c5b.log 2>&1; echo "rc=$?" >> gpurun_out/exp_c5b.log; }
run "300x64 cond6 +512" "COND_DECADES=6" $(python -c "print(','.join(['64']*300+['512']))")
run "300x64 cond6" "COND_DECADES=6" $(python -c "print(','.join(['64']*300))")
run "300x64 cond0 +512" "COND_DECADES=0" $(python -c "print(','.join(['64']*300+['512']))")
run "100x64 cond6 +512" "COND_DECADES=6" $(python -c "print(','.join(['64']*100+['512']))")
run "300x90 cond6" "COND_DECADES=6" $(python -c "print(','.join(['90']*300))")
run "300x64 cond3" "COND_DECADES=3" $(python -c "print(','.join(['64']*300))")
