mkdir -p gpurun_out
for sz in "512" "100,512" "64,512" "200,512" "300,512" "512,512,512" "450,512" "480,512" "500,512" "33,512" "65,512" "97,512" "129,512" "511,512" "257,512" "400,401,402,403,512"; do
  CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/repro_lc.py $sz >> gpurun_out/repro_lc.log 2>&1 || echo "$sz FAILED" >> gpurun_out/repro_lc.log
done
python - >> gpurun_out/repro_lc.log 2>&1 <<'PY'
import numpy as np
rng = np.random.default_rng(2402)
s = rng.integers(64, 513, size=60)
print(",".join(map(str, s)))
PY
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/repro_lc.py $(tail -1 gpurun_out/repro_lc.log) >> gpurun_out/repro_lc.log 2>&1 || echo "seeded60 FAILED" >> gpurun_out/repro_lc.log
