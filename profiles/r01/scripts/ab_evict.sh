mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "properties or c5 or vcycle" > gpurun_out/pytest_prop.log 2>&1; echo prop_rc=$? > gpurun_out/rc_ev.txt
for e in 1 0; do
  SMG_EVICT_FIRST=$e timeout 600 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > gpurun_out/bench_ev$e.json 2> gpurun_out/bench_ev$e.err
done
