mkdir -p gpurun_out
SMG_ASYNC_TILES=1 timeout 900 python -m pytest tests -x -q -m gpu -k "sparse or sweep or vcycle" > gpurun_out/pytest_async.log 2>&1; echo async_rc=$? > gpurun_out/rc_async.txt
for a in 1 0; do
  SMG_ASYNC_TILES=$a timeout 600 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > gpurun_out/bench_async$a.json 2> gpurun_out/bench_async$a.err
done
SMG_ASYNC_TILES=1 timeout 900 python bench.py --workload C5 --c5-grids 63 > gpurun_out/bench_c5_async.json 2> gpurun_out/bench_c5_async.err
