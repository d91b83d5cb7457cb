mkdir -p gpurun_out
for t in 8 4 2 16; do
  SMG_TILES_PER_SM=$t timeout 600 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > gpurun_out/bench_t$t.json 2> gpurun_out/bench_t$t.err
done
