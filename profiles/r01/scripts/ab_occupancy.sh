#!/bin/bash
# compile-time A/B of SpMV occupancy: CTAs per SM (register cap) x tile size
# (tools/build_variant.py; SMG_LIB selects the build)
mkdir -p gpurun_out
for v in base mb5 mb6 t1024mb6 t1024mb8; do
  if [ $v = base ]; then L=paper_2402_12947_b200/lib/libsimplexmg_b200.so; else L=paper_2402_12947_b200/lib/libsimplexmg_b200_$v.so; fi
  SMG_LIB=$L timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/occ_c2_$v.json 2> gpurun_out/occ_c2_$v.err
  echo "c2 $v rc=$?" >> gpurun_out/rc_occ.txt
  SMG_LIB=$L timeout 900 python bench.py --workload C5 --steps 100 --warmup 5 --no-cpu-baseline --c5-grids 63,126 > gpurun_out/occ_c5_$v.json 2> gpurun_out/occ_c5_$v.err
  echo "c5 $v rc=$?" >> gpurun_out/rc_occ.txt
done
