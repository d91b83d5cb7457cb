#!/bin/bash
# C4 level 2 (117,649 rows x 335 nonzeros, streamed, 460 SELL windows): SELL instead of single-chunk tiles, re-measured with the carve-out in place
O=gpurun_out/af
mkdir -p $O
SMG_SELL_MIN_WIN_LONG=400 timeout 1500 python bench.py --workload C4 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_C4_sell400.json 2> $O/bench_C4_sell400.err
echo "C4_sell400=$?" >> $O/rc.txt
SMG_SELL_MIN_WIN_LONG=400 SMG_SELL_LONG_UNROLL=16 timeout 1500 python bench.py --workload C4 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_C4_sell400_u16.json 2> $O/bench_C4_sell400_u16.err
echo "C4_sell400_u16=$?" >> $O/rc.txt
SMG_SELL4=2 timeout 1500 python bench.py --workload C4 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_C4_sell4.json 2> $O/bench_C4_sell4.err
echo "C4_sell4=$?" >> $O/rc.txt
