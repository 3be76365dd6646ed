#!/bin/bash
K='regex:k_lookup|k_attend|k_prefill|k_expand|k_fold|k_merge'
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in cfg2 cfg4; do
  timeout 600 ncu -k "$K" --metrics $M --clock-control none --csv --log-file gpurun_out/r01_launches_$c.csv \
    python bench.py --config $c --steps 3 --warmup 3 --no-graph --no-cpu-baseline --kmeans-iters 10 > gpurun_out/prof_$c.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend -s 3 -c 1 -o gpurun_out/r01_cfg2_attend \
  python bench.py --config cfg2 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --kmeans-iters 10 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_lookup_decode -s 3 -c 1 -o gpurun_out/r01_cfg2_lookup \
  python bench.py --config cfg2 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --kmeans-iters 10 > /dev/null 2>&1
