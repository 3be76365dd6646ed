#!/bin/bash
# ncu launch lists + full-set captures of the dominant kernels (run on the GPU box via gpurun)
set -x
K='regex:k_lookup|k_attend|k_prefill|k_expand|k_fold|k_merge'
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in cfg2 cfg3 cfg4; do
  timeout 600 ncu -k "$K" --metrics $M --clock-control none --csv --log-file gpurun_out/r01_launches_$c.csv \
    python bench.py --config $c --steps 3 --warmup 3 --no-graph --no-cpu-baseline --kmeans-iters 10 > gpurun_out/prof_$c.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend -s 3 -c 1 -o gpurun_out/r01_cfg2_attend \
  python bench.py --config cfg2 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --kmeans-iters 10 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_lookup_decode -s 3 -c 1 -o gpurun_out/r01_cfg2_lookup \
  python bench.py --config cfg2 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --kmeans-iters 10 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_prefill_attend_ws -s 2 -c 1 -o gpurun_out/r01_cfg3_attend \
  python bench.py --config cfg3 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --kmeans-iters 10 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_prefill_lookup_tc -s 3 -c 1 -o gpurun_out/r01_cfg3_lookup \
  python bench.py --config cfg3 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --kmeans-iters 10 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_attend -s 3 -c 1 -o gpurun_out/r01_cfg4_attend \
  python bench.py --config cfg4 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --kmeans-iters 10 > /dev/null 2>&1
ls -la gpurun_out/
