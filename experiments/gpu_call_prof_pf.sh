python -m paper_2411_09688_b200.build > gpurun_out/build.log 2>&1
K='regex:k_prefill|k_lookup|k_attend|k_expand|k_merge|k_fold|k_union'
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active
timeout 1200 ncu -k "$K" --metrics $M --clock-control none --csv --log-file gpurun_out/r02_launches_cfg5p.csv python bench.py --config cfg5p --steps 1 --warmup 3 --no-graph --no-cpu-baseline --no-parity --kmeans-iters-set 3 > gpurun_out/prof_cfg5p.log 2>&1
timeout 900 ncu -k "$K" --metrics $M --clock-control none --csv --log-file gpurun_out/r02_launches_cfg3.csv python bench.py --config cfg3 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-parity > gpurun_out/prof_cfg3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_prefill_attend_ws -s 3 -c 1 -o gpurun_out/r02_cfg3_attend python bench.py --config cfg3 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-parity > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_prefill_lookup_tc -s 3 -c 1 -o gpurun_out/r02_cfg3_lookup python bench.py --config cfg3 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-parity > /dev/null 2>&1
