# round-2 (late) decode step: default bench line, cfg2 launch list, k_attend full capture
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02b_bench_default.json 2> gpurun_out/r02b_bench_default.err; echo bench rc=$?
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu -k 'regex:k_lookup|k_attend|k_merge' --metrics $M --clock-control none --csv \
  --log-file gpurun_out/r02b_launches_cfg2.csv \
  python bench.py --config cfg2 --steps 3 --warmup 3 --no-graph --no-cpu-baseline --no-extra --no-parity > gpurun_out/prof_cfg2.log 2>&1; echo launches rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend -s 3 -c 1 -o gpurun_out/r02b_cfg2_attend \
  python bench.py --config cfg2 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-extra --no-parity > /dev/null 2>&1; echo full rc=$?
