# A/B: prefill attention segment order (pair-major vs head-major) on cfg3 / cfg5p
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for v in 1 0; do
  SQZ_NVCC_EXTRA="-DSQZ_PF_PAIR_MAJOR=$v" python -m paper_2411_09688_b200.build --force > /dev/null 2>&1
  echo "== pair_major=$v" >> gpurun_out/ab_pm.log
  timeout 600 python -m pytest -q -x tests/test_gpu_parity.py -k prefill 2>&1 | tail -1 >> gpurun_out/ab_pm.log
  for r in 1 2; do
    timeout 600 python bench.py --config cfg3 --no-cpu-baseline --no-parity 2>&1 | grep '^{"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', d['value'], d['phases_ms']['lookup'], d['phases_ms']['sparse_attention'], d['roofline']['frac'])" >> gpurun_out/ab_pm.log
  done
  timeout 1200 python bench.py --config cfg5p --no-cpu-baseline --no-parity --steps 5 --kmeans-iters-set 3 2>&1 | grep '^{"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5p', d['value'], d['phases_ms']['lookup'], d['phases_ms']['sparse_attention'], d['roofline']['frac'])" >> gpurun_out/ab_pm.log
  timeout 600 ncu -k regex:k_prefill_attend_ws --metrics $M --clock-control none --csv --log-file gpurun_out/ab_pm_$v.csv python bench.py --config cfg3 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-parity > /dev/null 2>&1
done
