# A/B: prefill K/V tiles with TMA boxes for consecutive 8-row groups vs all cp.async
for v in 1 0; do
  SQZ_NVCC_EXTRA="-DSQZ_PF_TMA_GROUPS=$v" python -m paper_2411_09688_b200.build --force > /dev/null 2>&1
  echo "== tma_groups=$v" >> gpurun_out/ab_pftma.log
  timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_shard.py -k "prefill or cfg3 or cfg5p" 2>&1 | tail -1 >> gpurun_out/ab_pftma.log
  for r in 1 2; do
    timeout 300 python bench.py --config cfg3 --no-cpu-baseline --no-parity 2>&1 | grep '^{"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', d['value'], d['phases_ms']['lookup'], d['phases_ms']['sparse_attention'], d['roofline']['frac'])" >> gpurun_out/ab_pftma.log
  done
  timeout 1200 python bench.py --config cfg5p --no-cpu-baseline --no-parity --steps 5 --kmeans-iters-set 3 2>&1 | grep '^{"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5p', d['value'], d['phases_ms']['lookup'], d['phases_ms']['sparse_attention'], d['roofline']['frac'])" >> gpurun_out/ab_pftma.log
done
