python -m paper_2411_09688_b200.build > /dev/null 2>&1
for v in "" "--sel-runs"; do
  for r in 1 2; do
    timeout 300 python bench.py --config cfg3 --no-cpu-baseline --no-parity $v 2>&1 | grep '^{"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 [$v]', d['value'], d['phases_ms']['lookup'], d['phases_ms']['sparse_attention'], d['roofline']['frac'])" >> gpurun_out/ab_selruns.log
  done
  timeout 1200 python bench.py --config cfg5p --no-cpu-baseline --no-parity --steps 5 --kmeans-iters-set 3 $v 2>&1 | grep '^{"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5p [$v]', d['value'], d['phases_ms']['lookup'], d['phases_ms']['sparse_attention'])" >> gpurun_out/ab_selruns.log
  timeout 300 python bench.py --no-prefill --no-extra --no-cpu-baseline --no-parity $v 2>&1 | grep '^{"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 [$v]', d['value'], d['phases_ms']['lookup'], d['phases_ms']['sparse_attention'])" >> gpurun_out/ab_selruns.log
done
