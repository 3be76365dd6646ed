python -m paper_2411_09688_b200.build > /dev/null 2>&1
for f in write write+read; do
  for r in 1 2; do
    timeout 300 python bench.py --no-prefill --no-extra --no-cpu-baseline --no-parity --flush $f 2>&1 | grep '^{"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 [$f]', d['value'], d['phases_ms']['lookup'], d['phases_ms']['sparse_attention'], d['e2e']['value'])" >> gpurun_out/ab_flush.log
  done
  timeout 300 python bench.py --config cfg3 --no-cpu-baseline --no-parity --flush $f 2>&1 | grep '^{"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 [$f]', d['value'], d['phases_ms']['lookup'], d['phases_ms']['sparse_attention'])" >> gpurun_out/ab_flush.log
done
python experiments/event_floor.py >> gpurun_out/ab_flush.log 2>&1
