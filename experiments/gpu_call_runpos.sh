python -m paper_2411_09688_b200.build > /dev/null 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -k "decode or prefill" 2>&1 | tail -1 > gpurun_out/runpos.log
for v in "" "--sel-runs"; do
  for r in 1 2; do
    timeout 300 python bench.py --no-prefill --no-extra --no-cpu-baseline --no-parity $v 2>&1 | grep '^{"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 [$v]', d['value'], d['phases_ms']['lookup'], d['phases_ms']['sparse_attention'])" >> gpurun_out/runpos.log
  done
  timeout 300 python bench.py --config cfg3 --no-cpu-baseline --no-parity $v 2>&1 | grep '^{"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 [$v]', d['value'], d['phases_ms']['lookup'], d['phases_ms']['sparse_attention'])" >> gpurun_out/runpos.log
done
