python -m paper_2411_09688_b200.build > /dev/null 2>&1
timeout 600 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "decode" 2>&1 | tail -1 >> gpurun_out/ab_minb.log
for r in 1 2; do
  timeout 300 python bench.py --no-prefill --no-extra --no-cpu-baseline --no-parity 2>&1 | grep '^{"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', d['value'], d['phases_ms']['sparse_attention'], d['roofline']['frac'])" >> gpurun_out/ab_minb.log
done
timeout 900 python bench.py --config cfg5 --no-cpu-baseline --steps 30 > gpurun_out/r02_bench_cfg5.log 2>&1
grep '^{"metric"' gpurun_out/r02_bench_cfg5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5', d['value'], d['phases_ms']['sparse_attention'], d['roofline']['frac'], d['parity']['ok'])" >> gpurun_out/ab_minb.log
timeout 900 python bench.py --config cfg5h3 --no-cpu-baseline --steps 30 > gpurun_out/r02_bench_cfg5h3.log 2>&1
grep '^{"metric"' gpurun_out/r02_bench_cfg5h3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5h3', d['value'], d['phases_ms']['sparse_attention'], d['roofline']['frac'], d['parity']['ok'])" >> gpurun_out/ab_minb.log
