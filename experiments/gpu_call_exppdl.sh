python -m paper_2411_09688_b200.build > /dev/null 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_shard.py -k "prefill or cfg3 or cfg5p or hier or shard" 2>&1 | tail -1 > gpurun_out/exppdl.log
for r in 1 2 3; do
  timeout 300 python bench.py --config cfg3 --no-cpu-baseline --no-parity 2>&1 | grep '^{"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', d['value'], d['phases_ms']['lookup'], d['phases_ms']['sparse_attention'], d['ms_per_step'])" >> gpurun_out/exppdl.log
done
