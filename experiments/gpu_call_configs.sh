# round 2: the configs the driver does not run (cfg1, cfg4, cfg5, cfg5p) + compute-sanitizer
python -m paper_2411_09688_b200.build > /dev/null 2>&1
timeout 300 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/r02_bench_cfg1.log 2>&1
timeout 600 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/r02_bench_cfg4.log 2>&1
timeout 900 python bench.py --config cfg5 --no-cpu-baseline --kmeans-iters-set 4 --steps 30 > gpurun_out/r02_bench_cfg5.log 2>&1
timeout 1200 python bench.py --config cfg5p --no-cpu-baseline --kmeans-iters-set 4 --steps 10 > gpurun_out/r02_bench_cfg5p.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest -q -x tests/test_gpu_parity.py -m gpu -k "cfg1_fp32 or (prefill and bf16_single) or (prefill and hier_bf16 and not d64)" > gpurun_out/r02_sanitizer_$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/r02_sanitizer_$tool.log
done
