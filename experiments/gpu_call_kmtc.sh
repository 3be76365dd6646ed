python -m paper_2411_09688_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_kmeans.py > gpurun_out/test_kmtc.log 2>&1
for m in tensor exact; do
  timeout 900 python bench.py --config cfg4 --no-cpu-baseline --steps 10 --kmeans-mode $m > gpurun_out/bench_cfg4_km_$m.log 2>&1
done
