python -m paper_2411_09688_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "prefill or hier" > gpurun_out/test_gather.log 2>&1
timeout 1500 python bench.py --config cfg5p --no-cpu-baseline --steps 10 > gpurun_out/r02_bench_cfg5p.log 2>&1
