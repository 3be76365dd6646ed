python -m paper_2411_09688_b200.build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest -q -x tests/test_gpu_diag.py > gpurun_out/test_diag.log 2>&1
timeout 300 python bench.py --no-prefill --no-cpu-baseline --steps 20 > gpurun_out/bench_diag_cfg2.log 2>&1
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --steps 20 > gpurun_out/bench_diag_cfg4.log 2>&1
