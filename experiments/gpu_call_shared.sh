python -m paper_2411_09688_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -k "shared or decode" > gpurun_out/test_shared.log 2>&1
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --steps 30 > gpurun_out/bench_cfg4_shared.log 2>&1
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --steps 30 --attn-per-row > gpurun_out/bench_cfg4_perrow.log 2>&1
