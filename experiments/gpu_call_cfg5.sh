python -m paper_2411_09688_b200.build > gpurun_out/build.log 2>&1
timeout 1200 python bench.py --config cfg5h3 --no-cpu-baseline --steps 30 > gpurun_out/r02_bench_cfg5h3.log 2>&1
timeout 1200 python bench.py --config cfg5 --no-cpu-baseline --steps 30 > gpurun_out/r02_bench_cfg5.log 2>&1
timeout 1500 python bench.py --config cfg5p --no-cpu-baseline --steps 10 > gpurun_out/r02_bench_cfg5p.log 2>&1
