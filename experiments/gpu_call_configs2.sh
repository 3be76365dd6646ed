# late round-2 bench lines of the configs the driver does not run
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg3 --steps 50 > gpurun_out/r02b_bench_cfg3.json 2>/dev/null; echo cfg3 rc=$?
timeout 900 python bench.py --config cfg4 --steps 50 > gpurun_out/r02b_bench_cfg4.json 2>/dev/null; echo cfg4 rc=$?
timeout 1200 python bench.py --config cfg5h3 --steps 30 --no-cpu-baseline > gpurun_out/r02b_bench_cfg5h3.json 2>/dev/null; echo cfg5h3 rc=$?
timeout 1500 python bench.py --config cfg5p --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_bench_cfg5p.json 2>/dev/null; echo cfg5p rc=$?
