# final validation of the round (after the late merge and lookup changes)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02d_gputest.txt 2>&1; echo tests rc=$?
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02d_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/r02d_bench_default.json 2> gpurun_out/r02d_bench_default.err; echo bench rc=$?
timeout 1500 python bench.py --config cfg5p --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02d_bench_cfg5p.json 2>/dev/null; echo cfg5p rc=$?
