# late round-2 validation: full GPU suite, smoke, default bench line, cfg1/cfg5 lines, reference arm
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02b_gputest.txt 2>&1; echo tests rc=$?
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02b_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/r02b_bench_default2.json 2> gpurun_out/r02b_bench_default2.err; echo bench rc=$?
timeout 600 python bench.py --config cfg1 --steps 50 > gpurun_out/r02b_bench_cfg1.json 2> /dev/null; echo cfg1 rc=$?
timeout 900 python bench.py --config cfg5 --steps 30 --no-cpu-baseline > gpurun_out/r02b_bench_cfg5.json 2> /dev/null; echo cfg5 rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02b_reference_cfg2.json 2> gpurun_out/r02b_reference_cfg2.err; echo ref rc=$?
