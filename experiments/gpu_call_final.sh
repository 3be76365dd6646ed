python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest_final.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_final.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.log 2>&1
