python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
s=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; e=$(date +%s)
echo "bench wall $((e-s)) s" >> gpurun_out/bench_default.log
