#!/bin/bash
# end-of-round measurements on the GPU box (bench lines + the reference arm + smoke)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final_bench_cfg2.json 2> gpurun_out/final_bench_cfg2.err
timeout 600 python bench.py --config cfg3 > gpurun_out/final_bench_cfg3.json 2> gpurun_out/final_bench_cfg3.err
timeout 600 python bench.py --config cfg4 --steps 50 > gpurun_out/final_bench_cfg4.json 2> gpurun_out/final_bench_cfg4.err
timeout 900 python bench.py --config cfg5 --steps 30 --no-cpu-baseline > gpurun_out/final_bench_cfg5.json 2> gpurun_out/final_bench_cfg5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref_cfg2.json 2> gpurun_out/final_ref_cfg2.err
