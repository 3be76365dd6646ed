# decode tail pool: tests, then same-box A/B pool vs no pool (cfg2 step, cfg2 calls, cfg4), trace
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "decode or fullsize or shard" > gpurun_out/t_pool.txt 2>&1; echo tests rc=$?
B="timeout 300 python bench.py --steps 50 --warmup 5 --no-extra --no-cpu-baseline --no-parity"
for rep in 1 2; do
$B > gpurun_out/pool_on_$rep.json 2>/dev/null; echo on rc=$?
SQZ_NO_POOL=1 $B > gpurun_out/pool_off_$rep.json 2>/dev/null; echo off rc=$?
done
$B --decode-path calls > gpurun_out/pool_on_calls.json 2>/dev/null
SQZ_NO_POOL=1 $B --decode-path calls > gpurun_out/pool_off_calls.json 2>/dev/null
SQZ_STEP=1 timeout 300 python experiments/trace_decode.py 0.3 > gpurun_out/trace_step.txt 2>&1; echo trace rc=$?
