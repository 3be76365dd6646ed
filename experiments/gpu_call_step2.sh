# decode step: full GPU suite, then A/B of attention occupancy (3 vs 4 CTAs/SM) and a trace
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_step.txt 2>&1; echo tests rc=$?
B="timeout 300 python bench.py --steps 50 --warmup 5 --no-extra --no-cpu-baseline --no-parity"
$B > gpurun_out/ab_m3.json 2>/dev/null; echo m3 rc=$?
SQZ_ATT_MINB=4 $B > gpurun_out/ab_m4.json 2>/dev/null; echo m4 rc=$?
$B > gpurun_out/ab_m3b.json 2>/dev/null; echo m3b rc=$?
SQZ_STEP=1 timeout 300 python experiments/trace_decode.py 0.3 > gpurun_out/trace_step.txt 2>&1; echo trace rc=$?
