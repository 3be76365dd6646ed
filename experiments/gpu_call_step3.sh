# decode step: merge kernel vs in-kernel ticket merge (same box), tests, trace
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "decode" > gpurun_out/t_step.txt 2>&1; echo tests rc=$?
B="timeout 300 python bench.py --steps 50 --warmup 5 --no-extra --no-cpu-baseline --no-parity"
$B > gpurun_out/ab_mk.json 2>/dev/null; echo mk rc=$?
SQZ_STEP_TICKET_MERGE=1 $B > gpurun_out/ab_tk.json 2>/dev/null; echo tk rc=$?
$B > gpurun_out/ab_mk2.json 2>/dev/null; echo mk2 rc=$?
SQZ_STEP=1 timeout 300 python experiments/trace_decode.py 0.3 > gpurun_out/trace_step.txt 2>&1; echo trace rc=$?
