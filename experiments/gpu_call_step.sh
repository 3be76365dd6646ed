# decode-step hand-off: parity tests, then same-box A/B of the decode paths on cfg2
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "decode_step" > gpurun_out/t_step.txt 2>&1; echo tests rc=$?
B="timeout 300 python bench.py --steps 50 --warmup 5 --no-extra --no-cpu-baseline --no-parity"
$B --decode-path step > gpurun_out/ab_step.json 2>/dev/null; echo step rc=$?
SQZ_STEP_NO_USER=1 $B --decode-path step > gpurun_out/ab_step_nouser.json 2>/dev/null; echo nouser rc=$?
$B --decode-path calls > gpurun_out/ab_calls.json 2>/dev/null; echo calls rc=$?
SQZ_STEP=1 timeout 300 python experiments/trace_decode.py 0.3 > gpurun_out/trace_step.txt 2>&1; echo trace rc=$?
