# merge kernel for every persistent decode call: full GPU suite, cfg2 A/B, cfg5 check
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_mk.txt 2>&1; echo tests rc=$?
B="timeout 300 python bench.py --steps 50 --warmup 5 --no-extra --no-cpu-baseline --no-parity"
$B > gpurun_out/ab_mk_step.json 2>/dev/null; echo step rc=$?
$B --decode-path calls > gpurun_out/ab_mk_calls.json 2>/dev/null; echo calls rc=$?
SQZ_TICKET_MERGE=1 $B --decode-path calls > gpurun_out/ab_tk_calls.json 2>/dev/null; echo tkcalls rc=$?
timeout 600 python bench.py --config cfg5 --steps 20 --warmup 3 --no-extra --no-cpu-baseline --no-parity > gpurun_out/ab_mk_cfg5.json 2>/dev/null; echo cfg5 rc=$?
SQZ_TICKET_MERGE=1 timeout 600 python bench.py --config cfg5 --steps 20 --warmup 3 --no-extra --no-cpu-baseline --no-parity > gpurun_out/ab_tk_cfg5.json 2>/dev/null; echo cfg5tk rc=$?
