# decode step: key_idx expansion in the lookup vs run-length selection read by the attention
mkdir -p gpurun_out
B="timeout 300 python bench.py --steps 50 --warmup 5 --no-extra --no-cpu-baseline --no-parity"
for rep in 1 2; do
$B > gpurun_out/sr_idx_$rep.json 2>/dev/null; echo idx rc=$?
$B --sel-runs > gpurun_out/sr_runs_$rep.json 2>/dev/null; echo runs rc=$?
done
