# fused decode step: device timeline per user-chunk mode, then the bench (both paths)
for um in 3 2 1 0; do
  echo "== SQZ_STEP_UMODE=$um" >> gpurun_out/trace_step.log
  SQZ_STEP_UMODE=$um timeout 300 python experiments/trace_step.py 2>&1 | grep -v "^ptxas\|^nvcc" >> gpurun_out/trace_step.log
done
python -m paper_2411_09688_b200.build --force > /dev/null 2>&1
for um in 3 2 0; do
  SQZ_STEP_UMODE=$um timeout 300 python bench.py --no-prefill --no-cpu-baseline --no-parity > gpurun_out/bench_step_u$um.log 2>&1
done
timeout 300 python bench.py --no-prefill --no-cpu-baseline --no-parity --decode-path calls > gpurun_out/bench_calls.log 2>&1
