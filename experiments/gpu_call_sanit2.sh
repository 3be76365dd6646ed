# compute-sanitizer on the late round-2 decode paths: the decode step (user chunks before the
# wait, ticket word / merge kernel), the st.async lookup exchange, k_merge_rows
mkdir -p gpurun_out
K='decode_step and (step_bf16_d128_nu37 or step_bf16_sparse_nu5 or step_fp32_d64_nu1 or step_bf16_h32 or user_chunks)'
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest -q -x tests/test_gpu_parity.py -m gpu -k "$K" > gpurun_out/r02b_sanitizer_$tool.log 2>&1
  echo "$tool exit=$?"
done
