# batch-shared decode: CUDA-core register streaming (LDG) vs the mma.sync ring kernel
for v in "" "-DSQZ_SHL_MINB8=3" "-DSQZ_SHD_LDG=0"; do
  SQZ_NVCC_EXTRA="$v" python -m paper_2411_09688_b200.build --force > /dev/null 2>&1 || echo "build failed $v"
  echo "== variant [$v]" >> gpurun_out/ab_shared.log
  timeout 300 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "shared or decode or cfg4" 2>&1 | tail -1 >> gpurun_out/ab_shared.log
  for r in 1 2; do
  timeout 600 python bench.py --config cfg4 --no-cpu-baseline --steps 30 --no-parity 2>&1 | grep '^{"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['phases_ms']['sparse_attention'], d['roofline']['frac'])" >> gpurun_out/ab_shared.log
  done
done
