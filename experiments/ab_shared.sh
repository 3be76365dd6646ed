# same-box A/B of the batch-shared decode kernel's ring / warp knobs on cfg4
for v in "" "-DSQZ_SHD_NW=3 -DSQZ_SHD_NST=4" "-DSQZ_SHD_NW=6 -DSQZ_SHD_NST=2" "-DSQZ_SHD_NW=5 -DSQZ_SHD_NST=2"; do
  SQZ_NVCC_EXTRA="$v" python -m paper_2411_09688_b200.build --force > /dev/null 2>&1 || echo "build failed $v"
  echo "== variant [$v]" >> gpurun_out/ab_shared.log
  timeout 300 python -m pytest -q -x tests/test_gpu_parity.py -k "shared" 2>&1 | tail -1 >> gpurun_out/ab_shared.log
  for r in 1 2; do
  timeout 600 python bench.py --config cfg4 --no-cpu-baseline --steps 30 --no-parity 2>&1 | grep '^{"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['phases_ms']['sparse_attention'], d['roofline']['frac'])" >> gpurun_out/ab_shared.log
  done
done
