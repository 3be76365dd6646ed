# merge_row: short chains + ex2.approx vs the previous build: decode tests, A/B cfg1/cfg2/cfg5
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "decode" > gpurun_out/t_mb.txt 2>&1; echo tests rc=$?
cp paper_2411_09688_b200/libsqz.so /tmp/libsqz_new.so
for rep in 1 2; do
for v in new old; do
  cp /tmp/libsqz_$v.so paper_2411_09688_b200/libsqz.so 2>/dev/null || cp experiments/libsqz_old.so paper_2411_09688_b200/libsqz.so
  timeout 300 python bench.py --config cfg1 --steps 50 --no-cpu-baseline --no-parity > gpurun_out/mb1_${v}_$rep.json 2>/dev/null
  timeout 300 python bench.py --steps 50 --no-extra --no-cpu-baseline --no-parity > gpurun_out/mb2_${v}_$rep.json 2>/dev/null
done
done
for v in new old; do
  cp /tmp/libsqz_$v.so paper_2411_09688_b200/libsqz.so 2>/dev/null || cp experiments/libsqz_old.so paper_2411_09688_b200/libsqz.so
  timeout 600 python bench.py --config cfg5 --steps 20 --warmup 3 --no-extra --no-cpu-baseline --no-parity --kmeans-iters-set 2 > gpurun_out/mb5_${v}.json 2>/dev/null
done
cp /tmp/libsqz_new.so paper_2411_09688_b200/libsqz.so
