# decode rows landing in per-warp smem rings by cp.async: parity (decode tests on the variant), same-box A/B
mkdir -p gpurun_out
cp paper_2411_09688_b200/libsqz.so /tmp/libsqz_reg.so
cp experiments/libsqz_smem.so paper_2411_09688_b200/libsqz.so
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "decode" > gpurun_out/t_smem.txt 2>&1; echo tests rc=$?
B="timeout 300 python bench.py --steps 50 --warmup 5 --no-extra --no-cpu-baseline --no-parity"
for rep in 1 2; do
for v in reg smem; do
  if [ $v = reg ]; then cp /tmp/libsqz_reg.so paper_2411_09688_b200/libsqz.so; else cp experiments/libsqz_smem.so paper_2411_09688_b200/libsqz.so; fi
  $B > gpurun_out/sm_${v}_$rep.json 2>/dev/null; echo $v rc=$?
  $B --decode-path calls > gpurun_out/smc_${v}_$rep.json 2>/dev/null
done
done
for v in reg smem; do
  if [ $v = reg ]; then cp /tmp/libsqz_reg.so paper_2411_09688_b200/libsqz.so; else cp experiments/libsqz_smem.so paper_2411_09688_b200/libsqz.so; fi
  timeout 600 python bench.py --config cfg5 --steps 20 --warmup 3 --no-extra --no-cpu-baseline --no-parity --kmeans-iters-set 2 > gpurun_out/sm5_${v}.json 2>/dev/null; echo cfg5 $v rc=$?
done
cp /tmp/libsqz_reg.so paper_2411_09688_b200/libsqz.so
