# decode L2 prefetch rounds ahead: same-box A/B of prebuilt libraries (pf0 = default)
mkdir -p gpurun_out
cp paper_2411_09688_b200/libsqz.so /tmp/libsqz_pf0.so
B="timeout 300 python bench.py --steps 50 --warmup 5 --no-extra --no-cpu-baseline --no-parity"
for rep in 1 2; do
for v in pf0 pf2 pf4; do
  if [ $v = pf0 ]; then cp /tmp/libsqz_pf0.so paper_2411_09688_b200/libsqz.so; else cp experiments/libsqz_$v.so paper_2411_09688_b200/libsqz.so; fi
  $B > gpurun_out/pf_${v}_$rep.json 2>/dev/null; echo $v rc=$?
done
done
for v in pf0 pf4; do
  if [ $v = pf0 ]; then cp /tmp/libsqz_pf0.so paper_2411_09688_b200/libsqz.so; else cp experiments/libsqz_$v.so paper_2411_09688_b200/libsqz.so; fi
  timeout 600 python bench.py --config cfg5 --steps 20 --warmup 3 --no-extra --no-cpu-baseline --no-parity --kmeans-iters-set 2 > gpurun_out/pf5_${v}.json 2>/dev/null; echo cfg5 $v rc=$?
done
cp /tmp/libsqz_pf0.so paper_2411_09688_b200/libsqz.so
