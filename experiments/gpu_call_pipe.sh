# same-box A/B of decode attention variants (prebuilt .so files): default (KR=16),
# KR=8, KR=8 + software pipelining (two rounds in flight per warp)
mkdir -p gpurun_out
cp paper_2411_09688_b200/libsqz.so /tmp/libsqz_default.so
B="timeout 300 python bench.py --steps 50 --warmup 5 --no-extra --no-cpu-baseline --no-parity"
for rep in 1 2; do
for v in default kr8 pipe; do
  if [ $v = default ]; then cp /tmp/libsqz_default.so paper_2411_09688_b200/libsqz.so; else cp experiments/libsqz_$v.so paper_2411_09688_b200/libsqz.so; fi
  $B > gpurun_out/ab_${v}_$rep.json 2>/dev/null; echo $v rc=$?
done
done
cp /tmp/libsqz_default.so paper_2411_09688_b200/libsqz.so
