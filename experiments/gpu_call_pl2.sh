# prefill lookup: per-half column partials (no pass-2 barrier) -- tests, same-box A/B on cfg3 and cfg5p
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "prefill or lookup or fullsize" > gpurun_out/t_pl.txt 2>&1; echo tests rc=$?
cp paper_2411_09688_b200/libsqz.so /tmp/libsqz_new.so
B="timeout 300 python bench.py --config cfg3 --steps 30 --warmup 5 --no-extra --no-cpu-baseline --no-parity"
for rep in 1 2; do
for v in new old; do
  cp /tmp/libsqz_$v.so paper_2411_09688_b200/libsqz.so 2>/dev/null || cp experiments/libsqz_old.so paper_2411_09688_b200/libsqz.so
  $B > gpurun_out/pl2_${v}_$rep.json 2>/dev/null; echo $v rc=$?
done
done
cp /tmp/libsqz_new.so paper_2411_09688_b200/libsqz.so
