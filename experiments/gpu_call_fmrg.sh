# flag-based row merge (k_merge_rows without griddepcontrol.wait): decode tests, same-box A/B, trace
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "decode or fullsize" > gpurun_out/t_fmrg.txt 2>&1; echo tests rc=$?
cp paper_2411_09688_b200/libsqz.so /tmp/libsqz_new.so
B="timeout 300 python bench.py --steps 50 --warmup 5 --no-extra --no-cpu-baseline --no-parity"
for rep in 1 2; do
for v in new old; do
  cp /tmp/libsqz_$v.so paper_2411_09688_b200/libsqz.so 2>/dev/null || cp experiments/libsqz_old.so paper_2411_09688_b200/libsqz.so
  $B > gpurun_out/fm_${v}_$rep.json 2>/dev/null; echo $v rc=$?
  $B --decode-path calls > gpurun_out/fmc_${v}_$rep.json 2>/dev/null
done
done
cp /tmp/libsqz_new.so paper_2411_09688_b200/libsqz.so
SQZ_STEP=1 timeout 300 python experiments/trace_decode.py 0.3 > gpurun_out/trace_step.txt 2>&1; echo trace rc=$?
