# decode lookup reductions with ex2.approx: lookup/decode tests, same-box A/B cfg2 (step) and cfg1
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "decode or lookup or fullsize or shard" > gpurun_out/t_lkf.txt 2>&1; echo tests rc=$?
cp paper_2411_09688_b200/libsqz.so /tmp/libsqz_new.so
for rep in 1 2 3; do
for v in new old; do
  cp /tmp/libsqz_$v.so paper_2411_09688_b200/libsqz.so 2>/dev/null || cp experiments/libsqz_old.so paper_2411_09688_b200/libsqz.so
  timeout 300 python bench.py --steps 50 --no-extra --no-cpu-baseline --no-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v $rep cfg2', d['value'], d['phases_ms']['lookup'])"
done
done
cp /tmp/libsqz_new.so paper_2411_09688_b200/libsqz.so
