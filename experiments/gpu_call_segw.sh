# prefill partition setup weight SEG_W sweep on cfg3 (prebuilt .so variants; default 6)
mkdir -p gpurun_out
cp paper_2411_09688_b200/libsqz.so /tmp/libsqz_segw6.so
B="timeout 300 python bench.py --config cfg3 --steps 30 --warmup 5 --no-extra --no-cpu-baseline --no-parity"
for w in 6 2 4 10 14 6; do
  if [ $w = 6 ]; then cp /tmp/libsqz_segw6.so paper_2411_09688_b200/libsqz.so; else cp experiments/libsqz_segw$w.so paper_2411_09688_b200/libsqz.so; fi
  $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('segw $w', d['value'], d['phases_ms']['sparse_attention'])"
done
cp /tmp/libsqz_segw6.so paper_2411_09688_b200/libsqz.so
