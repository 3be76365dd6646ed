# decode partition setup allowance SEG_KW sweep on the cfg2 step (prebuilt .so variants; default 128)
mkdir -p gpurun_out
cp paper_2411_09688_b200/libsqz.so /tmp/libsqz_kw128.so
B="timeout 300 python bench.py --steps 50 --warmup 5 --no-extra --no-cpu-baseline --no-parity"
for w in 128 0 64 192 256 128; do
  if [ $w = 128 ]; then cp /tmp/libsqz_kw128.so paper_2411_09688_b200/libsqz.so; else cp experiments/libsqz_kw$w.so paper_2411_09688_b200/libsqz.so; fi
  $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('kw $w', d['value'])"
done
cp /tmp/libsqz_kw128.so paper_2411_09688_b200/libsqz.so
