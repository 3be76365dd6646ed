# Level-2 decode lookup with the 80-register variant (3 CTAs per SM): same-box A/B on cfg4
mkdir -p gpurun_out
for rep in 1 2; do
for v in off on; do
  if [ $v = on ]; then export SQZ_L2_MINB3=1; else unset SQZ_L2_MINB3; fi
  timeout 600 python bench.py --config cfg4 --steps 30 --no-cpu-baseline --no-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v $rep cfg4', d['value'], d['phases_ms']['lookup'], d['phases_ms']['sparse_attention'])"
done
done
unset SQZ_L2_MINB3
SQZ_L2_MINB3=1 timeout 600 python -m pytest tests -m gpu -x -q -k "hier" > gpurun_out/t_l2m3.txt 2>&1; echo tests rc=$?
