# decode step: delay the user chunks behind the lookup's scan requests (A/B of SQZ_UP_DELAY_NS)
mkdir -p gpurun_out
B="timeout 300 python bench.py --steps 50 --warmup 5 --no-extra --no-cpu-baseline --no-parity"
for rep in 1 2; do
for dl in 0 1000 2000 3000; do
  SQZ_UP_DELAY_NS=$dl $B > gpurun_out/dl_${dl}_$rep.json 2>/dev/null; echo $dl rc=$?
done
done
