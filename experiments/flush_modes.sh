set -x
for f in write write+read; do
 for c in cfg2 cfg4; do
  python bench.py --config $c --steps 20 --warmup 5 --flush $f --no-cpu-baseline > gpurun_out/r02_fl_${c}_${f/+/_}.json 2>gpurun_out/r02_fl_${c}_${f/+/_}.err
 done
 python bench.py --config cfg3 --steps 20 --warmup 5 --flush $f --no-cpu-baseline > gpurun_out/r02_fl_cfg3_${f/+/_}.json 2>&1
done
