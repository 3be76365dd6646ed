# cfg3 prefill lookup: one --set full capture with source correlation
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_prefill_lookup_tc -s 3 -c 1 -o gpurun_out/r02b_cfg3_lookup \
  python bench.py --config cfg3 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-extra --no-parity > /dev/null 2>&1; echo full rc=$?
