# cfg2 decode lookup: one --set full capture with source correlation; cfg1 tiny-rule check
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_lookup_decode -s 5 -c 1 -o gpurun_out/r02b_cfg2_lookup \
  python bench.py --config cfg2 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-extra --no-parity > /dev/null 2>&1; echo full rc=$?
timeout 300 python bench.py --config cfg1 --steps 50 --no-cpu-baseline --no-parity > gpurun_out/cfg1_tiny.json 2>/dev/null; echo cfg1 rc=$?
