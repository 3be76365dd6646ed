# cfg3 prefill attention: one --set full capture with source correlation (run-length selection)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_prefill_attend_ws -s 2 -c 1 -o gpurun_out/r02b_cfg3_attend \
  python bench.py --config cfg3 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-extra --no-parity > /dev/null 2>&1; echo full rc=$?
