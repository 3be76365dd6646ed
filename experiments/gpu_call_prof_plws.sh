python -m paper_2411_09688_b200.build --force > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_prefill_lookup_ws -s 3 -c 1 -o gpurun_out/r02_cfg3_lookup_ws python bench.py --config cfg3 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-parity > /dev/null 2>&1
