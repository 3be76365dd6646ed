python -m paper_2411_09688_b200.build --force > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_attend_shared_ldg -s 2 -c 1 -o gpurun_out/r02_cfg4_ldg python bench.py --config cfg4 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-parity --kmeans-iters 10 > /dev/null 2>&1
