# N-rank bench code path on one GPU (gloo, all ranks on device 0): heads (cfg2, cfg4)
python -m paper_2411_09688_b200.build > /dev/null 2>&1
SQZ_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/dryrun_n2.log 2>&1
echo "exit=$?" >> gpurun_out/dryrun_n2.log
