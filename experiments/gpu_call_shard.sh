python -m paper_2411_09688_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest -q tests/test_gpu_shard.py tests/test_gpu_multi.py -rs > gpurun_out/test_shard.log 2>&1
