python -m paper_2411_09688_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest -q tests/test_gpu_kmeans.py tests/test_gpu_parity.py -k "three" > gpurun_out/test_l3.log 2>&1
timeout 1500 python -m pytest -q -x tests -m gpu > gpurun_out/gputest_all.log 2>&1
