python -m paper_2411_09688_b200.build > /dev/null 2>&1
timeout 900 python -m pytest -q tests/test_gpu_parity.py tests/test_gpu_kmeans.py tests/test_gpu_diag.py -k "empty_selections or T0_zero or tensor_core_assignment_separated or three_level" 2>&1 | tail -25 > gpurun_out/newtests.log
