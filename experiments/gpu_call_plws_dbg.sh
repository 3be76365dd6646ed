python -m paper_2411_09688_b200.build --force > /dev/null 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -k "prefill" 2>&1 | tail -40 > gpurun_out/plws_dbg.log
