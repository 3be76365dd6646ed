TRACE_FULL=40:48 timeout 300 python experiments/trace_prefill.py > gpurun_out/trace_prefill.log 2>&1
python -m paper_2411_09688_b200.build --force > /dev/null 2>&1
