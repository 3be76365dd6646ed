timeout 300 python experiments/trace_pl.py > gpurun_out/trace_pl.log 2>&1
