mkdir -p gpurun_out
SQZ_STEP=1 timeout 300 python experiments/trace_decode.py 0.3 > gpurun_out/trace_step.txt 2>&1; echo trace rc=$?
