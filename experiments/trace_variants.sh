#!/bin/bash
for v in "-DSQZ_TRACE" "-DSQZ_TRACE -DSQZ_NO_PDL" "-DSQZ_TRACE -DSQZ_CARVEOUT_MAX"; do
  echo "=== $v"
  SQZ_NVCC_EXTRA="$v" python paper_2411_09688_b200/build.py --force > /dev/null 2>&1 || echo build failed
  python experiments/trace_decode.py 0.3 | grep -E "event|lookup end|attn entry|attn prologue|attn end"
done
