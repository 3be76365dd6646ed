#!/bin/bash
# A/B of the fraction of exp2 pairs computed by the FMA-pipe polynomial in the
# warp-specialised prefill attention (SQZ_PF_EMU_MASK), cfg3 phases.
for m in "$@"; do
  SQZ_NVCC_EXTRA="-DSQZ_PF_EMU_MASK=$m" python -c "import paper_2411_09688_b200.build as b; b.build(force=True)" >/dev/null 2>&1
  echo "mask $m: $(timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | grep -o '"sparse_attention": [0-9.]*')"
done
