#!/bin/bash
# same-box A/B of the prefill merge slice size (cfg3 phases)
for m in 16 32 64; do
  SQZ_NVCC_EXTRA="-DSQZ_MERGE_ROWS=$m" python -c "import paper_2411_09688_b200.build as b; b.build(force=True)" >/dev/null 2>&1
  for rep in 1 2; do
    echo "rows $m: $(timeout 300 python bench.py --config cfg3 --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | grep -o '"sparse_attention": [0-9.]*')"
  done
done
