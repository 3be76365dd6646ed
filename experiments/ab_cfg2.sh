#!/bin/bash
# same-box A/B of a compile-time variant on cfg2 decode: $1 = extra nvcc flags
for v in "$1" ""; do
  SQZ_NVCC_EXTRA="$v" python -c "import paper_2411_09688_b200.build as b; b.build(force=True)" >/dev/null 2>&1
  for rep in 1 2 3; do
    echo "[$v] cfg2: $(timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*, "unit\|"lookup": [0-9.]*\|"sparse_attention": [0-9.]*' | tr '\n' ' ')"
  done
done
