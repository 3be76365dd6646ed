#!/bin/bash
# same-box A/B over compile-time flag sets: ab_flags.sh "<flags A>" "<flags B>" ... (CONFIGS env)
for v in "$@"; do
  SQZ_NVCC_EXTRA="$v" python -c "import paper_2411_09688_b200.build as b; b.build(force=True)" >/dev/null 2>&1
  for c in $CONFIGS; do
    for rep in 1 2; do
      echo "[$v] $c: $(timeout 300 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*, "unit\|"lookup": [0-9.]*\|"sparse_attention": [0-9.]*' | tr '\n' ' ')"
    done
  done
done
