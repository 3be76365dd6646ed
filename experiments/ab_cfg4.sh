#!/bin/bash
# same-box A/B of a compile-time variant on cfg4 (and cfg2, cfg5 sanity): $1 = extra nvcc flags of the OLD variant
for v in "" "$1"; do
  SQZ_NVCC_EXTRA="$v" python -c "import paper_2411_09688_b200.build as b; b.build(force=True)" >/dev/null 2>&1
  for c in cfg4 cfg2; do
    for rep in 1 2; do
      echo "[$v] $c: $(timeout 300 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*, "unit\|"lookup": [0-9.]*' | tr '\n' ' ')"
    done
  done
  echo "[$v] cfg5: $(timeout 600 python bench.py --config cfg5 --steps 20 --warmup 5 --no-cpu-baseline --kmeans-iters-set 1 2>&1 | grep -o '"value": [0-9.]*, "unit\|"lookup": [0-9.]*' | tr '\n' ' ')"
done
