#!/bin/bash
# cfg3 phases, 3 repetitions (same box)
for rep in 1 2 3; do
  echo "cfg3: $(timeout 300 python bench.py --config cfg3 --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*, "unit\|"lookup": [0-9.]*\|"sparse_attention": [0-9.]*' | tr '\n' ' ')"
done
