#!/bin/bash
# same-box A/B of the working-tree libsqz.so against experiments/libsqz_old.so
cp paper_2411_09688_b200/libsqz.so /tmp/libsqz_new.so
for v in new old; do
  cp /tmp/libsqz_$v.so paper_2411_09688_b200/libsqz.so 2>/dev/null || cp experiments/libsqz_old.so paper_2411_09688_b200/libsqz.so
  touch paper_2411_09688_b200/libsqz.so
  for c in $CONFIGS; do
    extra=""; [ "$c" = cfg5 ] && extra="--kmeans-iters-set 1"
    echo "[$v] $c: $(timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline $extra 2>&1 | grep -o '"value": [0-9.]*, "unit\|"lookup": [0-9.]*\|"sparse_attention": [0-9.]*' | tr '\n' ' ')"
  done
done
cp /tmp/libsqz_new.so paper_2411_09688_b200/libsqz.so
