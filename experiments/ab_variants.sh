#!/bin/bash
# A/B of attention kernel variants at two retentions (run on the GPU box)
run() { python bench.py --no-cpu-baseline --steps 50 --retention $2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 ret=$2', d['value'], d['phases_ms'], d['roofline']['achieved'], d['roofline']['frac'])"; }
python paper_2411_09688_b200/build.py --force > /dev/null 2>&1
run cpasync 0.3; run cpasync 1.0
cp paper_2411_09688_b200/csrc/attention.cu /tmp/attn_cur.cu
cp experiments/attention_tma.cu paper_2411_09688_b200/csrc/attention.cu
python paper_2411_09688_b200/build.py --force > /dev/null 2>&1
run tma 0.3; run tma 1.0
cp /tmp/attn_cur.cu paper_2411_09688_b200/csrc/attention.cu
