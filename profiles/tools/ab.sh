#!/bin/bash
# usage: scratch/ab.sh N  -- alternate bench runs of scratch/A.so and scratch/B.so (N rounds)
LIB=paper_2507_04991_b200/libperrk_b200.so
for i in $(seq 1 ${1:-2}); do
  for v in ${VARIANTS:-A B}; do
    cp scratch/$v.so $LIB
    r=$(python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.4f' % (d['value'], d['roofline']['ms_per_launch']))")
    echo "$v $r"
  done
done
