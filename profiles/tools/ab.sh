#!/bin/bash
# usage: ab/ab.sh ROUNDS V1 V2 ...  -- alternate bench runs of ab/V*.so
LIB=paper_2507_04991_b200/libperrk_b200.so
cp $LIB ab/orig.so.bak
R=$1; shift
for i in $(seq 1 $R); do
  for v in "$@"; do
    cp ab/$v.so $LIB
    r=$(timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $AB_ARGS 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.4f %s' % (d['value'], d['roofline']['ms_per_launch'], d['clocks']['sm_mhz']))" 2>&1)
    echo "$v $r"
  done
done
cp ab/orig.so.bak $LIB
