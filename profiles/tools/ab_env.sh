#!/bin/bash
# usage: profiles/tools/ab_env.sh ROUNDS NAME:LIB:ENV ...
# Alternate short bench runs of variants on one box.  LIB is a prebuilt
# library under ab/ (empty: the in-tree one), ENV a comma-separated list of
# VAR=VALUE pairs.  Columns: variant, DOF-stage/s, stage-kernel ms per launch,
# SM MHz.  AB_ARGS adds bench.py arguments (e.g. "--config c3").
LIB=paper_2507_04991_b200/libperrk_b200.so
cp $LIB ab/orig.so.bak
R=$1; shift
for i in $(seq 1 $R); do
  for spec in "$@"; do
    IFS=: read -r name lib envs <<< "$spec"
    if [ -n "$lib" ]; then cp ab/$lib.so $LIB; else cp ab/orig.so.bak $LIB; fi
    r=$(env $(echo $envs | tr ',' ' ') timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $AB_ARGS 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.4f %s' % (d['value'], d['roofline']['ms_per_launch'], d['clocks']['sm_mhz']))" 2>&1)
    echo "$name $r"
  done
done
cp ab/orig.so.bak $LIB
