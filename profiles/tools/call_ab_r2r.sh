# Round-2 (session 4) A/B, sixteenth pass: grad_kernel (C4, BR1) compiled for 12 / 16 resident blocks per SM
set -x
O=gpurun_out/ab_r2r
mkdir -p $O
AB_ARGS="--config c4" bash profiles/tools/ab_env.sh 3 new:: g12:g12: g16:g16: > $O/ab_c4.txt 2>&1
LIB=paper_2507_04991_b200/libperrk_b200.so
cp $LIB ab/orig.so.bak
for v in orig g12 g16; do
  [ $v = orig ] && cp ab/orig.so.bak $LIB || cp ab/$v.so $LIB
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:grad_kernel --launch-skip 8 -c 8 --csv --log-file $O/grad_$v.csv python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
cp ab/orig.so.bak $LIB
for c in c1 c3; do timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
echo done
