# Round-2 (session 4) A/B, fourteenth pass: L2 prefetch of the K1 traces the surface pre-pass reads (unfpf)
set -x
O=gpurun_out/ab_r2p
mkdir -p $O
bash profiles/tools/ab_env.sh 3 new:: unfpf:unfpf: > $O/ab.txt 2>&1
LIB=paper_2507_04991_b200/libperrk_b200.so
cp $LIB ab/orig.so.bak
for v in orig unfpf; do
  [ $v = orig ] && cp ab/orig.so.bak $LIB || cp ab/$v.so $LIB
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:stage3w --launch-skip 14 -c 14 --csv --log-file $O/launch_$v.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
cp ab/orig.so.bak $LIB
echo done
