# Round-2 (session 4) A/B, second pass: direct epilogue (COAL=0) with streaming
# cache operators, without the L2 prefetch, and with one 12- / 16-warp block per SM.
set -x
O=gpurun_out/ab_r2c
mkdir -p $O
bash profiles/tools/ab_env.sh 3 swz:swz: coal0:coal0: c0cs:c0cs: c0nopf:c0nopf: c0w12:c0w12: c0w12cs:c0w12cs: c0w16:c0w16: w12:w12: > $O/ab.txt 2>&1
LIB=paper_2507_04991_b200/libperrk_b200.so
cp $LIB ab/orig.so.bak
for v in coal0 c0cs c0nopf c0w12cs; do
  cp ab/$v.so $LIB
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:stage3w --launch-skip 14 -c 14 --csv --log-file $O/traffic_$v.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
cp ab/orig.so.bak $LIB
echo done
