# Round-2 (session 4) A/B, third pass: direct epilogue + streaming operators
# without the L2 prefetch, one 12-warp block per SM, register prefetches, brick order.
set -x
O=gpurun_out/ab_r2d
mkdir -p $O
bash profiles/tools/ab_env.sh 3 c0nopf:c0nopf: c0ncs:c0ncs: c0w12ncs:c0w12ncs: c0w12ncs_b0:c0w12ncs:PERRK_BRICK=0 c0w12ncse:c0w12ncse: c0w12ncspf:c0w12ncspf: c0w12ncsepf:c0w12ncsepf: c0w12e:c0w12e: > $O/ab.txt 2>&1
LIB=paper_2507_04991_b200/libperrk_b200.so
cp $LIB ab/orig.so.bak
for v in c0ncs c0w12ncs c0w12ncse; do
  cp ab/$v.so $LIB
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:stage3w --launch-skip 14 -c 14 --csv --log-file $O/traffic_$v.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
cp ab/c0w12ncs.so $LIB
PERRK_BRICK=0 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:stage3w --launch-skip 14 -c 14 --csv --log-file $O/traffic_c0w12ncs_b0.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
cp ab/orig.so.bak $LIB
echo done
