# Round-2 (session 4) A/B, fourth pass: own-block prefetch forms on the best 3D
# variant (12-warp block, direct streaming epilogue from registers, no L2
# prefetch), and the 2D kernels without their L2 prefetch (C3, C4).
set -x
O=gpurun_out/ab_r2e
mkdir -p $O
bash profiles/tools/ab_env.sh 3 c0w12ncse:c0w12ncse: c0w12ncseo:c0w12ncseo: c0w12cse_l2:c0w12cse_l2: c0ncse:c0ncse: c0ncs:c0ncs: > $O/ab.txt 2>&1
AB_ARGS="--config c3" bash profiles/tools/ab_env.sh 3 st1:c0w12ncse: st0:st0: > $O/ab_c3.txt 2>&1
AB_ARGS="--config c4" bash profiles/tools/ab_env.sh 3 st1:c0w12ncse: st0:st0: > $O/ab_c4.txt 2>&1
LIB=paper_2507_04991_b200/libperrk_b200.so
cp $LIB ab/orig.so.bak
for v in c0w12ncseo c0w12cse_l2; do
  cp ab/$v.so $LIB
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:stage3w --launch-skip 14 -c 14 --csv --log-file $O/traffic_$v.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
cp ab/orig.so.bak $LIB
echo done
