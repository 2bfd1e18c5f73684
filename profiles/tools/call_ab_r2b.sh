# Round-2 (session 4) A/B: brick traversal order, swizzle-entry masks, register
# prefetch of the next own state, direct epilogue, warps per block / registers.
set -x
O=gpurun_out/ab_r2b
mkdir -p $O
bash profiles/tools/ab_env.sh 3 b0:base:PERRK_BRICK=0 b8:base:PERRK_BRICK=8 b16:base:PERRK_BRICK=16 b4:base:PERRK_BRICK=4 \
  swz:swz: pf1:pf1: pf2:pf2: coal0:coal0: w6:w6: w12:w12: w6pf1:w6pf1: w6pf2:w6pf2: > $O/ab.txt 2>&1
# DRAM bytes of one step's 14 stage launches per traversal order
for b in 0 8 16; do
  PERRK_BRICK=$b timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:stage3w --launch-skip 14 -c 14 --csv --log-file $O/traffic_b$b.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
# correctness of the in-tree build (swizzle-entry masks, brick order on)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_slab.py tests/test_gpu_configs.py -q -x -p no:cacheprovider > $O/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> $O/gpu_tests.txt
echo done
