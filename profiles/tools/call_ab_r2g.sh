# Round-2 (session 4) A/B, fifth pass: fewer L1 data-pipe wavefronts per cell
# (the pipe is at 70-80% of its peak): z-face terms added by the owning lane
# (zown), own primitives from registers in the volume phase (ownreg), descriptor
# through registers (zod), z-face round from registers (zodr).
set -x
O=gpurun_out/ab_r2g
mkdir -p $O
bash profiles/tools/ab_env.sh 3 def:: zown:zown: ownreg:ownreg: zod:zod: zodr:zodr: > $O/ab.txt 2>&1
LIB=paper_2507_04991_b200/libperrk_b200.so
cp $LIB ab/orig.so.bak
cp ab/zodr.so $LIB
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_slab.py tests/test_gpu_configs.py -q -x -p no:cacheprovider > $O/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> $O/gpu_tests.txt
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:stage3w --launch-skip 14 -c 14 --csv --log-file $O/metrics_zodr.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
cp ab/orig.so.bak $LIB
echo done
