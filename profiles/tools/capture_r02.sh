# Round-2 evidence capture on one B200 (outputs under gpurun_out/r02/).
set -x
O=gpurun_out/r02
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt
nproc > $O/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > $O/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> $O/gpu_tests.txt
timeout 900 python tests/long_parity.py c1 c1ref c2 c3 c4 c5 --json $O/long_parity.json > $O/long_parity.txt 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
# launch list of the default workload (cold-cache, serialised: shares, not absolute times)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c5.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
# DRAM bytes of one step's 14 stage launches
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:stage3w --launch-skip 14 -c 14 --csv --log-file $O/stage_traffic.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
# full captures: stage 0 (all cells) and a level-1 stage of the warp-per-cell kernel
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage3w --launch-skip 14 -c 1 -f -o $O/w3_stage0 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage3w --launch-skip 20 -c 1 -f -o $O/w3_stage6 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:relax --launch-skip 0 -c 2 -f -o $O/relax python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:stage2w --launch-skip 20 -c 1 -f -o $O/c3_stage2w python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"grad_kernel|stage_kernel" --launch-skip 8 -c 2 -f -o $O/c4_kernels python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
# text exports on the box (gpurun copies back at most 64 MiB: the .ncu-rep files stay there)
for r in w3_stage0 w3_stage6 relax c3_stage2w c4_kernels; do
  [ -f $O/$r.ncu-rep ] && python profiles/summarize_ncu.py $O/$r.ncu-rep > $O/${r}_ncu.txt 2>&1
done
ncu -i $O/w3_stage6.ncu-rep --page source --csv --print-source sass > $O/w3_stage6_sass.csv 2>/dev/null
ncu -i $O/w3_stage6.ncu-rep --page source --csv --print-source cuda,sass > $O/w3_stage6_lines.csv 2>/dev/null
python profiles/tools/sass_mix.py $O/w3_stage6_sass.csv > $O/sass_mix.txt 2>&1
python profiles/tools/line_mix.py $O/w3_stage6_lines.csv >> $O/sass_mix.txt 2>&1
ncu -i $O/w3_stage6.ncu-rep --page details > $O/w3_stage6_details.txt 2>/dev/null
gzip -f $O/w3_stage6_sass.csv $O/w3_stage6_lines.csv
rm -f $O/*.ncu-rep
du -sh gpurun_out
# the reference arm at the driver's default K / W (full C5 mesh, all host threads)
timeout 1500 python bench.py --impl reference > $O/reference_arm.json 2> $O/reference_arm.err
echo done
