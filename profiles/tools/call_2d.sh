# 2D configurations (C3, C4): bench lines, launch lists, one full ncu capture
# of the block-per-cell stage kernel each; plus the SPEC-criteria GPU tests.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_spec_criteria.py -q -s -p no:cacheprovider > gpurun_out/spec_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/spec_tests.txt
for c in c3 c4; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage_kernel --launch-skip 12 -c 1 -f -o gpurun_out/stage2d_$c python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$c.log 2>&1
done
