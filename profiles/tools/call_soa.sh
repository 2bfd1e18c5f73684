# SoA layout: full GPU test suite, default bench, C3 bench, stage-kernel ncu.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage3w --launch-skip 20 -c 1 -f -o gpurun_out/w3_soa python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_soa.log 2>&1
echo done
