set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py -q -p no:cacheprovider > gpurun_out/fused_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/fused_tests.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage3w --launch-skip 20 -c 1 -f -o gpurun_out/w3_full python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
