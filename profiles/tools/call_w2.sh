set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_slab.py tests/test_gpu_long_parity.py tests/test_gpu_spectrum.py -q -p no:cacheprovider -x > gpurun_out/gpu_tests_w2.txt 2>&1
echo "rc=$?" >> gpurun_out/gpu_tests_w2.txt
AB_ARGS="--config c3" bash profiles/tools/ab.sh 3 w2off w2on > gpurun_out/ab_w2.txt 2>&1
echo done
