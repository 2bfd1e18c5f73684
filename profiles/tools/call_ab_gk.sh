set -x
mkdir -p gpurun_out
AB_ARGS="--config c4" bash profiles/tools/ab.sh 3 gk0 gk1 > gpurun_out/ab_gk.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_nsf.py tests/test_gpu_reference_numerics.py -q -s -p no:cacheprovider > gpurun_out/nsf_tests.txt 2>&1
echo done
