set -x
mkdir -p gpurun_out
bash profiles/tools/ab.sh 3 sp0 sp1 > gpurun_out/ab_sp.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_slab.py -q -p no:cacheprovider > gpurun_out/gpu_tests_sp.txt 2>&1
echo done
