set -x
mkdir -p gpurun_out
bash profiles/tools/ab.sh 4 pf0 pf1 > gpurun_out/ab_pf.txt 2>&1
cp ab/pf1.so paper_2507_04991_b200/libperrk_b200.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_slab.py -q -p no:cacheprovider > gpurun_out/pf1_tests.txt 2>&1
echo done
