# A/B: epilogue bulk loads (epi1) vs slice staging (epi0); then tests on epi1.
set -x
mkdir -p gpurun_out
bash profiles/tools/ab.sh 3 epi0 epi1 > gpurun_out/ab_epi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.txt
OUT=gpurun_out timeout 600 python configs/c1_pair_scan.py > gpurun_out/c1_pair_scan.txt 2>&1
echo done
