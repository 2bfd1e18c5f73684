set -x
mkdir -p gpurun_out
AB_ARGS="--config c4" bash profiles/tools/ab.sh 3 gr1 vs1 > gpurun_out/ab_vs.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.txt
timeout 900 python tests/long_parity.py c1 c1ref c2 c3 c4 c5 --json gpurun_out/long_parity.json > gpurun_out/long_parity.txt 2>&1
echo done
