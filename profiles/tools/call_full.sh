set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.txt
timeout 600 python tests/long_parity.py c1 c1ref c2 c3 c4 c5 --json gpurun_out/long_parity.json > gpurun_out/long_parity.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done
