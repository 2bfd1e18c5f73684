# Round-2 (session 4) A/B, eighteenth pass: grad_kernel at 10 (in-tree) and 8 resident blocks per SM
set -x
O=gpurun_out/ab_r2t
mkdir -p $O
AB_ARGS="--config c4" bash profiles/tools/ab_env.sh 3 gdesc10:: gdesc8:gdesc8: > $O/ab_c4.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_nsf.py tests/test_gpu_configs.py -q -x -p no:cacheprovider > $O/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> $O/gpu_tests.txt
timeout 600 python bench.py --config c4 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --config c2 > $O/bench_c2.json 2> $O/bench_c2.err
echo done
