# final round-2 bench lines (default C5 and the four 2D configurations) + the traversal-order test
set -x
O=gpurun_out/r02b
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_traversal.py tests/test_gpu_slab.py -q -p no:cacheprovider > $O/gpu_tests_extra.txt 2>&1
echo "pytest rc=$?" >> $O/gpu_tests_extra.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 300 python bench.py --gpus 2 > $O/bench_gpus2.txt 2>&1; echo "rc=$?" >> $O/bench_gpus2.txt
echo done
