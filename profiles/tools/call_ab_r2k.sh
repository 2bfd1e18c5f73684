# Round-2 (session 4) A/B, ninth pass: in-tree build (unformed-neighbour U staging, unguarded dH logarithm,
# 2D direct epilogue, record-buffer floor) against the previous build (flat)
set -x
O=gpurun_out/ab_r2k
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_configs.py tests/test_gpu_spec_criteria.py -q -x -p no:cacheprovider > $O/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> $O/gpu_tests.txt
bash profiles/tools/ab_env.sh 3 flat:flat: new:: > $O/ab.txt 2>&1
AB_ARGS="--config c3" bash profiles/tools/ab_env.sh 3 flat:flat: new:: > $O/ab_c3.txt 2>&1
AB_ARGS="--config c1" bash profiles/tools/ab_env.sh 2 flat:flat: new:: > $O/ab_c1.txt 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
echo done
