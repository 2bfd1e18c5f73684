# Round-2 (session 4) A/B, nineteenth pass: beta and sound speed of the own nodes from one reciprocal square root (rsq)
set -x
O=gpurun_out/ab_r2u
mkdir -p $O
bash profiles/tools/ab_env.sh 3 new:: rsq:rsq: > $O/ab.txt 2>&1
LIB=paper_2507_04991_b200/libperrk_b200.so
cp $LIB ab/orig.so.bak
cp ab/rsq.so $LIB
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_fused.py tests/test_gpu_slab.py tests/test_gpu_long_parity.py -q -x -p no:cacheprovider > $O/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> $O/gpu_tests.txt
timeout 600 python tests/long_parity.py c5 --json $O/long_parity_c5.json > $O/long_parity_c5.txt 2>&1
cp ab/orig.so.bak $LIB
echo done
