# Round-2 (session 4) A/B, fifteenth pass: 2D warp kernel with hoisted descriptor reads and straight-line
# staging / surface / gather (w2flat), C3 and C1
set -x
O=gpurun_out/ab_r2q
mkdir -p $O
AB_ARGS="--config c3" bash profiles/tools/ab_env.sh 3 new:: w2flat:w2flat: > $O/ab_c3.txt 2>&1
AB_ARGS="--config c1" bash profiles/tools/ab_env.sh 2 new:: w2flat:w2flat: > $O/ab_c1.txt 2>&1
LIB=paper_2507_04991_b200/libperrk_b200.so
cp $LIB ab/orig.so.bak
cp ab/w2flat.so $LIB
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> $O/gpu_tests.txt
cp ab/orig.so.bak $LIB
echo done
