# Round-2 (session 4) A/B, twentieth pass: neighbour sound speed as z rsqrt(z) in the surface flux (all stage
# kernels) and the 2D warp kernel's beta / c from one reciprocal square root (in-tree) against the build before (prev)
set -x
O=gpurun_out/ab_r2v
mkdir -p $O
bash profiles/tools/ab_env.sh 3 prev:prev: new:: > $O/ab.txt 2>&1
AB_ARGS="--config c3" bash profiles/tools/ab_env.sh 3 prev:prev: new:: > $O/ab_c3.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> $O/gpu_tests.txt
timeout 900 python tests/long_parity.py c1 c1ref c2 c3 c4 c5 --json $O/long_parity.json > $O/long_parity.txt 2>&1
echo done
