# Round-2 (session 4) A/B, eighth pass: L1 prefetch of the next cell's own block
set -x
O=gpurun_out/ab_r2j
mkdir -p $O
bash profiles/tools/ab_env.sh 3 flat:: l1pf1:l1pf1: l1pf2:l1pf2: > $O/ab.txt 2>&1
echo done
