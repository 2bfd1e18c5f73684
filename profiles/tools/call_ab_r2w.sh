# Round-2 (session 4) A/B, twenty-first pass: own stage state loaded past L1 (owncg)
set -x
O=gpurun_out/ab_r2w
mkdir -p $O
bash profiles/tools/ab_env.sh 3 base:base: ownel:ownel: > $O/ab.txt 2>&1
echo done
