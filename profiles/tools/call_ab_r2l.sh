# Round-2 (session 4) A/B, tenth pass: next own state into registers after the epilogue (regpf3)
set -x
O=gpurun_out/ab_r2l
mkdir -p $O
bash profiles/tools/ab_env.sh 3 new:: regpf3:regpf3: > $O/ab.txt 2>&1
echo done
