set -x
mkdir -p gpurun_out
bash profiles/tools/ab.sh 3 lp0 lp1 hp1 > gpurun_out/ab_lp.txt 2>&1
echo done
