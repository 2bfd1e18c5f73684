set -x
mkdir -p gpurun_out/ab_r2f
bash profiles/tools/ab_env.sh 3 def:: c8pf:c8pf: c8pfnc:c8pfnc: > gpurun_out/ab_r2f/ab.txt 2>&1
bash profiles/tools/capture_r02.sh > gpurun_out/capture.log 2>&1
echo done
