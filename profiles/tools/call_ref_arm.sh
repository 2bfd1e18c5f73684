set -x
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_arm_short.json 2> gpurun_out/ref_arm_short.err; echo "secs=$SECONDS" >> gpurun_out/ref_arm_short.err
echo done
