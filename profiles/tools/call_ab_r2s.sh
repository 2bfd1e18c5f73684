# Round-2 (session 4) A/B, seventeenth pass: grad_kernel with per-thread descriptor reads (gdesc: 12 blocks/SM, gdesc10: 10)
set -x
O=gpurun_out/ab_r2s
mkdir -p $O
AB_ARGS="--config c4" bash profiles/tools/ab_env.sh 3 g12:: gdesc:gdesc: gdesc10:gdesc10: > $O/ab_c4.txt 2>&1
LIB=paper_2507_04991_b200/libperrk_b200.so
cp $LIB ab/orig.so.bak
for v in gdesc gdesc10; do
  cp ab/$v.so $LIB
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:grad_kernel --launch-skip 8 -c 8 --csv --log-file $O/grad_$v.csv python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
cp ab/gdesc.so $LIB
timeout 600 python -m pytest tests/test_gpu_nsf.py tests/test_gpu_configs.py tests/test_gpu_long_parity.py -q -x -p no:cacheprovider > $O/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> $O/gpu_tests.txt
cp ab/orig.so.bak $LIB
echo done
