set -x
mkdir -p gpurun_out
AB_ARGS="--config c4" bash profiles/tools/ab.sh 3 gr0 gr1 > gpurun_out/ab_gr.txt 2>&1
cp ab/gr1.so paper_2507_04991_b200/libperrk_b200.so
timeout 600 python -m pytest tests/test_gpu_nsf.py tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/gr1_tests.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c4b.csv python bench.py --config c4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
