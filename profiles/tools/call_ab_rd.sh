set -x
mkdir -p gpurun_out
bash profiles/tools/ab.sh 3 rd0 rd1 > gpurun_out/ab_rd.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
