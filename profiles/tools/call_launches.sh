# launch list of the default bench (ncu gpu__time_duration, serialised) + checks
set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 python configs/check_families_krylov.py > gpurun_out/family_check_krylov.txt 2>&1
timeout 600 python configs/c1_pair_scan.py > gpurun_out/c1_pair_scan.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -s -k adapter -p no:cacheprovider > gpurun_out/adapter.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
echo done
