#!/bin/bash
# One GPU-box pass: GPU tests (with printed parity metrics), the default bench,
# the reference arm.  Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
nproc > gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
