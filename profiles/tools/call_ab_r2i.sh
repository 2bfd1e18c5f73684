# Round-2 (session 4) A/B, seventh pass: straight-line surface phase and staging (flat),
# and the 2 x 8-warp configuration with the new levers (h8: OWNREG, h8o: without)
set -x
O=gpurun_out/ab_r2i
mkdir -p $O
bash profiles/tools/ab_env.sh 3 hoist:: flat:flat: h8:h8: h8o:h8o: > $O/ab.txt 2>&1
LIB=paper_2507_04991_b200/libperrk_b200.so
cp $LIB ab/orig.so.bak
cp ab/flat.so $LIB
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_slab.py tests/test_gpu_configs.py tests/test_gpu_nsf.py -q -x -p no:cacheprovider > $O/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> $O/gpu_tests.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage3w --launch-skip 20 -c 1 -f -o $O/w3_stage6 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python profiles/summarize_ncu.py $O/w3_stage6.ncu-rep > $O/w3_stage6_ncu.txt 2>&1
ncu -i $O/w3_stage6.ncu-rep --page source --csv --print-source sass > $O/w3_stage6_sass.csv 2>/dev/null
gzip -f $O/w3_stage6_sass.csv
rm -f $O/*.ncu-rep
cp ab/orig.so.bak $LIB
echo done
