# compute-sanitizer (memcheck, racecheck) over smoke() and the partition / parity GPU tests of small meshes
set -x
O=gpurun_out/sanitize
mkdir -p $O
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 3 python -c "import __graft_entry__ as g; g.smoke()" > $O/memcheck_smoke.txt 2>&1; echo "rc=$?" >> $O/memcheck_smoke.txt
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 3 python -m pytest tests/test_gpu_slab.py tests/test_gpu_traversal.py -q -x -p no:cacheprovider > $O/memcheck_slab.txt 2>&1; echo "rc=$?" >> $O/memcheck_slab.txt
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 3 python -c "import __graft_entry__ as g; g.smoke()" > $O/racecheck_smoke.txt 2>&1; echo "rc=$?" >> $O/racecheck_smoke.txt
tail -5 $O/*.txt
echo done
