set -x
mkdir -p gpurun_out
cp paper_2507_04991_b200/libperrk_b200.so ab/cur.so
for v in gk0 gr0 gr1 cur; do
  cp ab/$v.so paper_2507_04991_b200/libperrk_b200.so
  timeout 300 python tests/long_parity.py c4 --json gpurun_out/lp_c4_$v.json > /dev/null 2>&1
done
cp ab/cur.so paper_2507_04991_b200/libperrk_b200.so
echo done
