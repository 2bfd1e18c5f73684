# Round-2 (session 4) A/B, eleventh pass: relaxation kernels with a register prefetch of the next
# block (rpf: 3 blocks/SM, spills; rpf2: 2 blocks/SM) against no prefetch (r3: 3 blocks/SM, r2: 2)
set -x
O=gpurun_out/ab_r2m
mkdir -p $O
LIB=paper_2507_04991_b200/libperrk_b200.so
cp $LIB ab/orig.so.bak
for v in r3 r2 rpf rpf2; do
  cp ab/$v.so $LIB
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:relax --launch-skip 10 -c 10 --csv --log-file $O/relax_$v.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
cp ab/orig.so.bak $LIB
bash profiles/tools/ab_env.sh 3 r3:r3: r2:r2: rpf:rpf: rpf2:rpf2: > $O/ab.txt 2>&1
echo done
