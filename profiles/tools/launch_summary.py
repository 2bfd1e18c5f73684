"""Launch list summary from `ncu --metrics gpu__time_duration.sum --csv` of a
bench run: the launches of the last full step (from the last begin_step_kernel
on... back one step) and each kernel's share of that step.  Times are
cold-cache and serialised: compare shares, not absolute times.
usage: python profiles/tools/launch_summary.py launches.csv > summary.txt"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
L = []
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[ix["Metric Value"]].replace(",", ""))
    u = r[ix["Metric Unit"]]
    v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(u, 1.0)
    name = r[ix["Kernel Name"]].split("(")[0].replace("perrk::dev::", "")
    L.append((name, v))
starts = [i for i, (n, _) in enumerate(L) if "begin_step_kernel" in n]
if len(starts) >= 2:
    a, b = starts[-2], starts[-1]
else:
    a, b = 0, len(L)
step = L[a:b]
tot = sum(v for _, v in step)
print(f"{len(L)} launches in the capture; launches {a}-{b - 1} = one full step, {tot:.1f} us (serialised, cold-cache)")
for i, (n, v) in enumerate(step):
    print(f"{i:6d} {n:48s} {v:10.1f} us")
agg = OrderedDict()
for n, v in step:
    agg.setdefault(n, [0, 0.0])
    agg[n][0] += 1
    agg[n][1] += v
print("\nshare of the step by kernel:")
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {n:48s} x{c:<3d} {v:10.1f} us  {100 * v / tot:5.1f} %")
