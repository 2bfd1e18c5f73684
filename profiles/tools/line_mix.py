"""Per source line: instructions executed and stall samples, from
ncu --page source --csv --print-source cuda,sass."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
cur_file = None
hdr = None
agg = defaultdict(lambda: [0, 0, ""])
ln = None
tot_i = tot_s = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or r[0] in ("Function Name",):
        continue
    if r[0].strip():
        ln = (cur_file, int(r[0]))
        agg[ln][2] = r[1].strip()[:70]
    try:
        n = int(r[hdr["Instructions Executed"]] or 0)
        s = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, IndexError):
        continue
    if ln:
        agg[ln][0] += n
        agg[ln][1] += s
        tot_i += n
        tot_s += s
print(f"total inst {tot_i}, samples {tot_s}")
top = sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 50]
for (f, l), (n, s, src) in top:
    print(f"{f}:{l:5d} {100.0 * n / tot_i:5.1f}%i {100.0 * s / tot_s:5.1f}%s  {src}")
