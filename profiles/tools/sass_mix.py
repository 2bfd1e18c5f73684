"""Dynamic instruction mix and stall attribution from an ncu source page
(ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
inst = defaultdict(int)
stall = defaultdict(lambda: defaultdict(int))
samples = defaultdict(int)
tot_inst = 0
tot_samp = 0
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    base = op.split(".")[0]
    n = int(r[ix["Instructions Executed"]] or 0)
    inst[base] += n
    tot_inst += n
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    samples[base] += s
    tot_samp += s
    for c in stall_cols:
        stall[base][c] += int(r[ix[c]] or 0)
print(f"total warp instructions {tot_inst}, stall samples {tot_samp}")
print(f"{'op':10s} {'inst':>12s} {'%inst':>6s} {'%samp':>6s}  top stalls")
for op, n in sorted(inst.items(), key=lambda x: -x[1])[:30]:
    st = sorted(stall[op].items(), key=lambda x: -x[1])[:3]
    sts = ", ".join(f"{k[6:]} {100.0 * v / max(tot_samp, 1):.1f}" for k, v in st if v)
    print(f"{op:10s} {n:12d} {100.0 * n / tot_inst:6.1f} {100.0 * samples[op] / tot_samp:6.1f}  {sts}")
