"""Summarise an ncu --page source --csv dump: top stall instructions per kernel with stall reasons.
usage: python scripts/ncu_src.py dump.csv [kernel_index] [topN]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
kidx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
blk = rows[starts[kidx]:starts[kidx + 1]]
print(blk[0][1])
hdr = blk[1]
data = [r for r in blk[2:] if len(r) == len(hdr)]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iw = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
base = int(data[0][ia], 16)
tot = sum(int(r[iw]) for r in data)
print("total samples", tot)
stall_cols = [(j, h) for j, h in enumerate(hdr) if h.startswith("stall_") and "(Not Issued)" not in h]
agg = {}
for r in data:
    for j, h in stall_cols:
        try:
            agg[h] = agg.get(h, 0) + float(r[j] or 0)
        except ValueError:
            pass
print("by reason:", ", ".join(f"{h[6:]}={v / tot:.1%}" for h, v in sorted(agg.items(), key=lambda x: -x[1])[:12]))
for r in sorted(data, key=lambda r: -int(r[iw]))[:top]:
    reasons = []
    for j, h in stall_cols:
        try:
            v = float(r[j] or 0)
        except ValueError:
            continue
        if v > 0.1 * int(r[iw]):
            reasons.append(f"{h[6:]}={int(v)}")
    print(f"{int(r[ia], 16) - base:6x} {int(r[iw]):7d} {int(r[ie]):9d}  {r[isrc].strip()[:60]:60s} {' '.join(reasons)}")
