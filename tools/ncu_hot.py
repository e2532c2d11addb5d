"""Summarise an ncu --page source --print-source sass CSV: hottest SASS lines
with their dominant stall reasons (tools for reading captures here, no GPU)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    top = sorted(((float(r[ix[h]] or 0), h[6:]) for h in stalls), reverse=True)[:3]
    data.append((s, r[0][-5:], r[1].strip()[:70], top, r[ix["Instructions Executed"]]))
tot = sum(d[0] for d in data) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for s, a, src, top, ex in sorted(data, reverse=True)[:n]:
    print(f"{s / tot * 100:5.1f}% {a} {src:70s} exec={ex:>10s} " + " ".join(f"{k}:{v:.0f}" for v, k in top if v))
