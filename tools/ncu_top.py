"""Top SASS instructions of one ncu --set full capture by warp-stall samples.

  ncu -i rep --page source --csv > src.csv ; python tools/ncu_top.py src.csv [N] [lo-hi hex window]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
win = None
if len(sys.argv) > 3:
    lo, hi = sys.argv[3].split("-")
    win = (int(lo, 16), int(hi, 16))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data, base = [], None
for r in rows[2:]:
    if len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    a = int(r[0], 16)
    base = a if base is None else base
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    ex = int(r[idx["Instructions Executed"]] or 0)
    data.append((a - base, s, ex, r[1].strip(), r))
tot = sum(d[1] for d in data)
print("total samples", tot)
sel = [d for d in data if win is None or win[0] <= d[0] <= win[1]]
if win is None:
    sel = sorted(sel, key=lambda d: -d[1])[:n]
for off, s, ex, src, r in sel:
    t = sorted(((int(r[idx[h]] or 0), h[6:]) for h in stalls), reverse=True)[:2]
    print(f"{off:6x} {s:5d} {100.0 * s / max(tot, 1):4.1f}% ex={ex:8d} {src[:64]:64s} {t}")
