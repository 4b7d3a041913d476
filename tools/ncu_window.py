"""Warp-stall samples of an ncu --set full capture, per SASS row window.

  ncu -i rep --page source --csv --print-source sass > sass.csv
  python tools/ncu_window.py sass.csv PATTERN [before] [after]   # window around rows matching PATTERN
  python tools/ncu_window.py sass.csv --top N [lo_row] [hi_row]  # top rows by samples
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def num(v):
    try:
        return int(float(v))
    except ValueError:
        return 0


def top_stalls(rs, k=6):
    tot = {s: sum(num(r[idx[s]]) for r in rs) for s in stalls}
    return {s[6:]: v for s, v in sorted(tot.items(), key=lambda x: -x[1])[:k] if v}


total = sum(num(r[2]) for r in data)
print("total samples", total, "rows", len(data))
if sys.argv[2] == "--top":
    n = int(sys.argv[3])
    lo = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    hi = int(sys.argv[5]) if len(sys.argv) > 5 else len(data)
    sel = sorted(range(lo, hi), key=lambda i: -num(data[i][2]))[:n]
    for i in sorted(sel):
        r = data[i]
        print(f"{i:6d} {r[1].strip()[:64]:64s} s={num(r[2]):5d} ex={num(r[5]):8d} {top_stalls([r], 2)}")
else:
    pat = sys.argv[2]
    before = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    after = int(sys.argv[4]) if len(sys.argv) > 4 else 80
    hits = [i for i, r in enumerate(data) if pat in r[1]]
    print("matches at rows", hits[:20])
    if hits:
        c = hits[0]
        w = data[max(0, c - before): c + after]
        print(f"window rows {max(0, c - before)}..{c + after}: samples {sum(num(r[2]) for r in w)}",
              top_stalls(w))
