"""Attribute ncu warp-stall samples (--page source --csv, SASS view) of one
kernel to CUDA source lines via `nvdisasm -gi` line info of the same cubin.

  python tools/ncu_lines.py <src.csv> <disasm.txt> <mangled kernel name> [top]
"""
import csv
import re
import sys
from collections import defaultdict

src_csv, dis, fun = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40

# offset -> "line (inlined-at chain)"
lines = {}
cur = None
in_fun = False
pending = None
for raw in open(dis):
    if raw.startswith("\t.text.") or ".text." in raw and raw.strip().endswith(":"):
        in_fun = fun in raw
    if not in_fun:
        continue
    m = re.search(r'//## File ".*?([^/]+)", line (\d+)(.*)', raw)
    if m:
        inl = re.findall(r'line (\d+)', m.group(3))
        pending = f"{m.group(1)}:{m.group(2)}" + (f" <- {','.join(inl)}" if inl else "")
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", raw)
    if m and pending:
        lines[int(m.group(1), 16)] = (pending, m.group(2).strip())

rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
base = None
agg = defaultdict(lambda: defaultdict(int))
tot = 0
for r in rows[2:]:
    if len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    a = int(r[0], 16)
    base = a if base is None else base
    off = a - base
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    tot += s
    key = lines.get(off, ("?", r[1]))[0]
    agg[key]["_"] += s
    for h in stalls:
        agg[key][h[6:]] += int(r[idx[h]] or 0)
print("total samples", tot)
for key, d in sorted(agg.items(), key=lambda kv: -kv[1]["_"])[:top]:
    t = sorted(((v, k) for k, v in d.items() if k != "_"), reverse=True)[:3]
    print(f"{d['_']:7d} {100.0 * d['_'] / max(tot, 1):5.1f}%  {key:40s} {t}")
