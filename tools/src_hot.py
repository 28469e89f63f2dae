"""Aggregate warp-stall samples of an `ncu --page source --csv --print-source cuda,sass`
export per CUDA source line.  Usage: python tools/src_hot.py mix.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, agg = None, None, {}
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0] != "":
        cur = (fname, int(r[0]), r[1][:90])
        num = lambda x: int(x) if x.strip().isdigit() else 0
        samp, ex = num(r[4]), num(r[7])
        a = agg.setdefault(cur, [0, 0])
        a[0] += samp
        a[1] += ex
tot = sum(v[0] for v in agg.values())
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]:7d} {100 * v[0] / max(tot, 1):5.1f}% inst={v[1]:8d}  {k[0]}:{k[1]}  {k[2]}")
