"""Summarise an ncu source page (--print-source cuda,sass --csv) by CUDA source line: warp-stall samples,
top N lines.   python tools/ncu_lines.py report.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur = None
data = []
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) >= 3 and r[0] == "Line No":
        hdr = r
        ix = hdr.index("Warp Stall Sampling (All Samples)")
        ixn = hdr.index("Warp Stall Sampling (Not-issued Samples)")
        ie = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) <= ix or not r[0]:
        continue
    try:
        v = float(r[ix]); vn = float(r[ixn]); ne = float(r[ie] or 0)
    except ValueError:
        continue
    data.append((v, vn, ne, cur, r[0], r[1][:100]))
tot = sum(d[0] for d in data)
print(f"total samples {tot:.0f}")
for d in sorted(data, reverse=True)[:top]:
    print(f"{d[0]:7.0f} {100 * d[0] / tot:5.1f}% (not-issued {d[1]:6.0f}, inst {d[2]:9.0f}) {d[3]}:{d[4]}: {d[5]}")
