"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
k = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[k]
body = [r for r in rows[k + 1:] if len(r) == len(hdr) and r[0] != "Address"]
si, src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[si] or 0) for r in body)
top = sorted(body, key=lambda r: -float(r[si] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for r in top:
    main = sorted(((float(r[hdr.index(c)] or 0), c[6:]) for c in cols), reverse=True)[:2]
    print(f"{float(r[si]) / tot * 100:5.1f}%  {r[src].strip()[:70]:70s} {main}")
