"""Shared-memory instructions with excessive wavefronts (bank conflicts) from an ncu SASS source page
(`ncu -i rep --page source --csv --print-source sass -k regex:K`), grouped by CUDA source line when the
report carries -lineinfo correlation (--print-source sass,cuda is not needed: SASS rows only)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
k = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[k]
body = [r for r in rows[k + 1:] if len(r) == len(hdr) and r[0] != "Address"]
ix = {h: i for i, h in enumerate(hdr)}
tot_w = sum(float(r[ix["L1 Wavefronts Shared"]] or 0) for r in body)
tot_x = sum(float(r[ix["L1 Wavefronts Shared Excessive"]] or 0) for r in body)
print(f"shared wavefronts {tot_w:.3e}, excessive {tot_x:.3e}")
top = sorted(body, key=lambda r: -float(r[ix["L1 Wavefronts Shared Excessive"]] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]
for r in top:
    x = float(r[ix["L1 Wavefronts Shared Excessive"]] or 0)
    if x <= 0:
        break
    print(f"{x / tot_x * 100:5.1f}%  {r[ix['Address']]}  {r[ix['Source']].strip()[:60]:60s} ideal {r[ix['L1 Wavefronts Shared Ideal']]} actual {r[ix['L1 Wavefronts Shared']]}")
