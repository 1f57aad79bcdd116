"""Markdown table of bench lines (profiles/<round>/<session>/bench_*.json): ms per iteration, throughput,
model bytes, iteration fraction, top kernel and its fraction, SM clock."""
import glob
import json
import os
import sys

d = sys.argv[1]
print("| file | ms per iteration | unknowns/s | model B/unknown | iteration frac | top kernel | its frac | SM MHz |")
print("|---|---|---|---|---|---|---|---|")
for f in sorted(glob.glob(os.path.join(d, "bench_*.json"))):
    try:
        j = json.load(open(f))
    except Exception:
        continue
    r = j.get("roofline") or {}
    it = r.get("iteration") or {}
    pk = r.get("per_kernel_ms") or {}
    k = r.get("kernel")
    c = j.get("clocks") or {}
    if not r:
        print(f"| {os.path.basename(f)} | {j.get('ms_per_step', 0):.4g} | {j.get('value', 0):.4g} | | | | | |")
        continue
    print(f"| {os.path.basename(f)} | {j['ms_per_step']:.4g} | {j['value']:.4g} | {it.get('model_bytes_per_unknown')} | "
          f"{it.get('frac', 0):.3f} | {k} {pk.get(k, 0):.4g} ms | {r.get('frac', 0):.3f} | {c.get('sm_mhz')} {','.join(c.get('reasons') or [])} |")
