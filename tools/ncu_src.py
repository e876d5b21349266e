#!/usr/bin/env python
"""Summarise an ncu source page (SASS): hottest instructions by stall samples
and executed count.  usage: ncu_src.py REPORT KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
body = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr) and r[0] != "Address"]
ix = {h: i for i, h in enumerate(hdr)}
def num(r, k):
    try:
        return float(r[ix[k]])
    except Exception:
        return 0.0
tot_s = sum(num(r, "Warp Stall Sampling (All Samples)") for r in body)
tot_i = sum(num(r, "Instructions Executed") for r in body)
print(f"instructions(warp)={tot_i:.0f} stall_samples={tot_s:.0f} sass_lines={len(body)}")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {h: sum(num(r, h) for r in body) for h in stalls}
print("stall totals:", ", ".join(f"{k[6:]}={v:.0f}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
body.sort(key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))
for r in body[:N]:
    top = max(stalls, key=lambda h: num(r, h))
    print(f"{r[0]:>6} {num(r,'Warp Stall Sampling (All Samples)'):7.0f} {num(r,'Instructions Executed'):10.0f} "
          f"{top[6:]:>14} {num(r,'L1 Conflicts Shared N-Way'):4.0f}  {r[1][:90]}")
