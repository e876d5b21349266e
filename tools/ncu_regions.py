#!/usr/bin/env python
"""Group SASS of one kernel into runs of equal execution count; print runs that
carry >1.5% of instructions or >2% of stall samples.
usage: ncu_regions.py REPORT KERNEL_REGEX [show_from show_to]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}


def f(x):
    try:
        return float(x)
    except Exception:
        return 0.0


body = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0] != "Address"]
seen, b2 = set(), []
for r in body:
    if r[0] in seen:
        continue
    seen.add(r[0])
    b2.append(r)
tot = sum(f(r[ix["Instructions Executed"]]) for r in b2)
ts = sum(f(r[ix["Warp Stall Sampling (All Samples)"]]) for r in b2)
stalls = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
agg = {x: sum(f(r[ix[x]]) for r in b2) for x in stalls}
print(f"instr={tot:.0f} stall_samples={ts:.0f} sass={len(b2)}")
print("stalls:", ", ".join(f"{k[6:]}={v/ts*100:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
if len(sys.argv) > 4:
    for r in b2[int(sys.argv[3]):int(sys.argv[4])]:
        print(f"{f(r[ix['Instructions Executed']]):10.0f} {f(r[ix['Warp Stall Sampling (All Samples)']]):6.0f} {r[ix['Source']][:90]}")
    sys.exit()
prev, start, n, st = None, 0, 0, 0.0
for k in range(len(b2) + 1):
    e = f(b2[k][ix["Instructions Executed"]]) if k < len(b2) else -1
    if e != prev:
        if prev is not None and (prev * n > tot * 0.015 or st > ts * 0.02):
            print(f"{start:5d}-{k-1:5d} n={n:4d} exec={prev:10.0f} instr={prev*n/tot*100:5.1f}% "
                  f"stall={st/ts*100:5.1f}%  {b2[start][ix['Source']][:48]}")
        prev, start, n, st = e, k, 0, 0.0
    if k < len(b2):
        n += 1
        st += f(b2[k][ix["Warp Stall Sampling (All Samples)"]])
