#!/usr/bin/env python
"""Instructions executed and stall samples per CUDA source line of one kernel
(ncu cuda,sass source view).  usage: ncu_lines.py REPORT KERNEL_REGEX [N]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
def f(x):
    try: return float(x)
    except Exception: return 0.0
fname, acc = "?", {}
ie = st = None
seen_launch = set()
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        ie = r.index("Instructions Executed"); st = r.index("Warp Stall Sampling (All Samples)"); continue
    if ie is None or len(r) <= ie: continue
    if r[0] != "":  # cuda line row with aggregated metrics
        key = (fname, int(r[0]))
        a = acc.setdefault(key, [0.0, 0.0, r[1].strip()])
        a[0] += f(r[ie]); a[1] += f(r[st])
tot = sum(v[0] for v in acc.values()) or 1; ts = sum(v[1] for v in acc.values()) or 1
print(f"total instr {tot:.3e}  stall samples {ts:.0f}")
for (fn, ln), (a, b, src) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:N]:
    print(f"{a/tot*100:5.1f}% stall {b/ts*100:5.1f}%  {fn}:{ln:<5d} {src[:90]}")
