#!/usr/bin/env python
"""Instruction mix of one kernel from an ncu source page: executed warp
instructions by opcode (first token), top N.  usage: ncu_opmix.py REPORT KERNEL [N]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
seen, mix = set(), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) != len(h) or r[0] in seen or r[0] == "Address":
        continue
    seen.add(r[0])
    try:
        e = float(r[ix["Instructions Executed"]])
    except Exception:
        continue
    toks = r[ix["Source"]].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    mix[op.split(".")[0]] += e
tot = sum(mix.values())
print(f"total {tot:.0f}")
for op, e in mix.most_common(N):
    print(f"{op:12s} {e:14.0f} {e/tot*100:5.1f}%")
