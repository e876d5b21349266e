"""Fast Radix overflow model table (NEXT-4): exact expectation (oracle),
Eq. 1 as printed with base 0 / base 1 (parity unpinned), and the GPU Monte
Carlo (dfr_overflow_mc) mean with its 95% half-width, for the (N, M) of the
paper's claim and of this build's passes."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import datagen
from oracle import overflow as ov

rows = [(1000, 256, 20000), (1 << 12, 256, 8000), (1 << 16, 256, 2000), (1 << 20, 256, 512),
        (1 << 24, 256, 64), (4096, 16, 4000)]
gpu = "--gpu" in sys.argv
if gpu:
    import torch
    import paper_2207_14334_b200 as dfr
print(f"{'N':>10} {'M':>5} {'exact E[ovf]/N':>15} {'Eq.1 base0':>11} {'Eq.1 base1':>11} {'GPU MC mean':>12} {'+-95%':>9} {'trials':>7}")
for n, m, trials in rows:
    ex = ov.expected_overflow(n, m)
    e0 = ov.eq1_fraction(n, m, 0.0) if n <= 1 << 16 else float("nan")
    e1 = ov.eq1_fraction(n, m, 1.0) if n <= 1 << 16 else float("nan")
    mc = hw = float("nan")
    if gpu:
        o = dfr.overflow_mc(n, m, trials, datagen.stream_key(11, f"table-{n}-{m}")).double().cpu().numpy() / n
        mc, hw = o.mean(), 1.96 * o.std(ddof=1) / math.sqrt(trials)
    print(f"{n:>10} {m:>5} {ex:>15.6g} {e0:>11.4g} {e1:>11.4g} {mc:>12.6g} {hw:>9.2g} {trials:>7}")
