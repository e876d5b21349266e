#!/usr/bin/env python
"""Measured sweeps on one B200.

  python tools/sweeps.py paper [--out F]   the paper's workloads (P:288, P:313,
        P:337; 16-byte records S:22-27) at N = 256^3, 256^3.25, 256^3.5, 2^29,
        256^3.75 = 2^30 (records up to 2^28)
  python tools/sweeps.py nd [--out F]      N_d in {16..256} on c5-uniform / c3
        inputs, and the ablations: separate last pass (no fusion), every pass
        run (no pass skipping), every deal stable (stable_deals), Fast Radix
        estimation, full LSD over all digits (u32)

Each cell: 2 warm-up sorts, then 5 timed sorts, each of a pristine resident
copy (CUDA events around the library call, allocation inside); median ms and
Gkeys/s; the last output is verified (sorted + multiset fingerprint; records:
the O(n) stable-sort certificate on the tags' input positions)."""
import argparse
import json
import math
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def measure(dfr, torch, keys, vals=None, reps=5, warm=2, **kw):
    dev = torch.device("cuda")
    tk = torch.from_numpy(keys.view(np.int64 if keys.dtype == np.uint64 else np.int32)).to(dev)
    tv = None
    if vals is not None:
        tv = torch.from_numpy(vals.view(np.int64 if vals.dtype == np.uint64 else np.int32)).to(dev)
    wk, wv = tk.clone(), (tv.clone() if tv is not None else None)
    times, st = [], None
    for r in range(warm + reps):
        wk.copy_(tk)
        if tv is not None:
            wv.copy_(tv)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dfr.sort(wk, wv, **kw)
        b.record()
        torch.cuda.synchronize()
        if r >= warm:
            times.append(a.elapsed_time(b))
    st = dfr.sort(wk.copy_(tk), wv.copy_(tv) if tv is not None else None, stats=True, **kw)
    ok = verify(wk.cpu().numpy().view(keys.dtype), None if wv is None else wv.cpu().numpy().view(vals.dtype),
                keys, vals)
    ms = statistics.median(times)
    return {"ms": round(ms, 4), "gkeys_s": round(keys.size / ms / 1e6, 3), "verified": ok,
            "level0_p": st["level0_p"], "fused": st["fused"], "level0_large": st["level0_large"]}


def verify(out_k, out_v, in_k, in_v):
    import datagen
    ok = bool(datagen.is_sorted(out_k)) and datagen.fingerprint(out_k) == datagen.fingerprint(in_k)
    if ok and out_v is not None:
        # tags are distinct random draws: map each output tag back to its input position
        pos = np.argsort(in_v, kind="stable")
        where = pos[np.searchsorted(in_v[pos], out_v)]
        ok = bool((in_v[where] == out_v).all()) and bool((in_k[where] == out_k).all())
        eq = out_k[1:] == out_k[:-1]
        ok = ok and bool((where[1:][eq] > where[:-1][eq]).all())
    return bool(ok)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["paper", "nd"])
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    import datagen
    import paper_2207_14334_b200 as dfr
    rows = []

    def emit(row):
        rows.append(row)
        print(json.dumps(row), flush=True)

    if args.what == "paper":
        for case in ["paper-uniform", "paper-wide-normal", "paper-narrow-normal", "paper-records"]:
            for n in [1 << 24, 1 << 26, 1 << 28, 1 << 29, 1 << 30]:
                if case == "paper-records" and n > 1 << 28:
                    continue
                k, v = datagen.make_case(case, n)
                r = measure(dfr, torch, k, v, reps=args.reps)
                emit({"sweep": "paper", "case": case, "n": n, "log256_n": round(math.log(n, 256), 3), **r})
                del k, v
                torch.cuda.empty_cache()
    else:
        for case, n in [("c5-uniform", 1 << 28), ("c3-normal", 1 << 26), ("c3-zipf", 1 << 26)]:
            k, _ = datagen.make_case(case, n)
            for nd in [16, 32, 64, 128, 256]:
                emit({"sweep": "n_d", "case": case, "n": n, "n_d": nd, **measure(dfr, torch, k, n_d=nd, reps=args.reps)})
            emit({"sweep": "ablation", "case": case, "n": n, "variant": "separate last pass",
                  **measure(dfr, torch, k, fused=False, reps=args.reps)})
            emit({"sweep": "ablation", "case": case, "n": n, "variant": "no pass skipping",
                  **measure(dfr, torch, k, skip_trivial=False, reps=args.reps)})
            emit({"sweep": "ablation", "case": case, "n": n, "variant": "stable deals (stable_deals=1)",
                  **measure(dfr, torch, k, stable_deals=True, reps=args.reps)})
            if n >= 1 << 27:
                emit({"sweep": "ablation", "case": case, "n": n, "variant": "Fast Radix estimation",
                      **measure(dfr, torch, k, fast_radix=True, reps=args.reps)})
            del k
            torch.cuda.empty_cache()
        k = datagen.uniform_u32(1 << 27, 31)
        emit({"sweep": "ablation", "case": "u32 uniform", "n": 1 << 27, "variant": "DFR (default)",
              **measure(dfr, torch, k, reps=args.reps)})
        emit({"sweep": "ablation", "case": "u32 uniform", "n": 1 << 27, "variant": "full LSD (4 passes)",
              **measure(dfr, torch, k, full_lsd=True, reps=args.reps)})
        emit({"sweep": "ablation", "case": "u32 uniform", "n": 1 << 27, "variant": "Fast Radix estimation",
              **measure(dfr, torch, k, fast_radix=True, reps=args.reps)})
    if args.out:
        with open(args.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
