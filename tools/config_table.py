#!/usr/bin/env python
"""Per-config results of BASELINE.md §5 on one B200 (run through gpurun).

  python tools/config_table.py gpu  OUT.jsonl   for each of the 13 inputs of the
        five BASELINE configs: 10 timed sorts of pristine resident copies (CUDA
        events around the library call), median / mean / min ms and Gkeys/s;
        the oracle (plain single-threaded C++ DFR) on the same input, timed on
        this host (1 thread, scratch allocation inside); bit-exact comparison
        of the GPU output (keys, and values for pairs) with the oracle's
  python tools/config_table.py one  CASE        one sort of CASE (for an ncu launch list)
  python tools/config_table.py ncu  OUT.jsonl   per config, from gpurun_out/cfg_<case>.csv:
        DRAM bytes and device time summed over the sort's kernels
  python tools/config_table.py table IN.jsonl [NCU.jsonl]   the markdown table
"""
import csv
import json
import math
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = ["c1", "c2", "c3-normal", "c3-exp", "c3-zipf", "c4-few", "c4-equal", "c5-uniform",
         "c5-sorted", "c5-reverse", "c5-nearly", "c5-runs", "c5-low20"]


def to_dev(torch, a):
    return torch.from_numpy(a.view(np.int64 if a.dtype == np.uint64 else np.int32)).cuda()


def gpu(out_path):
    import torch
    import datagen
    import oracle
    import paper_2207_14334_b200 as dfr
    cpu = None
    try:
        cpu = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except Exception:
        pass
    with open(out_path, "w") as f:
        for name in CASES:
            c = datagen.CASES[name]
            k, v = datagen.make_case(name)
            tk, tv = to_dev(torch, k), (to_dev(torch, v) if v is not None else None)
            wk, wv = tk.clone(), (tv.clone() if tv is not None else None)
            times = []
            for r in range(13):
                wk.copy_(tk)
                if tv is not None:
                    wv.copy_(tv)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                dfr.sort(wk, wv)
                b.record()
                torch.cuda.synchronize()
                if r >= 3:
                    times.append(a.elapsed_time(b))
            gk = wk.cpu().numpy().view(k.dtype)
            gv = wv.cpu().numpy().view(v.dtype) if v is not None else None
            t0 = time.perf_counter()
            rk, rv, _ = oracle.dfr_sort(k, v)
            osec = time.perf_counter() - t0
            exact = bool((gk == rk).all()) and (v is None or bool((gv == rv).all()))
            med = statistics.median(times)
            row = {"case": name, "config": c.config, "n": c.n, "key": c.key_dtype, "pairs": c.pairs,
                   "gpu_ms_median": round(med, 4), "gpu_ms_mean": round(statistics.mean(times), 4),
                   "gpu_ms_min": round(min(times), 4), "gkeys_s": round(c.n / med / 1e6, 3),
                   "compulsory_bytes": 2 * c.n * (int(c.key_dtype[1:]) // 8 + (4 if c.pairs else 0)),
                   "oracle_s": round(osec, 3), "oracle_threads": 1, "host_cpu": cpu,
                   "host_cpus": os.cpu_count(), "bit_exact": exact}
            print(json.dumps(row), flush=True)
            f.write(json.dumps(row) + "\n")
            del tk, tv, wk, wv
            torch.cuda.empty_cache()


def one(name):
    import torch
    import datagen
    import paper_2207_14334_b200 as dfr
    k, v = datagen.make_case(name)
    tk, tv = to_dev(torch, k), (to_dev(torch, v) if v is not None else None)
    torch.cuda.synchronize()
    dfr.sort(tk, tv)
    torch.cuda.synchronize()


def ncu(out_path):
    with open(out_path, "w") as f:
        for name in CASES:
            p = os.path.join(ROOT, "gpurun_out", f"cfg_{name}.csv")
            if not os.path.exists(p):
                continue
            rows = list(csv.reader(open(p)))
            h = next((r for r in rows if r and r[0] == "ID"), None)
            if h is None:
                continue
            ix = {k: i for i, k in enumerate(h)}
            per = {}
            for r in rows[rows.index(h) + 1:]:
                if len(r) != len(h):
                    continue
                per.setdefault(r[ix["ID"]], {})[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
            by = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in per.values())
            ns = sum(x.get("gpu__time_duration.sum", 0) for x in per.values())
            row = {"case": name, "kernels": len(per), "dram_bytes": by, "kernel_ms": ns / 1e6,
                   "dram_GBps": by / ns if ns else None}
            print(json.dumps(row))
            f.write(json.dumps(row) + "\n")


def table(path, ncu_path=None):
    nc = {}
    if ncu_path and os.path.exists(ncu_path):
        nc = {json.loads(l)["case"]: json.loads(l) for l in open(ncu_path)}
    print("| Config | Input | GPU Gkeys/s (median of 10) | GPU ms (median / mean / min) | "
          "compulsory 2(k+v)n bytes at 8 TB/s | ncu DRAM GB/s | Oracle s (1 core) | Bit-exact |")
    print("|---|---|---|---|---|---|---|---|")
    for l in open(path):
        d = json.loads(l)
        frac = d["compulsory_bytes"] / (d["gpu_ms_median"] / 1e3) / 8e12
        g = nc.get(d["case"], {}).get("dram_GBps")
        print(f'| {d["config"]} | {d["case"]}: 2^{int(round(math.log2(d["n"])))} {d["key"]}'
              f'{" pairs" if d["pairs"] else ""} | {d["gkeys_s"]:.2f} | {d["gpu_ms_median"]:.3f} / '
              f'{d["gpu_ms_mean"]:.3f} / {d["gpu_ms_min"]:.3f} | {frac:.3f} | '
              f'{f"{g:.0f}" if g else "—"} | {d["oracle_s"]:.2f} | {"yes" if d["bit_exact"] else "NO"} |')


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "gpu":
        gpu(sys.argv[2])
    elif cmd == "one":
        one(sys.argv[2])
    elif cmd == "ncu":
        ncu(sys.argv[2])
    else:
        table(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
