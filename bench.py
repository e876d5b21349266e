#!/usr/bin/env python
"""bench.py — headline benchmark of the B200 DFR sort (BASELINE.json metric:
"Gkeys/s sorting 2^28 uint64 keys on 1 B200; % of HBM roofline").

One step = one complete DFR sort (every hot-path row of SURVEY §8(a): plan,
histogram, p stable deals, diversion scan + small-bucket sort, recursion,
on-chip mid buckets) of 2^28 i.i.d. uniform uint64 keys (config c5-uniform,
SplitMix64 seed 5) already resident in HBM.  Each timed step sorts its own
pristine resident copy (2 GiB > 126 MB L2, so no step sees a warm L2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dfr|reference]

N > 1 (torchrun): independent replicas, one per GPU (the path does
not shard; no data-path collective), timed on the device, max over ranks.
--impl reference: the CPU oracle (oracle/, the only other place bench.py runs
it) on a bounded sample of the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gkeys/s sorting 2^28 uint64 keys on 1 B200; % of HBM roofline"
UNIT = "Gkeys/s"
# algorithmic bytes per key: one histogram
# read (8) + p=3 stable deals x (read 8 + write 8) + diversion read+write (16)
SORT_BYTES_PER_KEY_U64 = 72
PASS_BYTES_PER_KEY_U64 = 16  # one stable deal of a u64 key: read 8 + write 8
NOMINAL_HBM_GBS = 8000.0
FALLBACK_HBM_GBS = 6650.0

THROTTLE_BITS = {0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
                 0x80: "hw_power_brake_slowdown", 0x4: "sw_power_cap", 0x2: "applications_clocks",
                 0x1: "gpu_idle", 0x10: "sync_boost", 0x100: "display_clock"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="dfr", choices=["dfr", "reference"])
    ap.add_argument("--case", default="c5-uniform", help="datagen case (default: the headline)")
    ap.add_argument("--n", type=int, default=None, help="override the case size")
    ap.add_argument("--quick", action="store_true", help="skip e2e and cpu_baseline (for ncu runs)")
    ap.add_argument("--fused", default="auto", choices=["auto", "off"],
                    help="auto (default): the fused last deal + diversion where eligible; "
                         "off: dfr_config.fused_last_pass = 2 (separate kernels)")
    ap.add_argument("--phase-events", default="none", choices=["all", "deal", "none"],
                    help="phases timed with CUDA events inside the HEADLINE timed region (events "
                         "between kernels stop programmatic dependent launch from overlapping "
                         "them); the per-phase times always come from a separate run of K steps")
    ap.add_argument("--stable-deals", action="store_true",
                    help="dfr_config.stable_deals = 1 (every deal the stable ballot multi-split)")
    ap.add_argument("--no-cold", action="store_true", help="skip the cold-pool trial")
    ap.add_argument("--fast-radix", action="store_true",
                    help="dfr_config.fast_radix = 1 (Fast Radix estimation of the first group pass)")
    ap.add_argument("--out", default=None, help="also append the JSON line to this file")
    return ap.parse_args()


def peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Polls NVML every ~2 ms on a thread while the timed region runs."""

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= int(get_r(self.h))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        reasons = [name for bit, name in THROTTLE_BITS.items() if self.reasons & bit]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


def reduce_max_ms(ms, world, device="cpu"):
    """Timing of a multi-rank run: the MAX of the ranks' device-measured times
    (all ranks get it).  world == 1: unchanged."""
    if world == 1:
        return ms
    import torch
    import torch.distributed as dist
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_value(n, world, steps, ms):
    """Whole-job throughput in Gkeys/s: every rank sorts its own n keys per step
    (replicas, weak scaling), all ranks together in the max-over-ranks time."""
    return world * n * steps / (ms / 1e3) / 1e9


def workload(case, n):
    import datagen
    c = datagen.CASES[case]
    n = c.n if n is None else n
    desc = {
        "c5-uniform": "2^28 uint64 keys i.i.d. uniform over [0, 2^64) (SplitMix64 seed 5)",
    }.get(case, f"{case} recipe (datagen.make_case)")
    if n != c.n:
        desc += f", n={n}"
    return c, n, desc


def config_dict(case, n, c, desc, n_d=64):
    return {"workload": f"{case}: {desc}", "n": n, "key": c.key_dtype,
            "pairs": c.pairs, "n_d": n_d, "radix_bits": 8,
            "l2": "inputs larger than L2 (2 GiB/step vs 126 MB); each step sorts its own "
                  "pristine resident copy",
            "parallelism": "replicas (one independent sort per GPU)"}


# ---------------------------------------------------------------- reference
def run_reference(args, rank, world):
    """The CPU oracle (plain single-threaded DFR) on a bounded sample per step."""
    if rank != 0:
        return
    import datagen
    import oracle
    c, n, desc = workload(args.case, args.n)
    # the whole configured workload per step (about 8 s per 2^28-key sort on
    # one core) unless the run asks for so many steps that it would take more
    # than a few minutes: then the first 2^26 keys of the same input
    sample = n if args.steps + args.warmup <= 30 else min(n, 1 << 26)
    keys, vals = datagen.make_case(args.case, n)
    keys = keys[:sample].copy()
    vals = vals[:sample].copy() if vals is not None else None
    for _ in range(args.warmup):
        oracle.dfr_sort(keys, vals)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.dfr_sort(keys, vals)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = sample * args.steps / total / 1e9
    samp = (f"the whole {args.case} input ({n} keys)" if sample == n else
            f"first {sample} of the {n} keys of the {args.case} input") + \
        " per step, oracle.dfr_sort (1 thread, scratch allocation inside the timing)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": c.key_dtype, "data": "synthetic",
            "config": config_dict(args.case, n, c, desc),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": samp, "sample_n": sample, "cpu_model": cpu_model(),
                             "host_cpus": os.cpu_count()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line, args)


def emit(line, args):
    s = json.dumps(line)
    print(s, flush=True)
    if args.out:
        with open(args.out, "a") as f:
            f.write(s + "\n")


# ---------------------------------------------------------------- our arm
def run_dfr(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import datagen
    import paper_2207_14334_b200 as dfr

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    c, n, desc = workload(args.case, args.n)
    keys_h, vals_h = datagen.make_case(args.case, n)
    kdt = np.uint64 if c.key_dtype == "u64" else np.uint32
    tdt = torch.int64 if c.key_dtype == "u64" else torch.int32
    kb = np.dtype(kdt).itemsize
    vb = 4 if c.pairs else 0
    fp_in = datagen.fingerprint(keys_h)

    pristine = torch.from_numpy(keys_h.view(np.int64 if kb == 8 else np.int32)).to(dev)
    pristine_v = torch.from_numpy(vals_h.view(np.int32)).to(dev) if c.pairs else None
    K, W = args.steps, args.warmup
    free = torch.cuda.mem_get_info(dev)[0]
    per = n * (kb + vb)
    ws = dfr.workspace_bytes(n, kb, vb)
    nbuf = int(min(K + W, max(2, (free - 3 * per - ws - (4 << 30)) // per)))
    bufs = [pristine.clone() for _ in range(nbuf)]
    vbufs = [pristine_v.clone() for _ in range(nbuf)] if c.pairs else [None] * nbuf
    restore = nbuf < K + W  # not enough HBM for a copy per step: restore between steps
    stream = torch.cuda.current_stream()
    nph = len(dfr.PHASES)

    def make_events(which):
        timed = [which == "all" or (which == "deal" and name.startswith("scatter"))
                 for name in dfr.PHASES]
        evs = [[torch.cuda.Event(enable_timing=True) if timed[e // 2] else None
                for e in range(2 * nph)] for _ in range(K)]
        for row in evs:  # torch creates the CUDA event lazily, on its first record
            for e in row:
                if e is not None:
                    e.record(stream)
        return timed, evs

    head_timed, head_evs = make_events(args.phase_events)

    def sort_step(i, ev=None):
        b = bufs[i % nbuf]
        vbuf = vbufs[i % nbuf]
        kw = {"fast_radix": True} if args.fast_radix else {}
        if args.stable_deals:
            kw["stable_deals"] = True
        dfr.sort(b, vbuf, events=ev, fused=None if args.fused == "auto" else False, **kw)

    def restore_buf(i):
        bufs[i % nbuf].copy_(pristine)
        if c.pairs:
            vbufs[i % nbuf].copy_(pristine_v)

    for i in range(W):
        if restore:
            restore_buf(i)
        sort_step(i)
    torch.cuda.synchronize()

    # ---- timed region: exactly K steps (no phase events unless asked for)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_ms = []
    l0 = dfr.launch_counter()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        if not restore:
            start.record(stream)
            for i in range(K):
                sort_step(W + i, head_evs[i] if args.phase_events != "none" else None)
            stop.record(stream)
            torch.cuda.synchronize()
            elapsed = start.elapsed_time(stop)
        else:  # per-step events; the restore copy is outside each step's events
            for i in range(K):
                restore_buf(W + i)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                sort_step(W + i, head_evs[i] if args.phase_events != "none" else None)
                b.record(stream)
                torch.cuda.synchronize()
                step_ms.append(a.elapsed_time(b))
            elapsed = sum(step_ms)
    launches = dfr.launch_counter() - l0
    if world > 1:
        dist.barrier()
    elapsed = reduce_max_ms(elapsed, world, dev)
    last = bufs[(W + K - 1) % nbuf]
    last_v = vbufs[(W + K - 1) % nbuf]
    out_h = last.cpu().numpy().view(kdt)
    out_v = last_v.cpu().numpy().view(np.uint32) if c.pairs else None
    verified = verify_output(out_h, out_v, keys_h, vals_h, fp_in)
    del out_h, out_v

    # ---- per-phase device times: a separate run of K steps with CUDA events the
    # library records on this stream around each phase (the events stop
    # programmatic dependent launch from overlapping the kernels, so this run
    # is a little slower than the headline; its phases explain the headline)
    ph_timed, ph_evs = make_events("all")
    ph_step = []
    for i in range(K):
        restore_buf(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sort_step(i, ph_evs[i])
        b.record(stream)
        ph_step.append((a, b))
    torch.cuda.synchronize()
    phase_ms = {}
    for p, name in enumerate(dfr.PHASES):
        phase_ms[name] = statistics.mean(ph_evs[i][2 * p].elapsed_time(ph_evs[i][2 * p + 1])
                                         for i in range(K))
    phase_run_ms = statistics.mean(a.elapsed_time(b) for a, b in ph_step)

    # ---- one cold-pool trial: the stream-ordered pool trimmed to zero first, so
    # the call's cudaMallocAsync maps fresh memory (P:332 times allocation)
    cold_ms = None
    if not args.no_cold:
        restore_buf(0)
        torch.cuda.synchronize()
        if trim_default_pool(local_rank):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            sort_step(0)
            b.record(stream)
            torch.cuda.synchronize()
            cold_ms = a.elapsed_time(b)

    value = job_value(n, world, K, elapsed)
    ms_per_step = elapsed / K
    peak, peak_src = peak_hbm()

    # roofline of the dominant kernel: the phase with the largest
    # device time per sort; its algorithmic bytes per launch = its per-key bytes
    # x n.  Phases (dfr.h DFR_PHASE_*): hist = one read of the keys (kb); a deal
    # (scatter0/1, and scatter2 = the fused last deal + diversion on the fused
    # path, or the plain last deal) reads and writes each record (2(kb+vb));
    # divert = read + write of the records it sorts (2(kb+vb)).
    per_key = {"hist": kb, "scatter0": 2 * (kb + vb), "scatter1": 2 * (kb + vb),
               "scatter2": 2 * (kb + vb), "scatter3": 2 * (kb + vb), "divert": 2 * (kb + vb)}
    cand = {k: v for k, v in phase_ms.items() if k in per_key and v > 0.05}
    dominant = max(cand, key=lambda k: cand[k]) if cand else None
    fused_path = phase_ms.get("divert", 0.0) < 0.05 and phase_ms.get("scatter2", 0.0) > 0.05
    kname = {"hist": "k_hist (one read: the group digits' histograms)",
             "scatter0": "k_scatter (stable deal, lowest group digit)",
             "scatter1": "k_scatter_fh (stable deal, middle digit + joint histogram)",
             "scatter2": ("k_fused (last deal + diversion of its small buckets, one kernel)"
                          if fused_path else "k_scatter (stable deal, top group digit)"),
             "divert": "k_divert (scan for large buckets + small-bucket sort)"}.get(dominant, dominant)
    dom_ms = cand.get(dominant)
    dom_bytes = n * per_key[dominant] if dominant else None
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9 if dom_ms else None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        traffic = tj.get(f"{args.case}:{n}:{'k_fused' if dominant == 'scatter2' and fused_path else 'k_scatter'}")
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak if achieved else None, "traffic": traffic,
                "algorithmic_bytes_per_launch": dom_bytes, "avg_launch_ms": dom_ms,
                "peak_source": peak_src,
                "timing": "CUDA events the library records around each phase on the sort's stream, "
                          "in a separate run of K steps (phase_ms)"}
    # the whole sort against the bytes the executed path moves (fused path:
    # 8 histogram + 3 x 16 deals = 56 B/key for u64 keys; plain path: + 16 of
    # the diversion = 72, SURVEY §8(d)'s plan)
    sort_roof = None
    if not c.pairs:
        bpk = kb + 3 * 2 * kb + (0 if fused_path else 2 * kb)
        gbs = n * bpk / (ms_per_step / 1e3) / 1e9
        sort_roof = {"bytes_per_key": bpk, "achieved_GBps": gbs, "frac_of_measured_copy": gbs / peak,
                     "frac_of_8TBps": gbs / NOMINAL_HBM_GBS,
                     "survey_plan_72B_equiv_frac_of_8TBps": n * 9 * kb / (ms_per_step / 1e3) / 1e9 / NOMINAL_HBM_GBS}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": c.key_dtype, "data": "synthetic",
            "config": config_dict(args.case, n, c, desc), "verified": verified,
            "roofline": roofline, "sort_roofline": sort_roof,
            "phase_ms": {k: round(v, 4) for k, v in phase_ms.items()},
            "phase_run_ms_per_step": round(phase_run_ms, 4),
            "cold_pool_ms": round(cold_ms, 4) if cold_ms is not None else None,
            "headline_phase_events": args.phase_events,
            "gpu_launches": int(launches), "clocks": clk.summary()}

    if not args.quick:
        line["e2e"] = run_e2e(args, dfr, torch, dev, keys_h, vals_h, tdt, n, kb, vb, world)
        if rank == 0 and world == 1:
            line["cpu_baseline"] = run_cpu_baseline(args, keys_h, vals_h)
    if rank == 0:
        emit(line, args)


def run_e2e(args, dfr, torch, dev, keys_h, vals_h, tdt, n, kb, vb, world):
    """Same metric through the public API with HOST buffers: every step copies
    its input from pinned host memory (H2D), sorts it and reads the sorted
    result back (D2H), all inside the timing.  Steps are pipelined the way a
    serving loop would run them: the H2D of step i+1 and the D2H of step i-1
    (separate copy streams, PCIe is full duplex) overlap the sort of step i;
    NBUF device buffers rotate, a buffer is refilled only after its D2H."""
    import torch.distributed as dist
    hk = torch.from_numpy(keys_h.view(np.int64 if kb == 8 else np.int32)).pin_memory()
    ho = torch.empty_like(hk).pin_memory()
    hv = torch.from_numpy(vals_h.view(np.int32)).pin_memory() if vals_h is not None else None
    hvo = torch.empty_like(hv).pin_memory() if hv is not None else None
    NBUF = 3
    dks = [torch.empty(n, dtype=tdt, device=dev) for _ in range(NBUF)]
    dvs = [torch.empty(n, dtype=torch.int32, device=dev) if hv is not None else None
           for _ in range(NBUF)]
    s_h2d, s_sort, s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    freed = [None] * NBUF  # event: the buffer's last D2H is done

    def step(i):
        b = i % NBUF
        dk, dv = dks[b], dvs[b]
        e_in, e_out, e_free = (torch.cuda.Event() for _ in range(3))
        with torch.cuda.stream(s_h2d):
            if freed[b] is not None:
                s_h2d.wait_event(freed[b])
            dk.copy_(hk, non_blocking=True)
            if dv is not None:
                dv.copy_(hv, non_blocking=True)
            e_in.record(s_h2d)
        with torch.cuda.stream(s_sort):
            s_sort.wait_event(e_in)
            dfr.sort(dk, dv, stream=s_sort)
            e_out.record(s_sort)
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(e_out)
            ho.copy_(dk, non_blocking=True)
            if dv is not None:
                hvo.copy_(dv, non_blocking=True)
            e_free.record(s_d2h)
        freed[b] = e_free

    for i in range(min(args.warmup, 3)):
        step(i)
    torch.cuda.synchronize()
    K = args.steps
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    a.record(s_h2d)
    for i in range(K):
        step(i)
    b.record(s_d2h)
    torch.cuda.synchronize()
    ms = reduce_max_ms(a.elapsed_time(b), world, dev)
    ok = verify_output(ho.numpy().view(keys_h.dtype),
                       hvo.numpy().view(np.uint32) if hvo is not None else None,
                       keys_h, vals_h, datagen_fingerprint(keys_h))
    return {"value": job_value(n, world, K, ms), "unit": UNIT,
            "h2d_bytes_per_step": n * (kb + vb), "d2h_bytes_per_step": n * (kb + vb),
            "ms_per_step": ms / K, "pipelined_steps": NBUF, "verified": ok}


def datagen_fingerprint(a):
    import datagen
    return datagen.fingerprint(a)


def verify_output(out_k, out_v, in_k, in_v, fp_in):
    """The output is THE stable sort of the input: keys
    non-decreasing with the input's multiset (two independent 64-bit hash-sum
    fingerprints + count); pairs (values = input index, c4): the O(n)
    certificate -- values a permutation of 0..n-1, out_key[i] == in_key[out_val[i]],
    values strictly increasing inside runs of equal keys (stability)."""
    import datagen
    ok = bool(datagen.is_sorted(out_k)) and datagen.fingerprint(out_k) == fp_in
    if ok and out_v is not None:
        n = out_k.size
        ok = (np.array_equal(in_v, np.arange(n, dtype=in_v.dtype))
              and bool((np.bincount(out_v, minlength=n) == 1).all())
              and bool((in_k[out_v] == out_k).all()))
        eq = out_k[1:] == out_k[:-1]
        ok = ok and bool((out_v[1:][eq] > out_v[:-1][eq]).all())
    return bool(ok)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_cpu_baseline(args, keys_h, vals_h):
    """The oracle as it stands (1 thread, never tuned) on the FULL workload."""
    import oracle
    n = keys_h.size
    t0 = time.perf_counter()
    oracle.dfr_sort(keys_h, vals_h)  # sorts a copy; scratch allocation inside the timing
    dt = time.perf_counter() - t0
    return {"value": n / dt / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"the whole {args.case} input ({n} keys), one oracle.dfr_sort call "
                      f"(1 thread, scratch allocation inside the timing), {dt:.1f} s",
            "host_cpus": os.cpu_count(), "cpu_model": cpu_model()}


def trim_default_pool(device):
    """cudaMemPoolTrimTo(default pool of `device`, 0) through the CUDA runtime
    torch loads (the library keeps freed scratch mapped by raising the pool's
    release threshold; trimming makes the next call map it afresh)."""
    import ctypes
    import glob
    import torch
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart.so*"))
    cands += glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime",
                                    "lib", "libcudart.so*"))
    cands += ["libcudart.so.12", "libcudart.so"]
    for name in cands:
        try:
            rt = ctypes.CDLL(name)
            pool = ctypes.c_void_p()
            if rt.cudaDeviceGetDefaultMemPool(ctypes.byref(pool), int(device)) != 0:
                continue
            return rt.cudaMemPoolTrimTo(pool, ctypes.c_size_t(0)) == 0
        except OSError:
            continue
    return False


def self_launch(args):
    """`python bench.py --gpus N` without a torchrun environment: re-exec this
    script under torch.distributed.run with N ranks on this node (127.0.0.1),
    so that a plain invocation measures N replicas as the driver's does."""
    import socket
    import subprocess
    n = args.gpus
    try:
        import torch
        have = torch.cuda.device_count()
        if args.impl == "dfr" and have and have < n:
            print(f"bench.py: --gpus {n} but only {have} CUDA devices; running {have}",
                  file=sys.stderr)
            n = have
    except Exception:
        pass
    if n <= 1:
        return None
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    argv = [a for a in sys.argv[1:]]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + argv
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        rc = self_launch(args)
        if rc is not None:
            sys.exit(rc)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "dfr":
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_dfr(args, rank, world, local_rank)
    if world > 1 and args.impl == "dfr":
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
