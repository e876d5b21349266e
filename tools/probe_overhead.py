"""Per-call GPU time vs the sum of phase times, and host enqueue time."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen, paper_2207_14334_b200 as dfr
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
k, _ = datagen.make_case("c5-uniform", n)
base = torch.from_numpy(k.view(np.int64)).cuda()
bufs = [base.clone() for _ in range(8)]
s = torch.cuda.current_stream()
for b in bufs[:2]:
    dfr.sort(b)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(6)]
t0 = time.perf_counter()
for i in range(6):
    ev[i][0].record(s); dfr.sort(bufs[2 + i]); ev[i][1].record(s)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print("host enqueue ms/call", (t1 - t0) / 6 * 1e3, "wall ms/call", (t2 - t0) / 6 * 1e3)
print("gpu ms per call", [round(a.elapsed_time(b), 3) for a, b in ev])
print("gaps ms", [round(ev[i][1].elapsed_time(ev[i + 1][0]), 3) for i in range(5)])
