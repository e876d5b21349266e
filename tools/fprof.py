"""Phase profile of the fused pass (a -DDFR_FPROF build, DFR_LIB=...): three
2^28 c5-uniform sorts, then the per-phase SM-cycle sums of thread 0 of every CTA."""
import ctypes, numpy as np, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_2207_14334_b200 as dfr
k, _ = datagen.make_case(sys.argv[1] if len(sys.argv) > 1 else "c5-uniform")
t = torch.from_numpy(k.view(np.int64)).cuda()
for _ in range(3):
    x = t.clone(); dfr.sort(x)
torch.cuda.synchronize()
out = (ctypes.c_uint64 * 16)()
dfr.lib().dfr_debug_fprof(out)
names = ["tail(prev)", "layout", "comp stores+lb issue", "rank", "lookback+claim+load", "write+count", "zero"]
tot = sum(out[i] for i in range(7))
for i, n in enumerate(names):
    print(f"{n:16s} {out[i] / tot * 100:5.1f}%  cycles/tile {out[i] / max(1, out[8]):8.0f}")
print("tiles", out[8], "tiles with ties", out[9], f"({out[9] / max(1, out[8]) * 100:.1f}%)")
