"""Look-back statistics of the fused pass (a -DDFR_LB_STATS build, DFR_LIB=...):
one 2^28 c5-uniform sort, then the device counters."""
import ctypes, numpy as np, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_2207_14334_b200 as dfr
k, _ = datagen.make_case("c5-uniform")
t = torch.from_numpy(k.view(np.int64)).cuda()
for _ in range(3):
    x = t.clone(); dfr.sort(x)
torch.cuda.synchronize()
out = (ctypes.c_uint64 * 4)()
dfr.lib().dfr_debug_lb_stats(out)
print("extra rounds", out[0], "sleeps", out[1], "look-backs", out[2], "extra rounds per look-back", out[0] / max(1, out[2]),
      "extra rounds per tile-digit", out[0] / max(1, out[2]) / 256)
