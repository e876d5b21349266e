"""Context only (not a target): torch.sort (CUB radix sort) on the same 2^28
uint64 input, timed with CUDA events, next to one dfr sort."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen, paper_2207_14334_b200 as dfr
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
k, _ = datagen.make_case("c5-uniform", n)
# torch has no uint64 sort; flipping the sign bit maps uint64 order onto int64 order
flipped = torch.from_numpy((k ^ np.uint64(1 << 63)).view(np.int64)).cuda()
raw = torch.from_numpy(k.view(np.int64)).cuda()
def t_ms(fn, reps=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
ts = t_ms(lambda: torch.sort(flipped))
bufs = [raw.clone() for _ in range(7)]
it = iter(bufs)
td = t_ms(lambda: dfr.sort(next(it)))
print(f"n={n} torch.sort(int64) {ts:.3f} ms ({n/ts/1e6:.1f} Gkeys/s) ; dfr_sort_u64 {td:.3f} ms ({n/td/1e6:.1f} Gkeys/s)")
