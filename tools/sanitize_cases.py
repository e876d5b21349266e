"""Small sorts for compute-sanitizer runs: every export on a few sizes (tiny,
ragged, several tiles, the cooperative path), checked against numpy."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen
import paper_2207_14334_b200 as dfr

def dev(a):
    return torch.from_numpy(a.view(np.int64 if a.dtype == np.uint64 else np.int32)).cuda()

sizes = [int(x) for x in (sys.argv[1:] or ["1000", "70000", "1100000"])]
for n in sizes:
    k64 = datagen.uniform_u64(n, 11)
    t = dev(k64); dfr.sort(t); torch.cuda.synchronize()
    assert (t.cpu().numpy().view(np.uint64) == np.sort(k64)).all(), ("u64", n)
    k32 = datagen.uniform_u32(n, 12)
    t = dev(k32); dfr.sort(t); torch.cuda.synchronize()
    assert (t.cpu().numpy().view(np.uint32) == np.sort(k32)).all(), ("u32", n)
    v = np.arange(n, dtype=np.uint32)
    kk = (k32 & np.uint32(0xff)).copy()
    tk, tv = dev(kk), dev(v); dfr.sort(tk, tv); torch.cuda.synchronize()
    o = np.argsort(kk, kind="stable")
    assert (tv.cpu().numpy().view(np.uint32) == o).all(), ("pairs_u32", n)
    vv = datagen.uniform_u64(n, 13)
    tk, tv = dev(k64.copy()), dev(vv); dfr.sort(tk, tv); torch.cuda.synchronize()
    o = np.argsort(k64, kind="stable")
    assert (tv.cpu().numpy().view(np.uint64) == vv[o]).all(), ("pairs_u64", n)
    print("ok", n, flush=True)
