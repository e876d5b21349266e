"""Helpers shared by the GPU tests: numpy <-> CUDA tensors of raw key bits."""
import numpy as np


def to_dev(a: np.ndarray):
    import torch
    if a.dtype == np.uint64:
        t = torch.from_numpy(a.view(np.int64))
    elif a.dtype == np.uint32:
        t = torch.from_numpy(a.view(np.int32))
    else:
        raise TypeError(a.dtype)
    return t.to("cuda")


def to_host(t, dtype) -> np.ndarray:
    return t.cpu().numpy().view(dtype)


def gpu_sort(keys: np.ndarray, vals: np.ndarray | None = None, **kw):
    import torch
    import paper_2207_14334_b200 as dfr
    k = to_dev(keys)
    v = to_dev(vals) if vals is not None else None
    st = dfr.sort(k, v, **kw)
    torch.cuda.synchronize()
    return to_host(k, keys.dtype), (to_host(v, vals.dtype) if v is not None else None), st
