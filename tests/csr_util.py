"""Host helpers for the results-stitching tests (test infrastructure): a numpy segment
scatter with the semantics of gls_scatter_segments, and a window slice of a CSR."""
import numpy as np
import torch


def numpy_scatter(nseg, src_off, src, dst_off, dst):
    """dst[dst_off[i] + k] = src[src_off[i] + k] for k < src_off[i+1] - src_off[i] (torch CPU tensors)."""
    so, do = src_off.numpy(), dst_off.numpy()
    s, d = src.numpy(), dst.numpy()
    for i in range(nseg):
        a, b = so[i], so[i + 1]
        d[do[i]:do[i] + (b - a)] = s[a:b]


def window_csr(offsets, trans, lo, hi):
    """(counts [nets], transitions) of the entries with lo <= t <= hi, in net order."""
    offsets = np.asarray(offsets, np.int64)
    trans = np.asarray(trans).view(np.uint64)
    n = len(offsets) - 1
    net = np.repeat(np.arange(n, dtype=np.int64), np.diff(offsets))
    t = (trans >> np.uint64(2)).astype(np.int64)
    keep = (t >= lo) & (t <= hi)
    return np.bincount(net[keep], minlength=n).astype(np.int64), trans[keep].copy()


def cpu_alloc(k):
    return torch.zeros(max(1, k), dtype=torch.int64)
