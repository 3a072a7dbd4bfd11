"""Per-net window hash (DESIGN.md §5 definition, restricted to lo <= t <= hi) of a
waveform CSR, vectorised over nets with numpy — the host side of the full-size
parity checks.  Test infrastructure; pinned against the oracle's own per-net
hashes and a per-net loop by tests/test_winhash.py."""
import numpy as np

_C = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(x):
    x = x + _C
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def window_hash(offsets, trans, lo, hi):
    """h = splitmix64(C ^ n), then h = splitmix64(h ^ e) over the net's n entries e with
    lo <= time(e) <= hi, in order — for every net at once (one numpy pass per rank)."""
    offsets = np.asarray(offsets, np.int64)
    trans = np.asarray(trans).view(np.uint64)
    n = len(offsets) - 1
    net = np.repeat(np.arange(n, dtype=np.int64), np.diff(offsets))
    t = (trans >> np.uint64(2)).astype(np.int64)
    keep = (t >= lo) & (t <= hi)
    e, net = trans[keep], net[keep]
    cnt = np.bincount(net, minlength=n).astype(np.int64)
    with np.errstate(over="ignore"):
        h = splitmix64(_C ^ cnt.astype(np.uint64))
        if e.size == 0:
            return h
        start = np.zeros(n, np.int64)
        start[1:] = np.cumsum(cnt)[:-1]
        rank = np.arange(e.size, dtype=np.int64) - start[net]   # position inside the net's window
        order = np.argsort(rank, kind="stable")
        bounds = np.searchsorted(rank[order], np.arange(int(rank.max()) + 2))
        for j in range(len(bounds) - 1):
            idx = order[bounds[j]:bounds[j + 1]]
            nn = net[idx]                                       # distinct nets
            h[nn] = splitmix64(h[nn] ^ e[idx])
    return h
