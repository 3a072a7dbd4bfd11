"""Per-net window checksum (DESIGN.md §5 definition, restricted to lo <= t <= hi) of a
waveform CSR, vectorised over nets with numpy — the host side of the full-size
parity checks.  Test infrastructure; pinned against the oracle's own per-net
hashes and a per-net loop by tests/test_winhash.py."""
import numpy as np

_C = np.uint64(0x9E3779B97F4A7C15)
_K = np.uint64(0xD1B54A32D192ED03)


def splitmix64(x):
    x = x + _C
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def window_hash(offsets, trans, lo, hi):
    """h = splitmix64(C ^ n) XOR (XOR over j of splitmix64(e_j + (j + 1) * K)) over the net's n
    entries e_j with lo <= time(e_j) <= hi, j their position inside the window — for every
    net at once."""
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
        pos = (np.arange(e.size, dtype=np.int64) - start[net] + 1).astype(np.uint64)
        term = splitmix64(e + pos * _K)
        nz = np.flatnonzero(cnt)
        h[nz] ^= np.bitwise_xor.reduceat(term, start[nz])
    return h


def window_terms(offsets, trans, lo, hi, base=None, total=None):
    """Per-net stitching pieces (include/gls.h gls_get_net_hash_terms_device) for the
    entries with lo <= time <= hi: (counts, terms), terms keyed from base[n] + j and
    with the length term of total[n] XORed in when total is given."""
    offsets = np.asarray(offsets, np.int64)
    trans = np.asarray(trans).view(np.uint64)
    n = len(offsets) - 1
    net = np.repeat(np.arange(n, dtype=np.int64), np.diff(offsets))
    t = (trans >> np.uint64(2)).astype(np.int64)
    keep = (t >= lo) & (t <= hi)
    e, net = trans[keep], net[keep]
    cnt = np.bincount(net, minlength=n).astype(np.int64)
    base = np.zeros(n, np.int64) if base is None else np.asarray(base, np.int64)
    with np.errstate(over="ignore"):
        h = np.zeros(n, np.uint64) if total is None else splitmix64(_C ^ np.asarray(total).astype(np.uint64))
        if e.size:
            start = np.zeros(n, np.int64)
            start[1:] = np.cumsum(cnt)[:-1]
            pos = (np.arange(e.size, dtype=np.int64) - start[net] + base[net] + 1).astype(np.uint64)
            term = splitmix64(e + pos * _K)
            nz = np.flatnonzero(cnt)
            h[nz] ^= np.bitwise_xor.reduceat(term, start[nz])
    return cnt, h
