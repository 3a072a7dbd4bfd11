"""Multi-GPU partitioning of the simulation — host-side logic only.

Time windows: rank r of N owns clock cycles [r*C/N, (r+1)*C/N) and output times
[k_lo*PERIOD, k_hi*PERIOD) (the last rank up to the duration).  Its given
waveforms start `lookback_cycles(H)` cycles earlier, clamped there (reading R17),
so every net is exact on the owned window.  No exchange happens during the
simulation; results and timings are combined afterwards with all_gather.

Stitching (`stitch_hashes`): the per-net checksum of the whole run is
an XOR of position-keyed terms plus a length term, so it splits over time windows:
every rank counts its owned transitions per net, the counts are all-gathered (NCCL
over NVLink on the GPU box), each rank keys its terms from the exclusive prefix of
the counts over the ranks before it, rank 0 adds the length term, and the XOR of the
all-gathered terms is the full-run checksum of every net — 16 bytes per net and rank
on the wire instead of the transitions themselves.
"""
from __future__ import annotations

import math

import torch

from . import workloads as W


def time_window(rank: int, world: int, ncycles: int):
    """(k_lo, k_hi) cycles owned by `rank`."""
    return rank * ncycles // world, (rank + 1) * ncycles // world


def lookback_cycles(halo_ps: int) -> int:
    """Cycles of given waveforms to simulate before the owned window: the clamp
    time (k_lo - look) * PERIOD must be <= k_lo * PERIOD - halo."""
    return math.ceil(halo_ps / W.PERIOD) + 1


def rank_plan(rank: int, world: int, ncycles: int, halo_ps: int, duration: int):
    """Everything a rank needs: generated cycles, simulated duration, owned output window."""
    k_lo, k_hi = time_window(rank, world, ncycles)
    look = 0 if k_lo == 0 else lookback_cycles(halo_ps)
    sim_dur = duration if rank == world - 1 else k_hi * W.PERIOD
    own_lo = k_lo * W.PERIOD
    own_hi = duration if rank == world - 1 else k_hi * W.PERIOD - 1
    return {"gen_cycles": (max(0, k_lo - look), k_hi), "duration": sim_dur, "own": (own_lo, own_hi)}


def _host_staged(group=None) -> bool:
    """gloo moves CPU tensors only: device tensors are staged through host memory (used by
    the functional multi-rank runs on one GPU; NCCL, the product backend, takes them as they
    are)."""
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def all_gather_t(out, t, group=None):
    """dist.all_gather into the list `out` (tensors like t), any device."""
    import torch.distributed as dist
    if _host_staged(group) and t.is_cuda:
        oc = [torch.empty(o.shape, dtype=o.dtype) for o in out]
        dist.all_gather(oc, t.cpu(), group=group)
        for o, c in zip(out, oc):
            o.copy_(c)
    else:
        dist.all_gather(out, t, group=group)


def send_t(t, dst, group=None):
    import torch.distributed as dist
    dist.send(t.cpu() if _host_staged(group) and t.is_cuda else t, dst, group=group)


def recv_t(t, src, group=None):
    import torch.distributed as dist
    if _host_staged(group) and t.is_cuda:
        c = torch.empty(t.shape, dtype=t.dtype)
        dist.recv(c, src, group=group)
        t.copy_(c)
    else:
        dist.recv(t, src, group=group)


def all_gather_rows(values, device, group=None):
    """all_gather a small float64 vector from every rank -> [world, len] CPU tensor."""
    import torch.distributed as dist
    t = torch.as_tensor(values, dtype=torch.float64, device=device)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size(group))]
    all_gather_t(out, t, group=group)
    return torch.stack(out).cpu()


def stitch_hashes(counts, terms_fn, group=None):
    """Full-run per-net checksums from per-rank windows.

    counts: this rank's per-net counts of owned transitions (int64 tensor [nets]);
    terms_fn(base, total) -> this rank's per-net terms (int64 tensor holding the uint64
    bits), keyed from `base` (transitions of the net owned by lower ranks) and with the
    length term of `total` XORed in when `total` is not None (rank 0 only).
    Returns the stitched checksums (int64 tensor, uint64 bits) on every rank."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    allc = [torch.empty_like(counts) for _ in range(world)]
    all_gather_t(allc, counts, group=group)
    allc = torch.stack(allc)
    base = allc[:rank].sum(0) if rank > 0 else torch.zeros_like(counts)
    total = allc.sum(0) if rank == 0 else None
    terms = terms_fn(base, total)
    allt = [torch.empty_like(terms) for _ in range(world)]
    all_gather_t(allt, terms, group=group)
    h = allt[0].clone()
    for t in allt[1:]:
        h.bitwise_xor_(t)
    return h


def gls_window_stitch(ctx, own_lo, own_hi, device, group=None):
    """stitch_hashes for a gls context holding this rank's window run (device arrays)."""
    n = ctx.num_inputs + ctx.num_gates
    counts = torch.empty(n, dtype=torch.int64, device=device)
    ctx.gls_get_net_hash_terms_device(own_lo, own_hi, 0, 0, counts.data_ptr(), 0)

    def terms_fn(base, total):
        terms = torch.empty(n, dtype=torch.int64, device=device)
        scratch = torch.empty(n, dtype=torch.int64, device=device)     # the counts again
        ctx.gls_get_net_hash_terms_device(own_lo, own_hi, base.data_ptr(),
                                          total.data_ptr() if total is not None else 0,
                                          scratch.data_ptr(), terms.data_ptr())
        return terms

    return stitch_hashes(counts, terms_fn, group)


# ---------------------------------------------------------------- waveform stitching
# SURVEY §8(e) "Stitch": all_gather the per-net counts of every rank's owned window ->
# global offsets -> the rank segments go to the owner (point-to-point over NCCL / NVLink)
# -> the owner scatters each rank's per-net runs into the canonical CSR on its device.

def assemble(allc, bufs, scatter_fn, out_alloc):
    """Owner side: canonical CSR from the ranks' window CSRs.

    allc: [world, nets] int64 counts (rank r's transitions of net n in its window, the
    windows in time order); bufs[r]: rank r's window CSR transitions (net order);
    scatter_fn(nseg, src_off, src, dst_off, dst) copies segment i of src (src_off[i] ..
    src_off[i+1]) to dst + dst_off[i].  Returns (offsets [nets+1], transitions)."""
    world, n = allc.shape
    total_n = allc.sum(0)
    off = torch.zeros(n + 1, dtype=torch.int64, device=allc.device)
    torch.cumsum(total_n, 0, out=off[1:])
    out = out_alloc(int(off[-1]))
    before = torch.zeros(n, dtype=torch.int64, device=allc.device)     # transitions of the net in earlier windows
    for r in range(world):
        src_off = torch.zeros(n + 1, dtype=torch.int64, device=allc.device)
        torch.cumsum(allc[r], 0, out=src_off[1:])
        scatter_fn(n, src_off, bufs[r], off[:-1] + before, out)
        before += allc[r]
    return off, out


def stitch_waveforms(counts, buf, scatter_fn, out_alloc, dst=0, group=None):
    """Every rank: counts [nets] (int64) and buf (its window CSR transitions, int64 bits);
    the canonical CSR of the whole run on rank `dst` (None elsewhere)."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    allc = [torch.empty_like(counts) for _ in range(world)]
    all_gather_t(allc, counts, group=group)
    allc = torch.stack(allc)
    sizes = allc.sum(1).tolist()
    if rank != dst:
        if sizes[rank]:
            send_t(buf[:sizes[rank]].contiguous(), dst, group=group)
        return None
    bufs = []
    for r in range(world):
        if r == rank:
            bufs.append(buf)
        else:
            b = torch.empty(max(1, sizes[r]), dtype=torch.int64, device=counts.device)
            if sizes[r]:
                recv_t(b[:sizes[r]], r, group=group)
            bufs.append(b)
    return assemble(allc, bufs, scatter_fn, out_alloc)


def gls_window_csr(ctx, own_lo, own_hi, device, net_lo=0, net_hi=None):
    """This rank's owned window as a device CSR (gls_get_waveforms_range_device):
    (counts [nets], transitions)."""
    n_all = ctx.num_inputs + ctx.num_gates
    net_hi = n_all if net_hi is None else net_hi
    n = net_hi - net_lo
    offs = torch.empty(n + 1, dtype=torch.int64, device=device)
    total = ctx.gls_get_waveforms_range_device(net_lo, net_hi, own_lo, own_hi, offs.data_ptr())
    tr = torch.empty(max(1, total), dtype=torch.int64, device=device)
    ctx.gls_get_waveforms_range_device(net_lo, net_hi, own_lo, own_hi, offs.data_ptr(), tr.data_ptr(), tr.numel())
    return offs[1:] - offs[:-1], tr


def gls_scatter(ctx):
    """scatter_fn running gls_scatter_segments on ctx's device."""
    def fn(nseg, src_off, src, dst_off, dst):
        ctx.gls_scatter_segments(nseg, src_off.data_ptr(), src.data_ptr(), dst_off.contiguous().data_ptr(),
                                 dst.data_ptr())
    return fn


def gls_gather_waveforms(ctx, own_lo, own_hi, device, dst=0, group=None, net_lo=0, net_hi=None):
    """Canonical CSR of nets [net_lo, net_hi) over the whole run on rank `dst` (device
    tensors (offsets, transitions as int64 bits)), from the ranks' time windows."""
    counts, tr = gls_window_csr(ctx, own_lo, own_hi, device, net_lo, net_hi)
    return stitch_waveforms(counts, tr, gls_scatter(ctx),
                            lambda k: torch.empty(max(1, k), dtype=torch.int64, device=device), dst, group)
