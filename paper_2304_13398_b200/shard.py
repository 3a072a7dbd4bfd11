"""Multi-GPU partitioning of the simulation — host-side logic only.

Time windows: rank r of N owns clock cycles [r*C/N, (r+1)*C/N) and output times
[k_lo*PERIOD, k_hi*PERIOD) (the last rank up to the duration).  Its given
waveforms start `lookback_cycles(H)` cycles earlier, clamped there (reading R17),
so every net is exact on the owned window.  No exchange happens during the
simulation; results and timings are combined afterwards with all_gather.
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


def all_gather_rows(values, device, group=None):
    """all_gather a small float64 vector from every rank -> [world, len] CPU tensor."""
    import torch.distributed as dist
    t = torch.as_tensor(values, dtype=torch.float64, device=device)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return torch.stack(out).cpu()
