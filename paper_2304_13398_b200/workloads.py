"""Seeded synthetic inputs: netlists, delays and stimuli.

This module holds NO arithmetic of the simulation method (no gate function, no
delay selection, no filtering).  It only draws random netlists and given
waveforms with the shapes of the paper's workloads (Table 2),
following the recipe in DESIGN.md §6.  It is shared by both sides of every
parity check (the CUDA path and the oracle), which is allowed because it
produces inputs only.

Stimuli are COUNTER-BASED: the level of primary input i in epoch e is a pure
function hash(seed, i, e), so any time window of any PI can be generated
directly, on the CPU or on the GPU, with bit-identical results (int64 torch ops
with wrapping multiply; tests check CPU == GPU).  Netlists and per-PI activity
parameters are drawn on the host with numpy's PCG64.

Value codes: 0, 1, X = 2, Z = 3.  Packed transition: (t << 2) | v.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

BUF, NOT, AND, NAND, OR, NOR, XOR, XNOR, MUX2 = range(9)
TYPE_NAMES = ["BUF", "NOT", "AND", "NAND", "OR", "NOR", "XOR", "XNOR", "MUX2"]


# --------------------------------------------------------------------------
# data containers (plain arrays, the C-ABI layout)
# --------------------------------------------------------------------------
@dataclass
class Netlist:
    num_inputs: int
    gate_type: np.ndarray      # uint8 [G]
    fanin_offsets: np.ndarray  # int64 [G+1]
    fanin_net: np.ndarray      # int32 [E]
    pin_delay: np.ndarray      # uint32 [E, 4]  (rise->0, rise->1, fall->0, fall->1)
    names: list | None = None  # optional net names (small circuits)

    @property
    def num_gates(self) -> int:
        return int(self.gate_type.shape[0])

    @property
    def num_nets(self) -> int:
        return self.num_inputs + self.num_gates

    @property
    def num_pins(self) -> int:
        return int(self.fanin_net.shape[0])


@dataclass
class Stimuli:
    offsets: np.ndarray   # int64 [P+1]
    trans: np.ndarray     # uint64 [T]   packed (t << 2) | v

    @property
    def total(self) -> int:
        return int(self.trans.shape[0])


def pack(t, v) -> int:
    return (int(t) << 2) | int(v)


def stimuli_from_lists(waves) -> Stimuli:
    """waves: list (per PI) of [(t, v), ...]."""
    offs = np.zeros(len(waves) + 1, np.int64)
    flat = []
    for i, w in enumerate(waves):
        offs[i + 1] = offs[i] + len(w)
        flat.extend(pack(t, v) for t, v in w)
    return Stimuli(offs, np.array(flat, dtype=np.uint64))


def netlist_from_gates(num_inputs, gates, names=None) -> Netlist:
    """gates: list of (type, [fanin nets], [(r0,r1,f0,f1) per pin])."""
    G = len(gates)
    offs = np.zeros(G + 1, np.int64)
    nets, dl = [], []
    types = np.zeros(G, np.uint8)
    for g, (t, fin, d) in enumerate(gates):
        types[g] = t
        offs[g + 1] = offs[g] + len(fin)
        nets.extend(fin)
        dl.extend(d)
    return Netlist(num_inputs, types, offs, np.array(nets, np.int32).reshape(-1),
                   np.array(dl, np.uint32).reshape(-1, 4), names)


# --------------------------------------------------------------------------
# counter-based hashing (int64 torch ops, identical on CPU and GPU)
# --------------------------------------------------------------------------
def _i64(c: int) -> int:
    return c - (1 << 64) if c >= (1 << 63) else c


_K1 = _i64(0x9E3779B97F4A7C15)
_K2 = _i64(0xBF58476D1CE4E5B9)
_K3 = _i64(0x94D049BB133111EB)


def _srl(x: torch.Tensor, k: int) -> torch.Tensor:
    return (x >> k) & ((1 << (64 - k)) - 1)


def _mix(x: torch.Tensor) -> torch.Tensor:
    x = x + _K1
    x = (x ^ _srl(x, 30)) * _K2
    x = (x ^ _srl(x, 27)) * _K3
    return x ^ _srl(x, 31)


def _hash3(seed: int, a: torch.Tensor, b: torch.Tensor, tag: int) -> torch.Tensor:
    """uniform 63-bit non-negative hash of (seed, a, b, tag)."""
    x = _mix(torch.full_like(a, _i64((seed * 0x100000001B3 + tag * 0x9E37) & ((1 << 64) - 1))) ^ a)
    x = _mix(x ^ (b * _K3))
    return _srl(x, 1)


# --------------------------------------------------------------------------
# stimulus model: clocked, period 10,000 ps
# --------------------------------------------------------------------------
PERIOD = 10_000
_TAG_OFF, _TAG_PHASE, _TAG_JIT, _TAG_LVL = 11, 12, 13, 14


@dataclass
class StimSpec:
    """Clocked stimuli for `num_inputs` PIs over `ncycles` cycles.

    PI i toggles only at epoch boundaries; epoch length L_i cycles (1 for the
    "random" profile = the paper's 0.50 toggles/cycle designs, PAPER.md:527,529;
    lognormal-distributed for the "skewed" profile to reach a target WCV,
    Eq. 5).  In each epoch the level is 0/1 with 99 %
    probability (0.5 % X, 0.5 % Z); a transition happens where the level differs
    from the previous epoch's.  Times: cycle*PERIOD + offset_i + jitter(i,cycle)
    with offset_i in [20,80] and jitter in [0,5].
    """
    seed: int
    num_inputs: int
    ncycles: int
    epoch_len: np.ndarray = field(repr=False, default=None)  # int64 [P] (>=1)
    hot: np.ndarray = field(repr=False, default=None)        # int64 [P]: 0, or toggles per cycle of a hot PI

    @property
    def duration(self) -> int:
        # the paper's duration pattern: ncycles * 10^4 + 1 (e.g. 19,990,001 for 1,999 cycles)
        return self.ncycles * PERIOD + 1


HOT_WCV_COLD = 3.0          # WCV of the epoch-toggling PIs when hot PIs carry the rest of the skew


def _epochs(z, mean, w, ncycles):
    """Lognormal epoch lengths (cycles, >= 1) for a target mean transition count and WCV."""
    sigma = math.sqrt(math.log(1.0 + w * w))
    c = mean * np.exp(sigma * z - 0.5 * sigma * sigma)
    return np.clip(np.rint(0.5 * ncycles / np.maximum(c, 1e-9)), 1, ncycles).astype(np.int64)


def _wcv_of(L, hot, ncycles):
    """Expected per-PI transition counts (an epoch boundary changes the level with p ~ 1/2)."""
    e = np.where(hot > 0, hot * ncycles, 0.5 * ncycles / L)
    return float(e.std() / e.mean()), float(e.mean())


def make_stimspec(seed, num_inputs, ncycles, profile="random", mean_trans=None, wcv=None) -> StimSpec:
    hot = np.zeros(num_inputs, np.int64)
    if profile == "random":
        L = np.ones(num_inputs, np.int64)
    elif profile == "skewed":
        assert mean_trans and wcv
        rng = np.random.Generator(np.random.PCG64(seed + 7919))
        z = rng.standard_normal(num_inputs)
        L = _epochs(z, mean_trans, wcv, ncycles)
        if _wcv_of(L, hot, ncycles)[0] < 0.9 * wcv:
            # An epoch is >= 1 cycle, so one PI carries at most ~ncycles/2 transitions and
            # a lognormal mix saturates (WCV ~6 at 1,000 per PI over 297k cycles).  The
            # paper's skewed designs (WCV 17.1 and 54.5) need nets that toggle
            # more than once per cycle: the most active PIs become clock-like (h toggles
            # per cycle), the rest keep lognormal epochs (WCV 3), and the mean activity is
            # held at mean_trans.  The number of hot PIs is set by bisection on the WCV.
            order = np.argsort(-z, kind="stable")
            best = None
            for h in (1, 2, 4, 8, 16):
                H = h * ncycles
                hi_n = int(min(num_inputs // 4, mean_trans * num_inputs // H))

                def at(nh):
                    hh = np.zeros(num_inputs, np.int64)
                    hh[order[:nh]] = h
                    mc = (mean_trans * num_inputs - nh * H) / max(1, num_inputs - nh)
                    Lc = _epochs(z, max(mc, 1e-3), HOT_WCV_COLD, ncycles)
                    return hh, Lc, _wcv_of(Lc, hh, ncycles)[0]

                if hi_n < 1:
                    continue
                if at(hi_n)[2] < wcv:
                    best = at(hi_n)
                    continue
                lo_n = 0
                while hi_n - lo_n > 1:               # smallest count reaching the target
                    mid = (lo_n + hi_n) // 2
                    if at(mid)[2] >= wcv:
                        hi_n = mid
                    else:
                        lo_n = mid
                best = at(hi_n)
                break
            hot, L, _ = best
    else:
        raise ValueError(profile)
    return StimSpec(seed, num_inputs, ncycles, L, hot)


def _pi_params(spec: StimSpec, pis: torch.Tensor):
    dev = pis.device
    L = torch.as_tensor(spec.epoch_len, device=dev)[pis]
    off = 20 + _hash3(spec.seed, pis, torch.zeros_like(pis), _TAG_OFF) % 61
    phase = _hash3(spec.seed, pis, torch.zeros_like(pis), _TAG_PHASE) % L
    return L, off, phase


def _level(spec: StimSpec, pis: torch.Tensor, epoch: torch.Tensor) -> torch.Tensor:
    u = _hash3(spec.seed, pis, epoch, _TAG_LVL)
    r = u % 1000
    bit = (u >> 20) & 1
    lvl = torch.where(r < 5, torch.full_like(u, 2), torch.where(r < 10, torch.full_like(u, 3), bit))
    # the first epoch starts from the initial X: force a 0/1 level there
    return torch.where(epoch == 0, bit, lvl)


def _epoch_of_cycle(k, L, phase):
    # epoch 0 = cycles [0, L - phase); epoch e>=1 starts at cycle e*L - phase
    return torch.div(k + phase, L, rounding_mode="floor")


def _cold_batch(spec, dev, pis, n_ep, e_lo, L, phase, off, cycle_lo, cycle_hi, tot, chunks, counts, p0):
    """Epoch-toggling PIs of one batch: a transition at the first cycle of an epoch whose
    level differs from the previous epoch's."""
    rep = torch.repeat_interleave(torch.arange(pis.numel(), device=dev), n_ep)
    start = torch.cumsum(n_ep, 0) - n_ep
    e = e_lo[rep] + (torch.arange(tot, device=dev, dtype=torch.int64) - start[rep])
    pi = pis[rep]
    Lr, phr, offr = L[rep], phase[rep], off[rep]
    k = torch.clamp(e * Lr - phr, min=0)           # first cycle of the epoch
    ok = (k >= cycle_lo) & (k < cycle_hi) & (k < spec.ncycles)
    cur = _level(spec, pi, e)
    prv = torch.where(e == 0, torch.full_like(e, 2), _level(spec, pi, torch.clamp(e - 1, min=0)))
    m = ok & (cur != prv)
    pi, k, cur, offr = pi[m], k[m], cur[m], offr[m]
    jit = _hash3(spec.seed, pi, k, _TAG_JIT) % 6
    t = k * PERIOD + offr + jit
    chunks.append((pi.to(torch.int32), (t << 2) | cur))
    counts[p0:p0 + pis.numel()] += torch.bincount(pi - p0, minlength=pis.numel())


def generate_stimuli(spec: StimSpec, device="cpu", pi_batch=1 << 16,
                     cycle_lo: int = 0, cycle_hi: int | None = None):
    """All transitions of every PI whose cycle lies in [cycle_lo, cycle_hi).

    Returns (offsets int64 [P+1], trans int64-as-uint64 [T]) as torch tensors on
    `device`.  With cycle_lo = 0 and cycle_hi = ncycles this is the whole
    stimulus set.  Transition at cycle k of PI i exists iff k starts an epoch
    (or k = 0) and level(epoch(k)) != level(epoch(k) - 1) (level(-1) = X).
    """
    dev = torch.device(device)
    P = spec.num_inputs
    if cycle_hi is None:
        cycle_hi = spec.ncycles
    counts = torch.zeros(P, dtype=torch.int64, device=dev)
    chunks = []
    # batch PIs so that one batch covers at most ~`max_epochs` epochs (memory bound)
    max_epochs = 1 << 26
    allp = torch.arange(P, device=dev, dtype=torch.int64)
    L_all, _, ph_all = _pi_params(spec, allp)
    span = max(1, cycle_hi - cycle_lo)
    hot_all = torch.as_tensor(spec.hot if spec.hot is not None else np.zeros(P, np.int64), device=dev)
    ep = torch.where(hot_all > 0, hot_all * span,                      # entries a batch generates per PI
                     torch.div(torch.full_like(allp, span), L_all, rounding_mode="floor") + 2)
    cum = torch.cumsum(ep, 0).cpu().numpy()
    bounds, p0 = [], 0
    while p0 < P:
        base = cum[p0 - 1] if p0 else 0
        p1 = int(np.searchsorted(cum, base + max_epochs, side="right"))
        p1 = min(P, max(p1, p0 + 1), p0 + pi_batch)
        bounds.append((p0, p1))
        p0 = p1
    for p0, p1 in bounds:
        pis = torch.arange(p0, p1, device=dev, dtype=torch.int64)
        L, off, phase = _pi_params(spec, pis)
        e_lo = _epoch_of_cycle(torch.full_like(pis, cycle_lo), L, phase)
        e_hi = _epoch_of_cycle(torch.full_like(pis, max(cycle_hi - 1, cycle_lo)), L, phase)
        n_ep = torch.where(torch.full_like(pis, cycle_hi) > cycle_lo, e_hi - e_lo + 1, torch.zeros_like(pis))
        n_ep = torch.where(hot_all[p0:p1] > 0, torch.zeros_like(n_ep), n_ep)     # hot PIs: below
        tot = int(n_ep.sum().item())
        if tot > 0:
            _cold_batch(spec, dev, pis, n_ep, e_lo, L, phase, off, cycle_lo, cycle_hi, tot, chunks, counts, p0)
        # hot (clock-like) PIs: h transitions per cycle at offset_i + j * PERIOD / h, the value
        # alternating 0/1 from a per-PI start bit (never X: every transition changes the value)
        hp = torch.nonzero(hot_all[p0:p1] > 0).flatten() + p0
        if hp.numel() and cycle_hi > cycle_lo:
            h = hot_all[hp]
            k_hi = min(cycle_hi, spec.ncycles)
            per = (k_hi - cycle_lo) * h
            tot = int(per.sum().item())
            if tot:
                rep = torch.repeat_interleave(torch.arange(hp.numel(), device=dev), per)
                start = torch.cumsum(per, 0) - per
                n = torch.arange(tot, device=dev, dtype=torch.int64) - start[rep] + cycle_lo * h[rep]   # global index
                hr = h[rep]
                k = torch.div(n, hr, rounding_mode="floor")
                j = n - k * hr
                pi = hp[rep]
                _, off, _ = _pi_params(spec, pi)
                sb = _hash3(spec.seed, pi, torch.zeros_like(pi), _TAG_LVL) & 1
                t = k * PERIOD + off + j * torch.div(torch.full_like(hr, PERIOD), hr, rounding_mode="floor")
                chunks.append((pi.to(torch.int32), (t << 2) | ((sb + n) & 1)))
                counts.index_add_(0, hp, per)
    offs = torch.zeros(P + 1, dtype=torch.int64, device=dev)
    offs[1:] = torch.cumsum(counts, 0)
    trans = torch.empty(int(offs[-1].item()), dtype=torch.int64, device=dev)
    # every group holds whole PIs, each PI's entries time-sorted: scatter them to their CSR rows
    for pi, e in chunks:
        if pi.numel() == 0:
            continue
        first = torch.ones_like(pi, dtype=torch.bool)
        first[1:] = pi[1:] != pi[:-1]
        gstart = torch.cummax(torch.where(first, torch.arange(pi.numel(), device=dev), torch.zeros_like(pi)), 0)[0]
        trans[offs[pi.long()] + (torch.arange(pi.numel(), device=dev) - gstart)] = e
    del chunks
    return offs, trans


def window_stimuli(spec: StimSpec, cycle_lo: int, cycle_hi: int, device="cpu", pi_batch=1 << 16):
    """Given waveforms for the cycle window [cycle_lo, cycle_hi), for time-window
    sharding and oracle samples.  Every transition of those cycles is kept; all
    earlier transitions are collapsed into ONE transition at t_clamp =
    cycle_lo * PERIOD carrying the value in effect there (omitted if it is the
    initial X).  Transitions of cycle >= cycle_lo happen after t_clamp (offsets
    >= 20 ps), so the result is a valid waveform set.  With cycle_lo = 0 it is
    the plain prefix.  The halo argument that makes such windows exact is
    DESIGN.md §4 (reading R17).  Returns torch (offsets, trans) on `device`."""
    dev = torch.device(device)
    P = spec.num_inputs
    offs, tr = generate_stimuli(spec, dev, pi_batch=pi_batch, cycle_lo=cycle_lo, cycle_hi=cycle_hi)
    if cycle_lo <= 0:
        return offs, tr
    counts = offs[1:] - offs[:-1]
    pis = torch.arange(P, device=dev, dtype=torch.int64)
    L, _, phase = _pi_params(spec, pis)
    lvl = _level(spec, pis, _epoch_of_cycle(torch.full_like(pis, cycle_lo - 1), L, phase))
    if spec.hot is not None and (spec.hot > 0).any():
        h = torch.as_tensor(spec.hot, device=dev)
        sb = _hash3(spec.seed, pis, torch.zeros_like(pis), _TAG_LVL) & 1
        lvl = torch.where(h > 0, (sb + min(cycle_lo, spec.ncycles) * h - 1) & 1, lvl)   # its last value
    has = lvl != 2
    nc = has.to(torch.int64)
    new_off = torch.zeros(P + 1, dtype=torch.int64, device=dev)
    new_off[1:] = torch.cumsum(counts + nc, 0)
    out = torch.empty(int(new_off[-1].item()), dtype=torch.int64, device=dev)
    cl = torch.nonzero(has).flatten()
    out[new_off[cl]] = (cycle_lo * PERIOD << 2) | lvl[cl]
    if tr.numel():
        pi_of = torch.repeat_interleave(pis, counts)
        rank = torch.arange(tr.numel(), device=dev, dtype=torch.int64) - offs[pi_of]
        out[new_off[pi_of] + nc[pi_of] + rank] = tr
    return new_off, out


def to_stimuli(offs, tr) -> Stimuli:
    return Stimuli(offs.cpu().numpy().astype(np.int64), tr.cpu().numpy().astype(np.uint64))


# --------------------------------------------------------------------------
# netlist recipe (after SURVEY §8(d))
# --------------------------------------------------------------------------
_TYPE_W = {AND: 2, NAND: 3, OR: 2, NOR: 3, MUX2: 1, BUF: 1, NOT: 1}


def recipe_netlist(seed: int, num_gates: int, depth: int, num_inputs: int,
                   p_inj: float = 0.25, geo_p: float = 0.7, xor_frac: float = 0.05,
                   shuffle: bool = False) -> Netlist:
    rng = np.random.Generator(np.random.PCG64(seed))
    G, D, P = num_gates, depth, num_inputs
    lvl_size = np.full(D, G // D, np.int64)
    lvl_size[: G % D] += 1
    lvl_start = np.zeros(D + 1, np.int64)
    lvl_start[1:] = np.cumsum(lvl_size)
    level = np.repeat(np.arange(1, D + 1), lvl_size)            # level of each gate (1..D)

    # gate types
    tw = np.array([_TYPE_W[t] for t in sorted(_TYPE_W)], np.float64)
    tl = np.array(sorted(_TYPE_W), np.int64)
    types = tl[rng.choice(len(tl), size=G, p=tw / tw.sum())]
    isx = rng.random(G) < xor_frac
    types[isx] = np.where(rng.random(int(isx.sum())) < 0.5, XOR, XNOR)
    ar = rng.choice(np.array([2, 3, 4]), size=G, p=[0.6, 0.2, 0.2])
    arity = np.where((types == BUF) | (types == NOT), 1, np.where(types == MUX2, 3, ar))

    offs = np.zeros(G + 1, np.int64)
    offs[1:] = np.cumsum(arity)
    E = int(offs[-1])
    pin_gate = np.repeat(np.arange(G), arity)
    pin_idx = np.arange(E) - offs[pin_gate]
    pin_lvl = level[pin_gate]

    def pick_from_level(lv):
        """random net of level lv (0 = PIs) for each entry of array lv."""
        out = np.empty(lv.shape[0], np.int64)
        is_pi = lv <= 0
        out[is_pi] = rng.integers(0, P, size=int(is_pi.sum()))
        g = ~is_pi
        lg = lv[g]
        sz = lvl_size[lg - 1]
        out[g] = P + lvl_start[lg - 1] + (rng.random(int(g.sum())) * sz).astype(np.int64)
        return out

    src_lvl = np.where(pin_idx == 0, pin_lvl - 1, 0)
    extra = pin_idx > 0
    inj = rng.random(E) < p_inj
    back = rng.geometric(geo_p, size=E)
    src_lvl = np.where(extra, np.where(inj, 0, np.maximum(pin_lvl - back, 0)), src_lvl)
    fanin = pick_from_level(src_lvl).astype(np.int32)

    # delays (ps): per gate base U[5,40]; per pin/value +U[0,6]; in-edge +0..3; rise/fall +-4
    base = rng.integers(5, 41, size=G)[pin_gate]
    pv = rng.integers(0, 7, size=(E, 2))
    eo = rng.integers(0, 4, size=(E, 2))
    asym = rng.integers(-4, 5, size=E)
    d = np.empty((E, 4), np.int64)
    for e_ in range(2):
        for v_ in range(2):
            d[:, e_ * 2 + v_] = base + pv[:, v_] + eo[:, e_] + (asym if v_ == 1 else 0)
    d = np.maximum(d, 0).astype(np.uint32)

    nl = Netlist(P, types.astype(np.uint8), offs, fanin, d)
    if shuffle:
        nl = shuffle_gates(nl, seed + 1)
    return nl


def shuffle_gates(nl: Netlist, seed: int) -> Netlist:
    """Random permutation of the gate order (net ids remapped) — exercises levelisation."""
    rng = np.random.Generator(np.random.PCG64(seed))
    G, P = nl.num_gates, nl.num_inputs
    perm = rng.permutation(G)                  # new gate j = old gate perm[j]
    inv = np.empty(G, np.int64)
    inv[perm] = np.arange(G)
    ar = np.diff(nl.fanin_offsets)[perm]
    offs = np.zeros(G + 1, np.int64)
    offs[1:] = np.cumsum(ar)
    idx = np.concatenate([np.arange(nl.fanin_offsets[g], nl.fanin_offsets[g + 1]) for g in perm]) \
        if G else np.zeros(0, np.int64)
    fin = nl.fanin_net[idx].astype(np.int64)
    fin = np.where(fin >= P, P + inv[np.maximum(fin - P, 0)], fin)
    return Netlist(P, nl.gate_type[perm], offs, fin.astype(np.int32), nl.pin_delay[idx])


# --------------------------------------------------------------------------
# small random designs for parity tests (SPEC-style random DAGs)
# --------------------------------------------------------------------------
def random_dag(seed, num_inputs, num_gates, max_delay=10, min_delay=0, types=None) -> Netlist:
    rng = np.random.Generator(np.random.PCG64(seed))
    P = num_inputs
    types = list(range(9)) if types is None else list(types)
    gates = []
    for g in range(num_gates):
        t = int(rng.choice(types))
        k = 1 if t in (BUF, NOT) else (3 if t == MUX2 else int(rng.integers(2, 5)))
        fin = [int(rng.integers(0, P + g)) for _ in range(k)]
        d = [tuple(int(x) for x in rng.integers(min_delay, max_delay + 1, size=4)) for _ in range(k)]
        gates.append((t, fin, d))
    return shuffle_gates(netlist_from_gates(P, gates), seed + 3)


def random_stimuli(seed, num_inputs, max_trans, tmax, xz=0.2, min_gap=1, max_gap=None) -> Stimuli:
    """Random given waveforms: strictly increasing times in [0, tmax], no repeated value,
    first value not X; X/Z share `xz`."""
    rng = np.random.Generator(np.random.PCG64(seed))
    waves = []
    max_gap = max_gap or max(2, tmax // max(1, max_trans))
    for _ in range(num_inputs):
        n = int(rng.integers(0, max_trans + 1))
        w, t, prev = [], int(rng.integers(0, max_gap + 1)), 2
        for _ in range(n):
            if t > tmax:
                break
            while True:
                r = rng.random()
                v = (2 if rng.random() < 0.5 else 3) if r < xz else int(rng.integers(0, 2))
                if v != prev:
                    break
            w.append((t, v))
            prev = v
            t += int(rng.integers(min_gap, max_gap + 1))
        waves.append(w)
    return stimuli_from_lists(waves)


# --------------------------------------------------------------------------
# named configurations (BASELINE.json configs)
# --------------------------------------------------------------------------
def c17() -> tuple[Netlist, list]:
    names = ["N1", "N2", "N3", "N6", "N7", "N10", "N11", "N16", "N19", "N22", "N23"]
    ix = {n: i for i, n in enumerate(names)}
    g = [("N10", "N1", "N3"), ("N11", "N3", "N6"), ("N16", "N2", "N11"),
         ("N19", "N11", "N7"), ("N22", "N10", "N16"), ("N23", "N16", "N19")]
    gates = [(NAND, [ix[a], ix[b]], [(1, 1, 1, 1)] * 2) for _, a, b in g]
    return netlist_from_gates(5, gates, names), names


CONFIGS = {
    # name: (num_gates, depth, num_inputs, ncycles, profile, mean_trans, wcv)
    "c7552": dict(num_gates=3512, depth=40, num_inputs=207, ncycles=1999, profile="random"),
    "c3_1m": dict(num_gates=1 << 20, depth=200, num_inputs=104858, ncycles=19999, profile="random"),
    "c4_10m": dict(num_gates=10 * (1 << 20), depth=250, num_inputs=1 << 20, ncycles=297203,
                   profile="skewed", mean_trans=1000, wcv=17.0),
    "c5_set": dict(num_gates=1 << 20, depth=200, num_inputs=104858, ncycles=1999, profile="random"),
    # C4's per-net activity and skew on 1/10 of the gates (profiling stand-in for C4)
    "c4_mini": dict(num_gates=1 << 20, depth=100, num_inputs=104858, ncycles=297203,
                    profile="skewed", mean_trans=1000, wcv=17.0),
}


def union_netlist(nl: Netlist, k: int) -> Netlist:
    """k disjoint copies of a netlist as one (independent stimulus sets simulated in one
    launch).  Nets: the copies' given nets first (copy c's net p -> c*P + p), then the
    copies' gates (copy c's gate g -> k*P + c*G + g); see union_nets."""
    if k == 1:
        return nl
    P, G, E = nl.num_inputs, nl.num_gates, nl.num_pins
    fo = nl.fanin_offsets.astype(np.int64)
    src = nl.fanin_net.astype(np.int64)
    offs, nets = [np.zeros(1, np.int64)], []
    for c in range(k):
        offs.append(fo[1:] + c * E)
        nets.append(np.where(src < P, src + c * P, k * P + c * G + (src - P)))
    return Netlist(k * P, np.tile(nl.gate_type, k), np.concatenate(offs),
                   np.concatenate(nets).astype(np.int32), np.tile(nl.pin_delay, (k, 1)))


def union_nets(nl: Netlist, k: int, c: int) -> np.ndarray:
    """user net ids, in the single netlist's net order, of copy c inside union_netlist(nl, k)"""
    P, G = nl.num_inputs, nl.num_gates
    return np.concatenate([c * P + np.arange(P), k * P + c * G + np.arange(G)]).astype(np.int64)


def config_netlist(name: str, seed: int = 1) -> Netlist:
    c = CONFIGS[name]
    return recipe_netlist(seed, c["num_gates"], c["depth"], c["num_inputs"])


def config_stimspec(name: str, seed: int = 1, ncycles: int | None = None) -> StimSpec:
    c = CONFIGS[name]
    return make_stimspec(seed, c["num_inputs"], ncycles or c["ncycles"], c["profile"],
                         c.get("mean_trans"), c.get("wcv"))


def wcv(lengths) -> float:
    """Eq. 5: sigma / mean of the given waveforms' lengths
    (population sigma)."""
    x = np.asarray(lengths, np.float64)
    return float(x.std() / x.mean()) if x.size and x.mean() > 0 else 0.0


# --------------------------------------------------------------------------
# cell netlists (NEXT-2: multi-output cells / UDPs, 5-D delays with GLS_DELAY_INF)
# --------------------------------------------------------------------------
DELAY_INF = 0xFFFFFFFF

# the full adder as one 3-input, 2-output cell template: sum = (a ^ b) ^ cin,
# cout = (a & b) | ((a ^ b) & cin)
FULL_ADDER = dict(n_in=3, n_out=2, gates=[(XOR, [0, 1]), (XOR, [3, 2]), (AND, [0, 1]), (AND, [3, 2]), (OR, [5, 6])],
                  outputs=[4, 7])


def random_template(rng, n_in, n_out, n_gates):
    gates = []
    for j in range(n_gates):
        ty = int(rng.choice([BUF, NOT, AND, NAND, OR, NOR, XOR, XNOR, MUX2]))
        k = 1 if ty in (BUF, NOT) else 3 if ty == MUX2 else int(rng.integers(2, 5))
        nodes = [int(x) for x in rng.integers(0, n_in + j, size=k)]
        gates.append((ty, nodes))
    outs = [int(x) for x in rng.integers(max(0, n_in + n_gates - 3), n_in + n_gates, size=n_out)]
    return dict(n_in=n_in, n_out=n_out, gates=gates, outputs=outs)


def random_cells(seed, num_inputs, num_cells, max_delay=10, p_inf=0.15):
    """A random cell library (a full adder, 3-input and 4-input UDPs with 1-3 outputs) and
    a random DAG of cells over it; delays U[0, max_delay] per (in, out, edge, value),
    GLS_DELAY_INF with probability p_inf.  Returns (templates, cell_tpl, cell_fanin,
    cell_delay) — the arguments of gls_load_cells / oracle.simulate_cells."""
    rng = np.random.Generator(np.random.PCG64(seed))
    templates = [FULL_ADDER,
                 random_template(rng, 2, 2, 3), random_template(rng, 3, 1, 4),
                 random_template(rng, 3, 3, 5), random_template(rng, 4, 1, 4),
                 dict(n_in=1, n_out=2, gates=[(NOT, [0])], outputs=[1, 0])]     # NOT + pass-through
    cell_tpl, fanin, delay = [], [], []
    nets = num_inputs
    for _ in range(num_cells):
        t = int(rng.integers(0, len(templates)))
        tp = templates[t]
        cell_tpl.append(t)
        fanin += [int(x) for x in rng.integers(0, nets, size=tp["n_in"])]
        d = rng.integers(0, max_delay + 1, size=tp["n_in"] * tp["n_out"] * 4).astype(np.uint64)
        d[rng.random(d.size) < p_inf] = DELAY_INF
        delay += [int(x) for x in d]
        nets += tp["n_out"]
    return templates, np.array(cell_tpl, np.int32), np.array(fanin, np.int32), np.array(delay, np.uint32)
