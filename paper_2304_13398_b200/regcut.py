"""Register-cut sequential re-simulation (NEXT-4).

The paper simulates a combinational netlist whose registers have been cut: "the outputs
of registers are regarded as primary inputs (pseudo primary inputs) since their
waveforms are given" (PAPER.md:87 footnote), in a re-simulation flow where those
waveforms come from an earlier run.  This module supplies the step either side of
that path for a design with edge-triggered registers:

  * `cut`: a sequential design (true inputs, registers D -> Q, gates) becomes the
    combinational netlist the library simulates — register outputs are the given nets
    P_true .. P_true + F - 1, their D inputs are ordinary gate-output (or input) nets;
  * `sample_registers`: the register outputs a simulated run implies — each register
    samples its D net at the clock's rising edges (the value in effect just before the
    edge) and its Q takes that value clk_to_q later;
  * `check` (one pass: do the given register waveforms agree with what the combinational
    logic drives into the registers?) and `resimulate` (a fixed-point loop: simulate,
    re-derive the register outputs, repeat until they no longer change; each round fixes
    at least the next clock cycle of every register, so a design whose register state
    reaches back k cycles needs at most k + 1 rounds).

`simulate_fn(offsets, transitions) -> (offsets, transitions)` runs one pass over the whole
duration (gls: set inputs + simulate + get waveforms; the tests also pass the oracle).
Host-side control flow; every simulation runs in the library's kernels.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import workloads as W


@dataclass
class Register:
    d: int                  # net of the register's D input (in the cut netlist's numbering)
    clk_to_q: int = 0       # ps from the clock edge to the Q change
    init: int = 2           # Q before the first edge (0, 1, or X = 2)


def cut(num_true_inputs, registers, gates):
    """The combinational netlist of a register-cut design.  Net numbering: 0..P_true-1 the
    true inputs, P_true + r register r's Q (a pseudo primary input), then the gates'
    outputs in order; `gates` = [(type, [fanin nets], [(r0, r1, f0, f1) per pin])] in that
    numbering (register D nets may be any net)."""
    return W.netlist_from_gates(num_true_inputs + len(registers), gates)


def _value_before(offs, tr, net, t):
    a, b = offs[net], offs[net + 1]
    times = (tr[a:b] >> np.uint64(2)).astype(np.int64)
    k = np.searchsorted(times, t, side="left")            # transitions strictly before t
    return int(tr[a + k - 1] & np.uint64(3)) if k > 0 else 2


def sample_registers(offsets, transitions, registers, clock_edges, duration):
    """Register output waveforms implied by a run: Q = init until the first edge, then at
    edge e + clk_to_q the value D had just before e.  Returns one [(t, v)] list per register
    (given-waveform rules: strictly increasing times, no repeated value, no leading X)."""
    offs = np.asarray(offsets, np.int64)
    tr = np.asarray(transitions).view(np.uint64)
    out = []
    for r in registers:
        w, prev = [], 2
        if r.init != 2:
            w.append((0, int(r.init)))
            prev = int(r.init)
        for e in clock_edges:
            t = int(e) + int(r.clk_to_q)
            if t > duration:
                break
            v = _value_before(offs, tr, r.d, int(e))
            v = 2 if v == 3 else v                           # Z sampled as X
            if w and w[-1][0] == t:                          # an edge at t = 0 overrides init
                w.pop()
                prev = w[-1][1] if w else 2
            if v != prev:
                w.append((t, v))
                prev = v
        out.append(w)
    return out


def _given(true_waves, reg_waves):
    return W.stimuli_from_lists(list(true_waves) + list(reg_waves))


def check(simulate_fn, true_waves, reg_waves, registers, clock_edges, duration):
    """One re-simulation pass with the given register waveforms; returns (offsets,
    transitions, [indices of registers whose given waveform disagrees with the sampled D])."""
    st = _given(true_waves, reg_waves)
    offs, tr = simulate_fn(st.offsets, st.trans)
    implied = sample_registers(offs, tr, registers, clock_edges, duration)
    bad = [i for i, (a, b) in enumerate(zip(reg_waves, implied)) if list(a) != list(b)]
    return offs, tr, bad


def resimulate(simulate_fn, true_waves, registers, clock_edges, duration, max_rounds=64):
    """Fixed-point re-simulation: start from the registers' initial values, simulate, take
    the register outputs the run implies, repeat until they are stable.  Returns (offsets,
    transitions, register waveforms, rounds); raises RuntimeError without convergence."""
    reg = [[(0, int(r.init))] if r.init != 2 else [] for r in registers]
    for rnd in range(1, max_rounds + 1):
        offs, tr, bad = check(simulate_fn, true_waves, reg, registers, clock_edges, duration)
        if not bad:
            return offs, tr, reg, rnd
        reg = sample_registers(offs, tr, registers, clock_edges, duration)
    raise RuntimeError(f"register waveforms did not converge in {max_rounds} rounds")
