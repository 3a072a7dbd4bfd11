"""tests/refsim.py — independent pure-Python cross-checkers used as PINS for the
oracle.  Test-only; slow; for tiny inputs.  Nothing here is imported by the
product or by the oracle, and nothing here calls the oracle.

Each checker computes the same waveforms by a *different* route than the
oracle's literal Algorithm 2 + Eq. 1 list filter (oracle/gls_oracle.c):

* ``gate_closure``     — gate functions from the meaning of X ("0 or 1",
  PAPER.md:147) as the set of outputs over all 0/1 completions, instead of the
  Table-1 folds.  MUX2 is composed from closure AND/OR/NOT (reading R11).
* ``closed_form_gate`` — V(s) = value of the last-determined schedule whose
  appearance time is <= s (reading of Eq. 1 as a closed form), evaluated
  pointwise at every integer s, instead of the push/pop list.
* ``zero_delay_sim``   — with all delays 0 every net is the pointwise
  zero-delay function of the given waveforms (textbook zero-delay simulation).
* ``event_queue_sim``  — a classic global time-ordered event-driven simulator
  with per-output pending schedule lists (valid for delays >= 1).
"""
from __future__ import annotations

import itertools

V0, V1, VX, VZ = 0, 1, 2, 3
BUF, NOT, AND, NAND, OR, NOR, XOR, XNOR, MUX2 = range(9)
TYPE_NAMES = {"BUF": BUF, "NOT": NOT, "AND": AND, "NAND": NAND, "OR": OR, "NOR": NOR,
              "XOR": XOR, "XNOR": XNOR, "MUX2": MUX2}
VAL = {"0": V0, "1": V1, "x": VX, "X": VX, "z": VZ, "Z": VZ}
INF = float("inf")


def _choices(v):
    v = VX if v == VZ else v
    return (0, 1) if v == VX else (v,)


def _closure(fn, vals):
    outs = {fn(*bits) for bits in itertools.product(*[_choices(v) for v in vals])}
    return outs.pop() if len(outs) == 1 else VX


def _bool_fn(t):
    if t == BUF:
        return lambda a: a
    if t == NOT:
        return lambda a: 1 - a
    if t == AND:
        return lambda *a: int(all(a))
    if t == NAND:
        return lambda *a: 1 - int(all(a))
    if t == OR:
        return lambda *a: int(any(a))
    if t == NOR:
        return lambda *a: 1 - int(any(a))
    if t == XOR:
        return lambda *a: sum(a) & 1
    if t == XNOR:
        return lambda *a: 1 - (sum(a) & 1)
    raise ValueError(t)


def gate_closure(t, vals):
    if t == MUX2:
        a, b, s = vals
        l = _closure(_bool_fn(AND), [a, _closure(_bool_fn(NOT), [s])])
        r = _closure(_bool_fn(AND), [b, s])
        return _closure(_bool_fn(OR), [l, r])
    return _closure(_bool_fn(t), vals)


def _norm(v):
    return VX if v == VZ else v


def _rank(v):
    return {V0: 0, VX: 1, V1: 2}[_norm(v)]


def _value_at(w, s):
    """value of waveform w [(t,v)...] at time s (X before the first transition)."""
    v = VX
    for t, x in w:
        if t <= s:
            v = x
        else:
            break
    return v


def gate_events(t, ins, delays):
    """Events of one gate: list of (t_j, v_j, r_j) — steps 1-5 of DESIGN.md §3.
    delays[i] = (rise0, rise1, fall0, fall1)."""
    times = sorted({tt for w in ins for tt, _ in w})
    prev_x = [VX] * len(ins)
    prev_e = VX
    ev = []
    for tj in times:
        x = [_value_at(w, tj) for w in ins]
        e = gate_closure(t, x)
        if e != prev_e:
            d = INF
            for i in range(len(ins)):
                a, b = _norm(prev_x[i]), _norm(x[i])
                if a == b:
                    continue
                rise = _rank(b) > _rank(a)
                r0, r1, f0, f1 = delays[i]
                pair = (r0, r1) if rise else (f0, f1)
                dd = min(pair) if e == VX else pair[e]
                d = min(d, dd)
            ev.append((tj, e, tj + d))
        prev_e = e
        prev_x = x
    return ev


def closed_form_gate(t, ins, delays, duration):
    """W(g) = change points of V(s) = v_{j*}, j* = max{j : r_j <= s}, on integer
    0 <= s <= duration, V(-1) = X."""
    ev = gate_events(t, ins, delays)
    out = []
    prev = VX
    for s in range(0, duration + 1):
        v = VX
        for (_, vj, rj) in ev:  # later j wins
            if rj <= s:
                v = vj
        if v != prev:
            out.append((s, v))
            prev = v
    return out


def topo_order(num_inputs, gates):
    """gates: list of (type, [fanin nets], delays).  Kahn order."""
    n = num_inputs + len(gates)
    known = [True] * num_inputs + [False] * len(gates)
    order = []
    remaining = list(range(len(gates)))
    while remaining:
        nxt = [g for g in remaining if all(known[s] for s in gates[g][1])]
        assert nxt, "cycle"
        for g in nxt:
            known[num_inputs + g] = True
            order.append(g)
        remaining = [g for g in remaining if g not in set(nxt)]
    assert len(known) == n
    return order


def closed_form_sim(num_inputs, gates, stimuli, duration):
    waves = [list(w) for w in stimuli] + [None] * len(gates)
    for g in topo_order(num_inputs, gates):
        t, fin, dl = gates[g]
        waves[num_inputs + g] = closed_form_gate(t, [waves[s] for s in fin], dl, duration)
    return waves


def zero_delay_sim(num_inputs, gates, stimuli, duration):
    """Pointwise zero-delay evaluation: net value at s = f(fan-in values at s)."""
    order = topo_order(num_inputs, gates)
    times = sorted({t for w in stimuli for t, _ in w if t <= duration})
    waves = [list(w) for w in stimuli] + [[] for _ in gates]
    prev = [VX] * len(gates)
    for s in times:
        val = [_value_at(w, s) for w in stimuli] + [VX] * len(gates)
        for g in order:
            t, fin, _ = gates[g]
            val[num_inputs + g] = gate_closure(t, [val[x] for x in fin])
        for g in range(len(gates)):
            v = val[num_inputs + g]
            if v != prev[g]:
                waves[num_inputs + g].append((s, v))
                prev[g] = v
    return waves


def event_queue_sim(num_inputs, gates, stimuli, duration):
    """Classic global event-driven simulation (valid when every delay >= 1).

    State per gate: E (last zero-delay evaluation), pending schedules (time,
    value) sorted by time.  At each time step: apply all appearing changes,
    then evaluate every gate with a changed input, scheduling with the
    glitch-eaten rule (a new schedule denies pending ones at >= its time)."""
    n = num_inputs + len(gates)
    fanout = [[] for _ in range(n)]
    for g, (_, fin, _) in enumerate(gates):
        for i, s in enumerate(fin):
            fanout[s].append((g, i))
    cur = [VX] * n
    E = [VX] * len(gates)
    pend = [[] for _ in gates]
    waves = [list(w) for w in stimuli] + [[] for _ in gates]
    stim_ev = {}
    for p, w in enumerate(stimuli):
        for t, v in w:
            stim_ev.setdefault(t, []).append((p, v))
    while True:
        cand = [t for t in stim_ev]
        cand += [pl[0][0] for pl in pend if pl]
        if not cand:
            break
        t = min(cand)
        if t > duration:
            break
        old = list(cur)
        for p, v in stim_ev.pop(t, []):
            cur[p] = v
        for g, pl in enumerate(pend):
            if pl and pl[0][0] == t:
                _, v = pl.pop(0)
                cur[num_inputs + g] = v
                waves[num_inputs + g].append((t, v))
        changed_nets = [x for x in range(n) if _norm(cur[x]) != _norm(old[x])]
        touched = sorted({g for x in changed_nets for g, _ in fanout[x]})
        for g in touched:
            typ, fin, dl = gates[g]
            e = gate_closure(typ, [cur[s] for s in fin])
            if e == E[g]:
                continue
            d = INF
            for i, s in enumerate(fin):
                a, b = _norm(old[s]), _norm(cur[s])
                if a == b:
                    continue
                rise = _rank(b) > _rank(a)
                r0, r1, f0, f1 = dl[i]
                pair = (r0, r1) if rise else (f0, f1)
                d = min(d, min(pair) if e == VX else pair[e])
            E[g] = e
            r = t + d
            pl = pend[g]
            while pl and pl[-1][0] >= r:
                pl.pop()
            follow = pl[-1][1] if pl else cur[num_inputs + g]
            if follow != e:
                pl.append((r, e))
    return waves
