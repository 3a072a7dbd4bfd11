"""Pins for the CPU oracle (oracle/gls_oracle.c) — CPU only, no GPU.

Each test checks the oracle against something other than itself: values the
paper prints (Table 1, Fig. 2, Fig. 3), hand-derived worked examples
(tests/golden/), closed forms, invariants, textbook special cases (zero-delay
simulation, classic event-queue simulation), and brute force on tiny inputs
(tests/refsim.py).
"""
import itertools

import numpy as np
import pytest

import golden_io
import refsim
from oracle import oracle
from paper_2304_13398_b200 import workloads as W

OPS = {"AND": W.AND, "OR": W.OR, "XOR": W.XOR}


def run_oracle(nl, st, duration):
    return oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net,
                           nl.pin_delay, st.offsets, st.trans, duration)


def gates_of(nl):
    out = []
    for g in range(nl.num_gates):
        a, b = nl.fanin_offsets[g], nl.fanin_offsets[g + 1]
        out.append((int(nl.gate_type[g]), [int(x) for x in nl.fanin_net[a:b]],
                    [tuple(int(x) for x in nl.pin_delay[e]) for e in range(a, b)]))
    return out


def stim_lists(st):
    return [[(int(x >> 2), int(x & 3)) for x in st.trans[st.offsets[p]:st.offsets[p + 1]]]
            for p in range(len(st.offsets) - 1)]


# ---------------------------------------------------------------- Table 1
def test_table1_oracle():
    rows = golden_io.table1()
    assert len(rows) == 48
    for op, a, b, r in rows:
        assert oracle.eval_gate(OPS[op], [a, b]) == r, (op, a, b)


def test_table1_closure_checker():
    """The independent closure semantics (X = 0 or 1) reproduces Table 1."""
    for op, a, b, r in golden_io.table1():
        assert refsim.gate_closure(OPS[op], [a, b]) == r


@pytest.mark.parametrize("t", range(9))
def test_gate_functions_exhaustive(t):
    ks = [1] if t in (W.BUF, W.NOT) else ([3] if t == W.MUX2 else [2, 3, 4])
    for k in ks:
        for v in itertools.product(range(4), repeat=k):
            assert oracle.eval_gate(t, list(v)) == refsim.gate_closure(t, list(v)), (t, v)


def test_invariants():
    for t in range(9):
        k = 1 if t in (W.BUF, W.NOT) else (3 if t == W.MUX2 else 2)
        for v in itertools.product(range(4), repeat=k):
            o = oracle.eval_gate(t, list(v))
            assert o in (0, 1, 2)                          # never Z (R12)
            for i in range(k):                             # Z-opacity
                if v[i] == 3:
                    w = list(v)
                    w[i] = 2
                    assert oracle.eval_gate(t, w) == o
            if t != W.MUX2 and o != 2:                     # monotone X
                for i in range(k):
                    if v[i] in (2, 3):
                        for b in (0, 1):
                            w = list(v)
                            w[i] = b
                            assert oracle.eval_gate(t, w) == o
    for a, b in itertools.product(range(4), repeat=2):     # De Morgan
        assert oracle.eval_gate(W.NAND, [a, b]) == oracle.eval_gate(
            W.OR, [oracle.eval_gate(W.NOT, [a]), oracle.eval_gate(W.NOT, [b])])


def test_mux2_reading():
    """MUX2 = OR(AND(a, NOT s), AND(b, s)) (P:339 composition, reading R11)."""
    assert oracle.eval_gate(W.MUX2, [1, 1, 2]) == 2
    assert oracle.eval_gate(W.MUX2, [0, 1, 0]) == 0
    assert oracle.eval_gate(W.MUX2, [0, 1, 1]) == 1
    assert oracle.eval_gate(W.MUX2, [0, 0, 3]) == 0


# ---------------------------------------------------------------- worked examples
@pytest.mark.parametrize("ex", golden_io.examples(), ids=lambda e: e.name)
def test_worked_examples(ex):
    nl, st, dur, index, exp = ex.build()
    r = run_oracle(nl, st, dur)
    for net, wave in exp.items():
        assert r.wave(net) == wave, (ex.name, ex.cite, nl.names[net])


# ---------------------------------------------------------------- closed forms
def test_buf_pulse_closed_form():
    """BUF, pulse of width w: passes iff w > d_rise - d_fall, width w + d_fall - d_rise."""
    gates, waves, cases = [], [], []
    a = 100
    for dr in range(12):
        for df in range(12):
            for w in range(1, 15):
                p = len(waves)
                waves.append([(0, 0), (a, 1), (a + w, 0)])
                gates.append((W.BUF, [p], [(df, dr, df, dr)]))   # (rise0,rise1,fall0,fall1)
                cases.append((dr, df, w))
    P = len(waves)
    nl = W.netlist_from_gates(P, [(t, f, d) for t, f, d in gates])
    r = run_oracle(nl, W.stimuli_from_lists(waves), 1000)
    for g, (dr, df, w) in enumerate(cases):
        exp = [(df, 0)]
        if w > dr - df:
            exp += [(a + dr, 1), (a + w + df, 0)]
        assert r.wave(P + g) == exp, (dr, df, w)


@pytest.mark.parametrize("seed", range(6))
def test_uniform_delay_is_shifted_rle(seed):
    """All delays = d: nothing is eaten (r_j strictly increasing), so each gate
    output is the run-length encoding of its zero-delay evaluation, shifted by d."""
    d = 1 + seed
    nl = W.random_dag(seed, 6, 40, max_delay=0)
    nl.pin_delay[:] = d
    st = W.random_stimuli(seed, 6, 12, 200, xz=0.2)
    dur = 260
    r = run_oracle(nl, st, dur)
    for g, (t, fin, _) in enumerate(gates_of(nl)):
        ins = [r.wave(s) for s in fin]
        times = sorted({tt for w in ins for tt, _ in w})
        prev, exp = 2, []
        for tj in times:
            e = refsim.gate_closure(t, [refsim._value_at(w, tj) for w in ins])
            if e != prev:
                if tj + d <= dur:
                    exp.append((tj + d, e))
                prev = e
        assert r.wave(nl.num_inputs + g) == exp


@pytest.mark.parametrize("seed", range(20))
def test_zero_delay_is_pointwise(seed):
    nl = W.random_dag(100 + seed, 5, 30, max_delay=0)
    st = W.random_stimuli(seed, 5, 15, 120, xz=0.25)
    r = run_oracle(nl, st, 150)
    ref = refsim.zero_delay_sim(nl.num_inputs, gates_of(nl), stim_lists(st), 150)
    for n in range(nl.num_nets):
        assert r.wave(n) == ref[n], n


@pytest.mark.parametrize("seed", range(25))
def test_event_queue_equivalence(seed):
    """Delays >= 1: a classic global event-queue simulator agrees."""
    nl = W.random_dag(200 + seed, 5, 25, min_delay=1, max_delay=9)
    st = W.random_stimuli(seed, 5, 15, 150, xz=0.2, min_gap=1, max_gap=9)
    dur = 200
    r = run_oracle(nl, st, dur)
    ref = refsim.event_queue_sim(nl.num_inputs, gates_of(nl), stim_lists(st), dur)
    for n in range(nl.num_nets):
        assert r.wave(n) == ref[n], n


@pytest.mark.parametrize("seed", range(10))
def test_closed_form_netlists(seed):
    """Whole random netlists (zero delays allowed) against the pointwise closed form."""
    nl = W.random_dag(300 + seed, 4, 15, max_delay=6)
    st = W.random_stimuli(seed, 4, 10, 60, xz=0.25, max_gap=6)
    dur = 90
    r = run_oracle(nl, st, dur)
    ref = refsim.closed_form_sim(nl.num_inputs, gates_of(nl), stim_lists(st), dur)
    for n in range(nl.num_nets):
        assert r.wave(n) == ref[n], n


def _all_small_waves():
    """every waveform with <= 2 transitions at times {0..3}, no repeated value, first != X"""
    out = [[]]
    for n in (1, 2):
        for ts in itertools.combinations(range(4), n):
            for vs in itertools.product(range(4), repeat=n):
                prev, ok = 2, True
                for v in vs:
                    if v == prev:
                        ok = False
                    prev = v
                if ok:
                    out.append(list(zip(ts, vs)))
    return out


def test_bruteforce_single_gates():
    """Exhaustive tiny inputs: every 1- and 2-input gate over all small waveforms
    (random delay tables in 0..3) against the pointwise closed form."""
    small = _all_small_waves()
    rng = np.random.Generator(np.random.PCG64(5))
    gates, waves, meta = [], [], []
    for t in (W.BUF, W.NOT):
        for w in small:
            d = [tuple(int(x) for x in rng.integers(0, 4, 4))]
            gates.append((t, [len(waves)], d))
            waves.append(w)
    for t in (W.AND, W.NAND, W.OR, W.NOR, W.XOR, W.XNOR):
        for w1, w2 in itertools.product(small, small):
            d = [tuple(int(x) for x in rng.integers(0, 4, 4)) for _ in range(2)]
            gates.append((t, [len(waves), len(waves) + 1], d))
            waves += [w1, w2]
    for _ in range(3000):   # MUX2 / 3- and 4-input gates: sampled
        t = int(rng.choice([W.MUX2, W.AND, W.OR, W.XOR, W.NOR]))
        k = 3 if t == W.MUX2 else int(rng.integers(3, 5))
        d = [tuple(int(x) for x in rng.integers(0, 4, 4)) for _ in range(k)]
        gates.append((t, list(range(len(waves), len(waves) + k)), d))
        waves += [small[int(rng.integers(len(small)))] for _ in range(k)]
    P = len(waves)
    nl = W.netlist_from_gates(P, gates)
    dur = 8
    r = run_oracle(nl, W.stimuli_from_lists(waves), dur)
    for g, (t, fin, d) in enumerate(gates):
        exp = refsim.closed_form_gate(t, [waves[s] for s in fin], d, dur)
        assert r.wave(P + g) == exp, (t, [waves[s] for s in fin], d)


def test_recursive_glitch_eaten():
    """One late schedule denies three pending ones (4-value recursion, P:508;
    SPEC acceptance S:572): AND(a,b), a: 0,1,X,1 with slow (50 ps) delays,
    b falls at 13 with a 1 ps delay -> schedules at 60,61,62 are all denied and
    the result equals the prior 0: no change."""
    nl = W.netlist_from_gates(2, [(W.AND, [0, 1], [(50, 50, 50, 50), (1, 1, 1, 1)])])
    st = W.stimuli_from_lists([[(0, 0), (10, 1), (11, 2), (12, 1)], [(0, 1), (13, 0)]])
    r = run_oracle(nl, st, 200)
    assert r.wave(2) == [(1, 0)]
    assert r.events == 5   # 0@0, 1@10, X@11, 1@12, 0@13 (zero-delay output changes)


def test_counts():
    """gate_evals = sum over gates of distinct fan-in timestamps;
    out_trans = sum of gate output lengths."""
    nl = W.random_dag(7, 6, 50, max_delay=8)
    st = W.random_stimuli(7, 6, 20, 300, xz=0.1)
    r = run_oracle(nl, st, 400)
    ge = 0
    for g, (t, fin, _) in enumerate(gates_of(nl)):
        ge += len({tt for s in fin for tt, _ in r.wave(s)})
    assert r.gate_evals == ge
    assert r.out_trans == sum(len(r.wave(nl.num_inputs + g)) for g in range(nl.num_gates))


def test_pi_verbatim_and_hash():
    nl = W.random_dag(8, 4, 10)
    st = W.random_stimuli(8, 4, 10, 100)
    r = run_oracle(nl, st, 150)
    assert np.array_equal(r.trans[:st.total], st.trans)
    # hash definition recomputed in Python
    M = (1 << 64) - 1

    def sm(x):
        x = (x + 0x9E3779B97F4A7C15) & M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
        return x ^ (x >> 31)
    for n in range(nl.num_nets):
        e = r.trans[r.offsets[n]:r.offsets[n + 1]]
        h = sm(0x9E3779B97F4A7C15 ^ len(e))
        for j, x in enumerate(e):
            h ^= sm((int(x) + (j + 1) * 0xD1B54A32D192ED03) & M)
        assert h == int(r.hashes[n])


def test_cycle_rejected():
    nl = W.netlist_from_gates(1, [(W.AND, [0, 2], [(1,) * 4] * 2), (W.BUF, [1], [(1,) * 4])])
    with pytest.raises(oracle.OracleError):
        run_oracle(nl, W.stimuli_from_lists([[(0, 1)]]), 10)


# ---------------------------------------------------------------- time windows (halo)
def _max_arrival(nl):
    P, G = nl.num_inputs, nl.num_gates
    A = np.zeros(P + G, np.int64)
    order = refsim.topo_order(P, gates_of(nl))
    for g in order:
        a, b = nl.fanin_offsets[g], nl.fanin_offsets[g + 1]
        dmax = int(nl.pin_delay[a:b].max())
        A[P + g] = max(int(A[s]) for s in nl.fanin_net[a:b]) + dmax
    return int(A.max())


def _clamp_window(waves, t_clamp, t_hi):
    out = []
    for w in waves:
        v = 2
        rest = []
        for t, x in w:
            if t <= t_clamp:
                v = x
            elif t <= t_hi:
                rest.append((t, x))
        out.append(([(t_clamp, v)] if v != 2 else []) + rest)
    return out


@pytest.mark.parametrize("seed", range(12))
def test_time_window_with_halo_is_exact(seed):
    """Reading R17: simulating a window [T0, T1] from given
    waveforms clamped at T0 - H (every earlier transition collapsed into one at
    T0 - H), H = 1 + max path delay, reproduces every net on [T0, T1]."""
    nl = W.random_dag(400 + seed, 5, 40, max_delay=12)
    st = W.random_stimuli(seed, 5, 40, 600, xz=0.15, max_gap=20)
    dur = 700
    full = run_oracle(nl, st, dur)
    H = _max_arrival(nl) + 1
    waves = stim_lists(st)
    for T0, T1 in [(150, 300), (301, 450), (451, 700)]:
        win = W.stimuli_from_lists(_clamp_window(waves, T0 - H, T1))
        r = run_oracle(nl, win, T1)
        for n in range(nl.num_inputs, nl.num_nets):
            a = [x for x in full.wave(n) if T0 <= x[0] <= T1]
            b = [x for x in r.wave(n) if T0 <= x[0] <= T1]
            # value just before T0 must also agree
            va = refsim._value_at(full.wave(n), T0 - 1)
            vb = refsim._value_at(r.wave(n), T0 - 1)
            assert (a, va) == (b, vb), (seed, T0, n)
