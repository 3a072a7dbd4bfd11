"""Pins of the oracle's cell path (oracle_simulate_cells: multi-output cells / UDPs composed
of basic gates, §3.3; the 5-D delay matrix with `inf` = no relation, §3.2
P:329-333, reading R9), against things other than itself:

  * a one-gate template IS that basic gate: a random netlist of basic gates, given as
    one-gate cells, equals the basic-gate oracle (its own Table-1 evaluation and Alg. 2
    loop) net by net, with the same counts;
  * a multi-output cell is its outputs: the full adder as one 2-output cell equals two
    1-output cells (sum, carry) with the matching delay slices;
  * zero delays: every cell output is the pointwise closed form of its template (the
    full adder's sum / carry in 0/1 arithmetic, X propagation by its invariants);
  * worked `inf` examples derived by hand (tests/golden/cells.txt);
  * a NOT + pass-through template's outputs equal the basic NOT / BUF gates."""
import numpy as np
import pytest

from oracle import oracle
from paper_2304_13398_b200 import workloads as W

INF = W.DELAY_INF


def _one_gate_cells(nl):
    """A basic netlist as one-gate cells: one template per (type, arity)."""
    tpls, index, cell_tpl, delay = [], {}, [], []
    for g in range(nl.num_gates):
        a, b = nl.fanin_offsets[g], nl.fanin_offsets[g + 1]
        key = (int(nl.gate_type[g]), int(b - a))
        if key not in index:
            index[key] = len(tpls)
            tpls.append(dict(n_in=key[1], n_out=1, gates=[(key[0], list(range(key[1])))], outputs=[key[1]]))
        cell_tpl.append(index[key])
        for pin in range(a, b):
            r0, r1, f0, f1 = (int(x) for x in nl.pin_delay[pin])
            delay += [r0, r1, f0, f1]            # [in][out=0][edge RISE, FALL][value 0, 1]
    return tpls, np.array(cell_tpl, np.int32), np.asarray(nl.fanin_net, np.int32), np.array(delay, np.uint32)


@pytest.mark.parametrize("seed", range(20))
def test_one_gate_templates_equal_basic_gates(seed):
    rng = np.random.default_rng(seed)
    nl = W.random_dag(3000 + seed, int(rng.integers(2, 8)), int(rng.integers(5, 80)), max_delay=int(rng.integers(0, 12)))
    st = W.random_stimuli(seed, nl.num_inputs, 30, 400, xz=0.2)
    ref = oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay,
                          st.offsets, st.trans, 450)
    tpls, ct, cf, cd = _one_gate_cells(nl)
    got = oracle.simulate_cells(nl.num_inputs, tpls, ct, cf, cd, st.offsets, st.trans, 450)
    assert np.array_equal(got.offsets, ref.offsets) and np.array_equal(got.trans, ref.trans)
    assert (got.gate_evals, got.events, got.out_trans) == (ref.gate_evals, ref.events, ref.out_trans)


def test_multi_output_cell_is_its_outputs():
    sum_only = dict(W.FULL_ADDER, n_out=1, outputs=[4])
    carry_only = dict(W.FULL_ADDER, n_out=1, outputs=[7])
    rng = np.random.default_rng(7)
    for trial in range(30):
        d = rng.integers(0, 9, size=(3, 2, 2, 2)).astype(np.uint32)        # [in][out][edge][value]
        d[rng.random(d.shape) < 0.2] = INF
        st = W.random_stimuli(trial, 3, 25, 300, xz=0.15)
        both = oracle.simulate_cells(3, [W.FULL_ADDER], [0], [0, 1, 2], d.reshape(-1), st.offsets, st.trans, 330)
        split = oracle.simulate_cells(3, [sum_only, carry_only], [0, 1], [0, 1, 2, 0, 1, 2],
                                      np.concatenate([d[:, 0:1].reshape(-1), d[:, 1:2].reshape(-1)]),
                                      st.offsets, st.trans, 330)
        assert np.array_equal(both.offsets, split.offsets) and np.array_equal(both.trans, split.trans)


def test_full_adder_zero_delay_closed_form():
    """0/1 stimuli all starting at t = 0 (no X anywhere): at zero delay the outputs are the
    change points of sum = a ^ b ^ cin and cout = (a & b) | (cin & (a ^ b))."""
    rng = np.random.default_rng(3)
    for trial in range(20):
        lists = []
        for i in range(3):
            t, v, w = 0, int(rng.integers(0, 2)), []
            while t < 200:
                w.append((t, v))
                t += int(rng.integers(1, 15))
                v ^= 1
            lists.append(w)
        st = W.stimuli_from_lists(lists)
        r = oracle.simulate_cells(3, [W.FULL_ADDER], [0], [0, 1, 2], np.zeros(24, np.uint32),
                                  st.offsets, st.trans, 220)
        waves = [dict(w) for w in lists]
        times = sorted({t for w in lists for t, _ in w})

        def val(w, t):
            return w[max(k for k in w if k <= t)]
        exp_s, exp_c, last_s, last_c = [], [], 2, 2
        for t in times:
            a, b, c = (val(w, t) for w in waves)
            s_, c_ = a ^ b ^ c, (a & b) | (c & (a ^ b))
            if s_ != last_s:
                exp_s.append((t, s_))
                last_s = s_
            if c_ != last_c:
                exp_c.append((t, c_))
                last_c = c_
        assert r.wave(3) == exp_s and r.wave(4) == exp_c


def _golden():
    """tests/golden/cells.txt: hand-derived cell examples (see the file for each derivation)."""
    import os
    out, cur = [], None
    for line in open(os.path.join(os.path.dirname(__file__), "golden", "cells.txt")):
        line = line.split("#")[0].strip()
        if not line:
            continue
        k, v = line.split(":", 1)
        k, v = k.strip(), v.strip()
        if k == "case":
            cur = dict(name=v, inputs=[], expect={})
            out.append(cur)
        elif k == "template":
            cur["template"] = eval(v, {"AND": W.AND, "OR": W.OR, "XOR": W.XOR, "NOT": W.NOT, "NAND": W.NAND})
        elif k == "delay":
            cur["delay"] = [INF if x == "inf" else int(x) for x in v.split()]
        elif k == "input":
            cur["inputs"].append(eval(v))
        elif k.startswith("out"):
            cur["expect"][int(k[3:])] = eval(v)
        elif k == "duration":
            cur["duration"] = int(v)
    return out


@pytest.mark.parametrize("case", _golden(), ids=lambda c: c["name"])
def test_golden_inf_examples(case):
    st = W.stimuli_from_lists(case["inputs"])
    n_in = case["template"]["n_in"]
    r = oracle.simulate_cells(n_in, [case["template"]], [0], list(range(n_in)), case["delay"],
                              st.offsets, st.trans, case["duration"])
    for q, wave in case["expect"].items():
        assert r.wave(n_in + q) == wave, (case["name"], q, r.wave(n_in + q))


@pytest.mark.parametrize("seed", range(10))
def test_not_and_pass_through_template(seed):
    """A 1-input template with outputs NOT(in) and the input itself: each output equals the
    basic NOT / BUF gate with that output's delay slice."""
    tpl = [dict(n_in=1, n_out=2, gates=[(W.NOT, [0])], outputs=[1, 0])]
    rng = np.random.default_rng(seed)
    d = rng.integers(0, 9, size=(1, 2, 2, 2)).astype(np.uint32)
    st = W.random_stimuli(seed, 1, 30, 300, xz=0.2)
    r = oracle.simulate_cells(1, tpl, [0], [0], d.reshape(-1), st.offsets, st.trans, 330)
    for q, ty in [(0, W.NOT), (1, W.BUF)]:
        r0, r1 = d[0, q, 0]
        f0, f1 = d[0, q, 1]
        nl = W.netlist_from_gates(1, [(ty, [0], [(int(r0), int(r1), int(f0), int(f1))])])
        ref = oracle.simulate(1, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay, st.offsets, st.trans, 330)
        assert r.wave(1 + q) == ref.wave(1)
