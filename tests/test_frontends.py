"""NEXT-4 front / back ends on CPU: VCD import / export (io_vcd), SDF-like IOPATH import
(io_sdf) and the register-cut sequential re-simulation loop (regcut), the simulation step
of the loop run by the oracle (the GPU runs it in test_gpu_frontends.py)."""
import io

import numpy as np
import pytest

from oracle import oracle
from paper_2304_13398_b200 import io_sdf, io_vcd, regcut
from paper_2304_13398_b200 import workloads as W


def test_vcd_round_trip_and_parsing():
    st = W.random_stimuli(3, 6, 25, 400, xz=0.2)
    buf = io.StringIO()
    io_vcd.write_vcd(buf, [f"in{i}" for i in range(6)], st.offsets, st.trans)
    o, t = io_vcd.read_vcd(buf.getvalue(), [f"in{i}" for i in range(6)])
    assert np.array_equal(o, st.offsets) and np.array_equal(t, st.trans)
    vcd = """$timescale 10ps $end
$scope module top $end
$var wire 1 ! a $end
$var wire 4 # bus [3:0] $end
$upscope $end
$enddefinitions $end
#0
$dumpvars
x!
b0x10 #
$end
#3
1!
b1111 #
#5
0!
0!
"""
    o, t = io_vcd.read_vcd(vcd, ["a", "bus[0]", "bus[2]", "top.bus[3]", "absent"])
    waves = [[(int(x >> 2), int(x & 3)) for x in t[o[i]:o[i + 1]]] for i in range(5)]
    # a leading x is the initial X (dropped); a repeated value is no transition; 10 ps units
    assert waves == [[(30, 1), (50, 0)], [(0, 0), (30, 1)], [(30, 1)], [(0, 0), (30, 1)], []]


def test_sdf_iopaths():
    nl = W.netlist_from_gates(2, [(W.NAND, [0, 1], [(1, 1, 1, 1)] * 2), (W.NOT, [2], [(1, 1, 1, 1)]),
                                  (W.MUX2, [0, 1, 2], [(1, 1, 1, 1)] * 3)])
    sdf = """(DELAYFILE (SDFVERSION "3.0") (TIMESCALE 1ns)
     (CELL (CELLTYPE "NAND2") (INSTANCE u1)
       (DELAY (ABSOLUTE (IOPATH A Y (0.003:0.004:0.005) (0.002)) (IOPATH (posedge B) Y (7) (8)))))
     (CELL (CELLTYPE "INV") (INSTANCE u2) (DELAY (INCREMENT (IOPATH A Y (0.010)))))
     (CELL (CELLTYPE "MX2") (INSTANCE u3) (DELAY (ABSOLUTE (IOPATH S Y (0.020) (0.030)))))
    )"""
    pd = io_sdf.read_sdf(sdf, ["u1", "u2", "u3"], nl.fanin_offsets, nl.pin_delay.copy(), gate_type=nl.gate_type)
    # (rise->0, rise->1, fall->0, fall->1): SDF rise = output to 1, fall = output to 0
    assert pd[0].tolist() == [2, 4, 2, 4]
    assert pd[1].tolist() == [8000, 7000, 1, 1]          # posedge B only
    assert pd[2].tolist() == [11, 11, 11, 11]            # INCREMENT
    assert pd[5].tolist() == [30, 20, 30, 20]            # MUX2 select pin S
    with pytest.raises(ValueError):
        io_sdf.read_sdf("(DELAYFILE (CELL (INSTANCE nope)))", ["u1"], nl.fanin_offsets, nl.pin_delay.copy())


def _oracle_fn(nl, duration):
    def fn(offsets, trans):
        r = oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay,
                            offsets, trans, duration)
        return r.offsets, r.trans
    return fn


def _shift_register(n=3):
    # net 0: in; nets 1..n: register Q; gates: BUF(in) -> D0, BUF(Q_k) -> D_{k+1}
    gates = [(W.BUF, [0], [(3, 3, 3, 3)])] + [(W.BUF, [1 + k], [(3, 3, 3, 3)]) for k in range(n - 1)]
    regs = [regcut.Register(d=1 + n + k, clk_to_q=5, init=0) for k in range(n)]
    return regcut.cut(1, regs, gates), regs


def test_shift_register_fixed_point_closed_form():
    n, period, cycles = 3, 100, 12
    nl, regs = _shift_register(n)
    edges = [period * (j + 1) for j in range(cycles)]
    dur = period * (cycles + 1)
    rng = np.random.default_rng(1)
    bits = [int(x) for x in rng.integers(0, 2, size=cycles + 1)]
    inw, prev = [], 2
    for j, b in enumerate(bits):                         # in changes 50 ps into each cycle
        if b != prev:
            inw.append((period * j + 50, b))
            prev = b
    offs, tr, reg, rounds = regcut.resimulate(_oracle_fn(nl, dur), [inw], regs, edges, dur)
    assert rounds <= n + 2
    # closed form: after edge j, Q_k holds the input of cycle j - k (0 before the pipe fills)
    for k in range(n):
        exp, prev = [(0, 0)], 0
        for j in range(cycles):
            v = bits[j - k] if j - k >= 0 else 0
            if v != prev:
                exp.append((edges[j] + 5, v))
                prev = v
        assert reg[k] == exp, (k, reg[k], exp)
    # one pass with the converged register waveforms agrees; a corrupted one is reported
    _, _, bad = regcut.check(_oracle_fn(nl, dur), [inw], reg, regs, edges, dur)
    assert bad == []
    wrong = [list(r) for r in reg]
    wrong[1] = [(0, 0), (edges[2] + 5, 1)] if wrong[1] != [(0, 0), (edges[2] + 5, 1)] else [(0, 0)]
    _, _, bad = regcut.check(_oracle_fn(nl, dur), [inw], wrong, regs, edges, dur)
    assert 1 in bad


def test_counter_fixed_point():
    # 2-bit counter: q0' = NOT q0, q1' = q1 XOR q0 (nets: 0 = unused input, 1 = q0, 2 = q1)
    gates = [(W.NOT, [1], [(4, 4, 4, 4)]), (W.XOR, [2, 1], [(6, 6, 6, 6)] * 2)]
    regs = [regcut.Register(d=3, clk_to_q=2, init=0), regcut.Register(d=4, clk_to_q=2, init=0)]
    nl = regcut.cut(1, regs, gates)
    period, cycles = 50, 9
    edges = [period * (j + 1) for j in range(cycles)]
    dur = period * (cycles + 1)
    offs, tr, reg, rounds = regcut.resimulate(_oracle_fn(nl, dur), [[]], regs, edges, dur)
    q0 = [(0, 0)] + [(edges[j] + 2, (j + 1) % 2) for j in range(cycles)]
    q1, prev = [(0, 0)], 0
    for j in range(cycles):
        v = ((j + 1) >> 1) & 1
        if v != prev:
            q1.append((edges[j] + 2, v))
            prev = v
    assert reg[0] == q0 and reg[1] == q1
