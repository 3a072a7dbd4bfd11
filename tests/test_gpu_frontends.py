"""NEXT-4 on the GPU: the register-cut re-simulation loop (regcut) with the library doing
every simulation pass, against the same loop run by the oracle, and a VCD round trip of
a simulated result."""
import io

import numpy as np
import pytest

from oracle import oracle
from paper_2304_13398_b200 import gls, io_vcd, regcut
from paper_2304_13398_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _gls_fn(ctx, nl, duration):
    ctx.load(nl)

    def fn(offsets, trans):
        ctx.gls_set_input_waveforms(nl.num_inputs, offsets, trans)
        ctx.gls_simulate(duration)
        w = ctx.gls_get_waveforms()
        return w.offsets, w.trans
    return fn


def _oracle_fn(nl, duration):
    def fn(offsets, trans):
        r = oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay,
                            offsets, trans, duration)
        return r.offsets, r.trans
    return fn


def test_register_cut_loop_gpu_equals_oracle():
    # an LFSR-like ring: 6 registers, XOR feedback, a data input mixed in
    P_true, F = 1, 6
    gates, regs = [], []
    for k in range(F):
        src = P_true + (k - 1) % F
        if k == 0:
            gates.append((W.XOR, [P_true + F - 1, P_true + 3], [(7, 8, 6, 9)] * 2))
            gates.append((W.XOR, [P_true + F + 0, 0], [(5, 6, 5, 7)] * 2))
            regs.append(regcut.Register(d=P_true + F + 1, clk_to_q=4, init=1))
        else:
            gates.append((W.BUF, [src], [(3, 4, 3, 4)]))
            regs.append(regcut.Register(d=P_true + F + len(gates) - 1, clk_to_q=4, init=0))
    nl = regcut.cut(P_true, regs, gates)
    period, cycles = 200, 24
    edges = [period * (j + 1) for j in range(cycles)]
    dur = period * (cycles + 1)
    rng = np.random.default_rng(4)
    data, prev = [], 2
    for j in range(cycles):
        b = int(rng.integers(0, 2))
        if b != prev:
            data.append((period * j + 90, b))
            prev = b
    with gls.Context(0) as ctx:
        go, gt, greg, grounds = regcut.resimulate(_gls_fn(ctx, nl, dur), [data], regs, edges, dur)
    oo, ot, oreg, orounds = regcut.resimulate(_oracle_fn(nl, dur), [data], regs, edges, dur)
    assert greg == oreg and grounds == orounds
    assert np.array_equal(go, oo) and np.array_equal(gt, ot)


def test_vcd_export_of_gpu_result_round_trips():
    nl = W.random_dag(41, 5, 60, max_delay=9)
    st = W.random_stimuli(41, 5, 40, 800, xz=0.1)
    with gls.Context(0) as ctx:
        ctx.load(nl)
        ctx.gls_set_input_waveforms(5, st.offsets, st.trans)
        ctx.gls_simulate(900)
        w = ctx.gls_get_waveforms()
    names = [f"n{i}" for i in range(nl.num_nets)]
    buf = io.StringIO()
    io_vcd.write_vcd(buf, names, w.offsets, w.trans)
    o, t = io_vcd.read_vcd(buf.getvalue(), names)
    assert np.array_equal(o, w.offsets) and np.array_equal(t, w.trans)
