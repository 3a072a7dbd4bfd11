"""The paper's scheduling claim on the device (Fig. 8/9; SPEC.md:573
criterion 9): with Alg. 1's unlock rule a task starts as soon as its own predecessors
are complete, even while a slower task of an earlier topological layer is still running —
"task F is allowed to begin as long as task C is completed without waiting for the finish
of task A".  A 9-task, 3-layer DAG with the costs emulated by stimulus length (A's
input toggles thousands of times, C's a few), run with the dataflow scheduler and a
per-gate trace (gls_config.trace): F is planned before A completes, and F's consumer too.
Under level barriers (scheduler 1) nothing of layer 2 may complete before A."""
import numpy as np
import pytest

from paper_2304_13398_b200 import gls
from paper_2304_13398_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _dag():
    # nets: 0 a_in (long), 1 b_in, 2 c_in (short); gates (layer): A=0 B=1 C=2 (1), D=3 E=4 F=5 (2),
    # G=6 H=7 I=8 (3)
    d = [(3, 3, 3, 3)]
    gates = [(W.BUF, [0], d), (W.BUF, [1], d), (W.BUF, [2], d),                  # A, B, C
             (W.AND, [3, 4], d * 2), (W.BUF, [4], d), (W.NOT, [5], d),           # D(A,B), E(B), F(C)
             (W.OR, [6, 7], d * 2), (W.BUF, [7], d), (W.NOT, [8], d)]            # G(D,E), H(E), I(F)
    nl = W.netlist_from_gates(3, gates)
    long_in = [(10 * (j + 1), j % 2) for j in range(400_000)]                   # A: the slow task
    mid_in = [(1000 * (j + 1), j % 2) for j in range(200)]
    short_in = [(7, 1), (5000, 0)]
    return nl, W.stimuli_from_lists([long_in, mid_in, short_in]), 10 * 400_001 + 10


def test_dataflow_starts_f_before_a_finishes():
    nl, st, dur = _dag()
    with gls.Context(0) as ctx:
        ctx.gls_set_config(trace=1, chunk_events=1 << 30)     # one chunk per gate: A is one long task
        ctx.load(nl)
        ctx.gls_set_input_waveforms(3, st.offsets, st.trans)
        ctx.gls_simulate(dur)
        tr = ctx.gls_get_trace().astype(np.int64)
    plan, done = tr[:, 0], tr[:, 1]
    A, C, F, I = 0, 2, 5, 8
    assert done[A] - plan[A] > 0
    assert plan[F] < done[A], "F waited for A (a layer barrier)"
    assert done[F] < done[A] and plan[I] < done[A], "F's chain did not overtake A"
    assert plan[F] >= done[C]                                   # ... but it did wait for its own input
