"""NEXT-2 on the GPU: multi-output cells / UDPs (gls_load_cells: templates composed of
basic gates, §3.3) with the 5-D delay matrix and GLS_DELAY_INF (§3.2
P:329-333, reading R9), through the C ABI, bit-exact against oracle.simulate_cells on
every net, with the oracle's counts — both engines and both schedulers, small work items
(time chunks and slices of the cells without `inf`), the worked `inf` examples, and the
error paths."""
import numpy as np
import pytest

from oracle import oracle
from paper_2304_13398_b200 import gls
from paper_2304_13398_b200 import workloads as W

pytestmark = pytest.mark.gpu
ENGINES = [dict(engine=0), dict(engine=0, scheduler=1), dict(engine=1)]
EIDS = ["units-df", "units-lvl", "lane"]


@pytest.fixture(scope="module")
def ctx():
    c = gls.Context(0)
    yield c
    c.close()


def _check(ctx, P, tpl, ct, cf, cd, st, dur, **cfg):
    ref = oracle.simulate_cells(P, tpl, ct, cf, cd, st.offsets, st.trans, dur)
    ctx.gls_set_config(**cfg)
    ctx.gls_load_cells(P, tpl, ct, cf, cd)
    ctx.gls_set_input_waveforms(P, st.offsets, st.trans)
    ctx.gls_simulate(dur)
    w = ctx.gls_get_waveforms()
    if not (np.array_equal(w.offsets, ref.offsets) and np.array_equal(w.trans, ref.trans)):
        for n in range(len(ref.offsets) - 1):
            assert w.wave(n) == ref.wave(n), f"net {n}: gpu {w.wave(n)[:12]} oracle {ref.wave(n)[:12]}"
    s = ctx.gls_get_stats()
    assert (s["gate_evals"], s["events"], s["out_transitions"]) == (ref.gate_evals, ref.events, ref.out_trans)
    assert np.array_equal(ctx.gls_get_net_hashes(), ref.hashes)
    return s


@pytest.mark.parametrize("engine", ENGINES, ids=EIDS)
def test_random_cell_netlists(ctx, engine):
    rng = np.random.default_rng(11)
    for d in range(150):
        P = int(rng.integers(1, 8))
        tpl, ct, cf, cd = W.random_cells(500 + d, P, int(rng.integers(1, 60)), max_delay=int(rng.integers(0, 15)),
                                         p_inf=float(rng.choice([0.0, 0.1, 0.4])))
        st = W.random_stimuli(d, P, int(rng.integers(0, 50)), 500, xz=float(rng.random() * 0.3),
                              max_gap=int(rng.integers(1, 30)))
        try:
            _check(ctx, P, tpl, ct, cf, cd, st, 550, chunk_events=int(rng.choice([0, 3, 17])), **engine)
        except AssertionError as e:
            raise AssertionError(f"design {d}: {e}")


@pytest.mark.parametrize("engine", ENGINES, ids=EIDS)
def test_cells_large_activity(ctx, engine):
    """Long waveforms through cells: time chunks, slices and splits of the cells without
    `inf`, single units for the ones with it."""
    tpl, ct, cf, cd = W.random_cells(77, 12, 400, max_delay=30, p_inf=0.05)
    st = W.random_stimuli(77, 12, 3000, 60000, xz=0.02, min_gap=3, max_gap=40)
    _check(ctx, 12, tpl, ct, cf, cd, st, 61000, chunk_events=256, **engine)


def test_ripple_carry_adder_of_cells(ctx):
    """An 8-bit ripple-carry adder of full-adder cells (the carry chain runs through cell
    outputs), zero delay, against the oracle."""
    nbits = 8
    P = 2 * nbits + 1
    ct, cf = [], []
    carry = 2 * nbits
    for i in range(nbits):
        ct.append(0)
        cf += [i, nbits + i, carry]
        carry = P + 2 * i + 1                   # this cell's cout
    cd = np.zeros(len(ct) * 3 * 2 * 4, np.uint32)
    st = W.random_stimuli(5, P, 40, 1000, xz=0.0)
    s = _check(ctx, P, [W.FULL_ADDER], ct, cf, cd, st, 1100)
    assert s["gate_evals"] > 0


def test_cell_errors(ctx):
    tpl = [W.FULL_ADDER]
    with pytest.raises(gls.GlsError) as e:                                 # template id
        ctx.gls_load_cells(3, tpl, [1], [0, 1, 2], np.zeros(24, np.uint32))
    assert e.value.code == gls.GLS_EINVAL
    with pytest.raises(gls.GlsError) as e:                                 # delay >= 2^31, not inf
        ctx.gls_load_cells(3, tpl, [0], [0, 1, 2], np.full(24, 1 << 31, np.uint32))
    assert e.value.code == gls.GLS_EINVAL
    bad = dict(n_in=2, n_out=1, gates=[(W.AND, [0, 2])], outputs=[2])   # gate reads itself
    with pytest.raises(gls.GlsError) as e:
        ctx.gls_load_cells(2, [bad], [0], [0, 1], np.zeros(8, np.uint32))
    assert e.value.code == gls.GLS_EINVAL
    with pytest.raises(gls.GlsError) as e:                                 # combinational loop
        ctx.gls_load_cells(1, [dict(n_in=1, n_out=1, gates=[(W.NOT, [0])], outputs=[1])], [0, 0], [2, 1],
                           np.zeros(8, np.uint32))
    assert e.value.code == gls.GLS_ECYCLE
    # too many distinct 4-input functions for the LUT area
    rng = np.random.default_rng(1)
    many = [W.random_template(rng, 4, 1, 6) for _ in range(12)]
    with pytest.raises(gls.GlsError) as e:
        ctx.gls_load_cells(4, many, list(range(12)), [0, 1, 2, 3] * 12, np.zeros(12 * 16, np.uint32))
    assert e.value.code == gls.GLS_EINVAL
    # time windows need finite delays
    tpl2, ct, cf, cd = W.random_cells(3, 4, 20, p_inf=0.5)
    ctx.gls_load_cells(4, tpl2, ct, cf, cd)
    st = W.random_stimuli(3, 4, 10, 100)
    ctx.gls_set_input_waveforms(4, st.offsets, st.trans)
    with pytest.raises(gls.GlsError) as e:
        ctx.gls_simulate_window(50, 80, 120)
    assert e.value.code == gls.GLS_EINVAL


@pytest.mark.parametrize("engine", ENGINES, ids=EIDS)
def test_golden_inf_examples_gpu(ctx, engine):
    import test_oracle_cells as toc
    for case in toc._golden():
        st = W.stimuli_from_lists(case["inputs"])
        n_in = case["template"]["n_in"]
        ctx.gls_set_config(**engine)
        ctx.gls_load_cells(n_in, [case["template"]], [0], list(range(n_in)), case["delay"])
        ctx.gls_set_input_waveforms(n_in, st.offsets, st.trans)
        ctx.gls_simulate(case["duration"])
        w = ctx.gls_get_waveforms()
        for q, wave in case["expect"].items():
            assert w.wave(n_in + q) == wave, (case["name"], q)
