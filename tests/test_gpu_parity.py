"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
bit-exact on every transition time and value of every net, plus the oracle's
counts (gate-evals, events, output transitions) and per-net hashes."""
import numpy as np
import pytest
import torch

import golden_io
from oracle import oracle
from paper_2304_13398_b200 import gls
from paper_2304_13398_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = gls.Context(0)
    yield c
    c.close()


def run_oracle(nl, st, dur):
    return oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net,
                           nl.pin_delay, st.offsets, st.trans, dur)


# engine 0 = lanes on re-balanced time-slice units (default), 1 = one chunk per lane;
# scheduler 0 = dataflow (default), 1 = level barriers
ENGINES = [dict(engine=0), dict(engine=0, scheduler=1), dict(engine=1)]
EIDS = ["units-df", "units-lvl", "lane"]
# the engines running the 32-bit sweep (rebase, u16 delay table, long-delay fallback)
SWEEP = ENGINES[:2]
SIDS = EIDS[:2]
# engine 2 = the paper's CSRP pages + Alg. 1 (A/B baseline), small page lengths included
CSRP = [dict(engine=2), dict(engine=2, csrp_pagelen=2), dict(engine=2, csrp_pagelen=7)]
CIDS = ["csrp256", "csrp2", "csrp7"]


def run_gpu(c, nl, st, dur, **cfg):
    c.gls_set_config(**cfg)
    c.load(nl)
    c.gls_set_input_waveforms(nl.num_inputs, st.offsets, st.trans)
    c.gls_simulate(dur)
    return c.gls_get_waveforms(), c.gls_get_stats()


def assert_same(c, nl, st, dur, ref=None, hashes=True, **cfg):
    ref = ref or run_oracle(nl, st, dur)
    w, s = run_gpu(c, nl, st, dur, **cfg)
    if not np.array_equal(w.offsets, ref.offsets) or not np.array_equal(w.trans, ref.trans):
        for n in range(nl.num_nets):
            if w.wave(n) != ref.wave(n):
                raise AssertionError(f"net {n} differs: gpu {w.wave(n)[:20]} oracle {ref.wave(n)[:20]}")
        raise AssertionError("csr differs")
    assert s["gate_evals"] == ref.gate_evals
    assert s["events"] == ref.events
    assert s["out_transitions"] == ref.out_trans
    if hashes:
        assert np.array_equal(c.gls_get_net_hashes(), ref.hashes)
    return s


@pytest.mark.parametrize("engine", ENGINES, ids=EIDS)
@pytest.mark.parametrize("ex", golden_io.examples(), ids=lambda e: e.name)
def test_worked_examples(ctx, ex, engine):
    nl, st, dur, index, exp = ex.build()
    w, _ = run_gpu(ctx, nl, st, dur, **engine)
    for net, wave in exp.items():
        assert w.wave(net) == wave, (ex.name, nl.names[net])
    assert_same(ctx, nl, st, dur, **engine)


@pytest.mark.parametrize("engine", ENGINES, ids=EIDS)
def test_random_designs_1000(ctx, engine):
    """SPEC-style acceptance: >= 1000 random designs."""
    rng = np.random.Generator(np.random.PCG64(2024))
    for d in range(1000):
        P = int(rng.integers(1, 12))
        G = int(rng.integers(1, 120))
        nl = W.random_dag(10_000 + d, P, G, max_delay=int(rng.integers(0, 15)))
        st = W.random_stimuli(d, P, int(rng.integers(0, 40)), 400, xz=float(rng.random() * 0.3),
                              max_gap=int(rng.integers(1, 30)))
        try:
            assert_same(ctx, nl, st, 450, hashes=(d % 10 == 0), **engine)
        except AssertionError as e:
            raise AssertionError(f"design {d}: {e}")


@pytest.mark.parametrize("engine", ENGINES, ids=EIDS)
@pytest.mark.parametrize("M", [1, 2, 3, 5, 17, 300])
def test_small_chunks_exact(ctx, M, engine):
    """Many (gate, time-chunk) items per gate: halo starts, chunk value-before
    and cross-chunk cursors all exercised."""
    for seed in range(15):
        nl = W.random_dag(500 + seed, 6, 80, max_delay=20)
        st = W.random_stimuli(seed, 6, 60, 3000, xz=0.1, max_gap=60)
        assert_same(ctx, nl, st, 3100, chunk_events=M, hashes=False, **engine)


@pytest.mark.parametrize("ring", [1, 2, 3])
def test_deep_backtrace_path(ctx, ring):
    """Pending-schedule ring overflow -> exact deep path (reading R13), per-lane engine."""
    deep = 0
    for seed in range(12):
        nl = W.random_dag(700 + seed, 5, 60, max_delay=40)
        st = W.random_stimuli(seed, 5, 80, 800, xz=0.2, max_gap=4)
        s = assert_same(ctx, nl, st, 900, ring_limit=ring, chunk_events=int(8 + seed), hashes=False, engine=1)
        deep += s["deep_chunks"]
    assert deep > 0


@pytest.mark.parametrize("engine", ENGINES, ids=EIDS)
def test_zero_and_huge_delays(ctx, engine):
    for seed in range(10):
        nl = W.random_dag(800 + seed, 4, 50, max_delay=0)
        st = W.random_stimuli(seed, 4, 30, 200, xz=0.3)
        assert_same(ctx, nl, st, 250, hashes=False, **engine)
    nl = W.random_dag(900, 4, 40, max_delay=10)
    nl.pin_delay[::3] = (1 << 31) - 1
    st = W.random_stimuli(9, 4, 30, 200)
    assert_same(ctx, nl, st, 250, **engine)
    assert_same(ctx, nl, st, (1 << 33), **engine)


@pytest.mark.parametrize("engine", ENGINES, ids=EIDS)
def test_large_times(ctx, engine):
    base = 1 << 59
    nl = W.random_dag(901, 3, 30, max_delay=50)
    waves = [[(base + 10 * j + p, (j + p) % 2) for j in range(20)] for p in range(3)]
    st = W.stimuli_from_lists(waves)
    assert_same(ctx, nl, st, (1 << 61) - 1, **engine)
    # sparse, far-apart transitions: tiles limited by the 2^28 ps key span
    waves = [[(j * (1 << 29) + 7 * p, (j + p) % 2) for j in range(12)] for p in range(3)]
    assert_same(ctx, nl, W.stimuli_from_lists(waves), 13 * (1 << 29), **engine)


@pytest.mark.parametrize("engine", SWEEP, ids=SIDS)
@pytest.mark.parametrize("lo,hi", [(5000, 5200), (0, 1000), (60000, 70000)])
def test_delay_spread_paths(ctx, lo, hi, engine):
    """Delays below 2^16 take the 32-bit sweep (u16 delay table), larger ones the per-lane
    ring engine (fallback units); both with large and small per-gate spreads."""
    for seed in range(3):
        nl = W.random_dag(970 + seed, 5, 60, max_delay=hi, min_delay=lo)
        st = W.random_stimuli(seed, 5, 60, 40 * hi + 400, xz=0.2, max_gap=hi // 3 + 5)
        assert_same(ctx, nl, st, 40 * hi + 500, chunk_events=int(7 + 5 * seed), **engine)


@pytest.mark.parametrize("engine", SWEEP, ids=SIDS)
@pytest.mark.parametrize("seed", range(4))
def test_rebase_boundaries(ctx, seed, engine):
    """Glitch-dense bursts straddling multiples of 2^29 ps: the 32-bit sweep moves its
    time base there (gls_lanes.cuh) with schedules pending across the move."""
    rng = np.random.Generator(np.random.PCG64(4000 + seed))
    nl = W.random_dag(950 + seed, 4, 40, max_delay=30)
    waves = []
    for p in range(4):
        ts = set()
        for k in range(1, 9):
            c = k * (1 << 29) + int(rng.integers(-60, 60))
            ts.update(int(x) for x in c + rng.integers(-40, 40, size=6))
        w, prev = [], 2
        for t in sorted(ts):
            v = int(rng.choice([x for x in range(4) if x != prev and not (not w and x == 2)]))
            w.append((t, v))
            prev = v
        waves.append(w)
    st = W.stimuli_from_lists(waves)
    assert_same(ctx, nl, st, 9 * (1 << 29), chunk_events=int(rng.integers(3, 40)), **engine)


@pytest.mark.parametrize("engine", ENGINES, ids=EIDS)
def test_empty_and_constant_inputs(ctx, engine):
    nl = W.random_dag(902, 4, 30, max_delay=5)
    st = W.stimuli_from_lists([[], [], [], []])
    assert_same(ctx, nl, st, 100, **engine)
    st = W.stimuli_from_lists([[(0, 1)], [], [(5, 3)], [(0, 0), (7, 2)]])
    assert_same(ctx, nl, st, 100, **engine)
    # PIs only
    nl0 = W.netlist_from_gates(2, [])
    st0 = W.stimuli_from_lists([[(1, 0)], [(2, 3), (4, 1)]])
    w, s = run_gpu(ctx, nl0, st0, 10)
    assert w.wave(1) == [(2, 3), (4, 1)] and s["gate_evals"] == 0


@pytest.mark.parametrize("engine", ENGINES, ids=EIDS)
def test_c7552_shaped(ctx, engine):
    nl = W.config_netlist("c7552")
    spec = W.config_stimspec("c7552")
    o, t = W.generate_stimuli(spec)
    st = W.Stimuli(o.numpy(), t.numpy().astype(np.uint64))
    s = assert_same(ctx, nl, st, spec.duration, **engine)
    assert s["gate_evals"] > 1_000_000


def test_determinism_and_launch_shapes(ctx):
    nl = W.recipe_netlist(5, 3000, 30, 200, shuffle=True)
    spec = W.make_stimspec(5, 200, 300, "skewed", mean_trans=40, wcv=5.0)
    o, t = W.generate_stimuli(spec)
    st = W.Stimuli(o.numpy(), t.numpy().astype(np.uint64))
    ref = run_oracle(nl, st, spec.duration)
    base = None
    for cfg in [dict(), dict(blocks_per_sm=1), dict(chunk_events=32), dict(chunk_events=4096), dict(engine=1),
                dict(engine=1, chunk_events=64), dict(chunk_events=7), dict(chunk_events=64, blocks_per_sm=1),
                dict(scheduler=1), dict(scheduler=1, chunk_events=64), dict(deep_per_warp=64), dict()]:
        w, _ = run_gpu(ctx, nl, st, spec.duration, **cfg)
        assert np.array_equal(w.trans, ref.trans)
        if base is None:
            base = w.trans.copy()
        assert np.array_equal(base, w.trans)


def test_device_inputs_and_resimulation(ctx):
    nl = W.random_dag(903, 5, 100, max_delay=9)
    ctx.gls_set_config()
    ctx.load(nl)
    for seed in range(3):
        st = W.random_stimuli(seed, 5, 50, 1000)
        ref = run_oracle(nl, st, 1100)
        d_off = torch.as_tensor(st.offsets, device="cuda")
        d_tr = torch.as_tensor(st.trans.astype(np.int64), device="cuda")
        ctx.gls_set_input_waveforms_device(5, d_off.data_ptr(), d_tr.data_ptr(), st.total)
        ctx.gls_simulate(1100)
        w = ctx.gls_get_waveforms()
        assert np.array_equal(w.trans, ref.trans)
        d_h = torch.zeros(nl.num_nets, dtype=torch.int64, device="cuda")
        ctx.gls_get_net_hashes_device(d_h.data_ptr())
        assert np.array_equal(d_h.cpu().numpy().astype(np.uint64), ref.hashes)
        cnt = ctx.gls_get_net_counts()
        assert np.array_equal(cnt, np.diff(ref.offsets))


def test_error_codes(ctx):
    ok = W.random_dag(904, 2, 5)
    with pytest.raises(gls.GlsError) as e:   # cycle
        ctx.load(W.netlist_from_gates(1, [(W.AND, [0, 2], [(1,) * 4] * 2), (W.BUF, [1], [(1,) * 4])]))
    assert e.value.code == gls.GLS_ECYCLE
    for bad in [
        W.netlist_from_gates(1, [(9, [0], [(1,) * 4])]),                        # unknown type
        W.netlist_from_gates(1, [(W.AND, [0], [(1,) * 4])]),                    # arity
        W.netlist_from_gates(1, [(W.BUF, [5], [(1,) * 4])]),                    # net id
        W.netlist_from_gates(1, [(W.BUF, [0], [(1 << 31, 0, 0, 0)])]),          # delay
    ]:
        with pytest.raises(gls.GlsError) as e:
            ctx.load(bad)
        assert e.value.code == gls.GLS_EINVAL
    ctx.load(ok)
    with pytest.raises(gls.GlsError) as e:
        ctx.gls_simulate(10)
    assert e.value.code == gls.GLS_ESTATE
    for waves in ([[(5, 1), (5, 0)], []], [[(1, 1), (2, 1)], []], [[(1, 2)], []]):
        st = W.stimuli_from_lists(waves)
        with pytest.raises(gls.GlsError) as e:
            ctx.gls_set_input_waveforms(2, st.offsets, st.trans)
        assert e.value.code == gls.GLS_EINVAL
    # violations deep inside long waveforms (another lane / loop trip of the validator),
    # through the host and the device path
    good = [(10 * (j + 1), j % 2) for j in range(200)]
    for pos, kind in [(77, "time"), (150, "value"), (33, "time"), (199, "value")]:
        w = list(good)
        if kind == "time":
            w[pos] = (w[pos - 1][0], w[pos][1])
        else:
            w[pos] = (w[pos][0], w[pos - 1][1])
            w[pos + 1:] = [(t, 1 - v) for t, v in w[pos + 1:]]
        st = W.stimuli_from_lists([good, w])
        with pytest.raises(gls.GlsError) as e:
            ctx.gls_set_input_waveforms(2, st.offsets, st.trans)
        assert e.value.code == gls.GLS_EINVAL, (pos, kind)
        d_off = torch.as_tensor(st.offsets, device="cuda")
        d_tr = torch.as_tensor(st.trans.astype(np.int64), device="cuda")
        with pytest.raises(gls.GlsError) as e:
            ctx.gls_set_input_waveforms_device(2, d_off.data_ptr(), d_tr.data_ptr(), st.total)
        assert e.value.code == gls.GLS_EINVAL, (pos, kind)
    st = W.stimuli_from_lists([good, good[:150]])
    ctx.gls_set_input_waveforms(2, st.offsets, st.trans)           # valid long waveforms pass
    st = W.stimuli_from_lists([[(50, 1)], []])
    ctx.gls_set_input_waveforms(2, st.offsets, st.trans)
    with pytest.raises(gls.GlsError) as e:
        ctx.gls_simulate(40)
    assert e.value.code == gls.GLS_ERANGE
    ctx.gls_simulate(60)
    assert ctx.gls_get_halo() >= 1


def test_arena_too_small_reports_enomem():
    nl = W.random_dag(905, 4, 200, max_delay=5)
    st = W.random_stimuli(1, 4, 200, 5000)
    with gls.Context(0) as c:
        c.gls_set_config(arena_bytes=8 * (st.total + 16))
        c.load(nl)
        c.gls_set_input_waveforms(4, st.offsets, st.trans)
        with pytest.raises(gls.GlsError) as e:
            c.gls_simulate(6000)
        assert e.value.code == gls.GLS_ENOMEM and "arena" in str(e.value)


def test_generator_cpu_equals_gpu():
    spec = W.make_stimspec(3, 300, 500, "skewed", mean_trans=30, wcv=4.0)
    o1, t1 = W.generate_stimuli(spec, "cpu")
    o2, t2 = W.generate_stimuli(spec, "cuda")
    assert torch.equal(o1, o2.cpu()) and torch.equal(t1, t2.cpu())


@pytest.mark.parametrize("seed", range(6))
def test_deep_pending_and_scratch_overflow(ctx, seed):
    """Large delay spreads with dense events: long pending lists (the Eq. 1 stack; the
    per-lane engine's ring -> deep path); long single-chunk gates overflow the lane
    scratch (-> fallback units)."""
    nl = W.random_dag(1200 + seed, 4, 40, max_delay=400, min_delay=0)
    st = W.random_stimuli(seed, 4, 600, 3000, xz=0.05, min_gap=1, max_gap=3)
    for eng in (0, 1):
        for sch in (0, 1):
            assert_same(ctx, nl, st, 4000, engine=eng, scheduler=sch, chunk_events=1 << 20, hashes=False)
    nl = W.random_dag(1300 + seed, 3, 30, max_delay=2, types=[W.BUF, W.NOT, W.XOR])
    st = W.random_stimuli(seed, 3, 3000, 60000, xz=0.0, min_gap=5, max_gap=30)
    for eng in (0, 1):
        for sch in (0, 1):
            assert_same(ctx, nl, st, 61000, engine=eng, scheduler=sch, chunk_events=1 << 20, hashes=False)


@pytest.mark.parametrize("engine", ENGINES, ids=EIDS)
def test_simulate_window_matches_full_run(ctx, engine):
    """gls_simulate_window (reading R17 inside the library): on [t_begin, t_end) the
    window run's transitions equal the full run's (oracle), for windows at the start,
    inside, across chunk boundaries and at the end, in any order; a later plain
    gls_simulate runs the full inputs again."""
    from winhash import window_hash
    for seed in range(4):
        nl = W.recipe_netlist(70 + seed, 900, 15, 60)
        spec = W.make_stimspec(70 + seed, 60, 400, "skewed", mean_trans=60, wcv=3.0)
        o, t = W.generate_stimuli(spec)
        st = W.to_stimuli(o, t)
        dur = spec.duration
        ref = run_oracle(nl, st, dur)
        ctx.gls_set_config(chunk_events=64 if seed % 2 else 0, **engine)
        ctx.load(nl)
        ctx.gls_set_input_waveforms(nl.num_inputs, st.offsets, st.trans)
        for t0, t1 in [(2_000_000, 2_500_000), (0, 300_000), (1_234_567, 3_000_001), (dur - 77_777, dur + 1),
                       (1_000_000, 1_000_000)]:
            ctx.gls_simulate_window(t0, t1, dur)
            if t1 == t0:                                            # empty window: nothing promised
                continue
            got = ctx.gls_get_net_hashes_window(t0, t1 - 1)
            assert np.array_equal(got, window_hash(ref.offsets, ref.trans, t0, t1 - 1)), (seed, t0, t1)
        ctx.gls_simulate(dur)                                       # the full inputs again
        assert np.array_equal(ctx.gls_get_waveforms().trans, ref.trans)
        with pytest.raises(gls.GlsError) as e:
            ctx.gls_simulate_window(10, 5, dur)
        assert e.value.code == gls.GLS_EINVAL


@pytest.mark.parametrize("windows", [2, 3, 5])
def test_window_stitch_matches_full_run(ctx, windows):
    """Time-window stitching through the device ABI (gls_get_net_hash_terms_device +
    shard's combination): windows simulated one after the other as the ranks would,
    counts first, then the terms keyed from the exclusive prefix of the counts, XOR =
    the oracle's full-run per-net checksums."""
    nl = W.recipe_netlist(91, 1200, 18, 80)
    spec = W.make_stimspec(91, 80, 300, "skewed", mean_trans=50, wcv=3.0)
    o, t = W.generate_stimuli(spec)
    st = W.to_stimuli(o, t)
    dur = spec.duration
    ref = run_oracle(nl, st, dur)
    ctx.gls_set_config(chunk_events=96)
    ctx.load(nl)
    ctx.gls_set_input_waveforms(nl.num_inputs, st.offsets, st.trans)
    n = nl.num_nets
    dev = torch.device("cuda", 0)
    cuts = [dur * k // windows for k in range(windows)] + [dur + 1]
    counts = []
    for a, b in zip(cuts, cuts[1:]):
        ctx.gls_simulate_window(a, b, dur)
        c = torch.empty(n, dtype=torch.int64, device=dev)
        ctx.gls_get_net_hash_terms_device(a, b - 1, 0, 0, c.data_ptr(), 0)
        counts.append(c)
    total = torch.stack(counts).sum(0)
    base = torch.zeros(n, dtype=torch.int64, device=dev)
    h = torch.zeros(n, dtype=torch.int64, device=dev)
    for k, (a, b) in enumerate(zip(cuts, cuts[1:])):
        ctx.gls_simulate_window(a, b, dur)
        tt = torch.empty(n, dtype=torch.int64, device=dev)
        scratch = torch.empty(n, dtype=torch.int64, device=dev)
        ctx.gls_get_net_hash_terms_device(a, b - 1, base.data_ptr(), total.data_ptr() if k == 0 else 0,
                                          scratch.data_ptr(), tt.data_ptr())
        assert torch.equal(scratch, counts[k])
        h.bitwise_xor_(tt)
        base += counts[k]
    assert np.array_equal(h.cpu().numpy().view(np.uint64), ref.hashes)
    assert np.array_equal(total.cpu().numpy(), np.diff(ref.offsets))


def test_window_stitch_over_nccl_single_rank(ctx):
    """shard.gls_window_stitch end to end over a (one-rank) NCCL process group: the
    stitched checksums of a run owning [0, duration] are the run's own."""
    import os
    import socket
    import torch.distributed as dist
    from paper_2304_13398_b200 import shard
    nl = W.recipe_netlist(93, 800, 12, 50)
    spec = W.make_stimspec(93, 50, 200, "random")
    o, t = W.generate_stimuli(spec)
    st = W.to_stimuli(o, t)
    ctx.gls_set_config()
    ctx.load(nl)
    ctx.gls_set_input_waveforms(nl.num_inputs, st.offsets, st.trans)
    ctx.gls_simulate(spec.duration)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        h = shard.gls_window_stitch(ctx, 0, spec.duration, dev)
        torch.cuda.synchronize(dev)
    finally:
        dist.destroy_process_group()
    assert np.array_equal(h.cpu().numpy().view(np.uint64), ctx.gls_get_net_hashes())


@pytest.mark.parametrize("engine", CSRP, ids=CIDS)
def test_csrp_engine_parity(ctx, engine):
    """NEXT-3: the paper's design on the GPU — CSRP pages, next-page pointers, terminate
    markers, an atomic page iterator (§3.1) and Alg. 1's static one-thread-
    per-cell assignment — bit-exact against the oracle, with Eq. 4's waste bound
    M_w <= pagelen * k * M_t on the page slots."""
    rng = np.random.Generator(np.random.PCG64(77))
    for d in range(120):
        P = int(rng.integers(1, 10))
        nl = W.random_dag(20_000 + d, P, int(rng.integers(1, 150)), max_delay=int(rng.integers(0, 15)))
        st = W.random_stimuli(d, P, int(rng.integers(0, 60)), 400, xz=float(rng.random() * 0.3),
                              max_gap=int(rng.integers(1, 30)))
        s = assert_same(ctx, nl, st, 450, hashes=(d % 10 == 0), **engine)
        L = engine.get("csrp_pagelen", 256)
        k = nl.num_nets
        assert 0 <= s["csrp_waste"] <= L * k
        assert s["csrp_pages"] >= k
    for ex in golden_io.examples():
        nl, st, dur, index, exp = ex.build()
        w, _ = run_gpu(ctx, nl, st, dur, **engine)
        for net, wave in exp.items():
            assert w.wave(net) == wave, (ex.name, nl.names[net])


def test_csrp_engine_c7552_and_cells(ctx):
    nl = W.config_netlist("c7552")
    spec = W.config_stimspec("c7552")
    o, t = W.generate_stimuli(spec)
    st = W.Stimuli(o.numpy(), t.numpy().astype(np.uint64))
    assert_same(ctx, nl, st, spec.duration, engine=2)
    tpl, ct, cf, cd = W.random_cells(91, 6, 120, max_delay=12, p_inf=0.2)
    st = W.random_stimuli(91, 6, 80, 2000, xz=0.1)
    ref = oracle.simulate_cells(6, tpl, ct, cf, cd, st.offsets, st.trans, 2100)
    ctx.gls_set_config(engine=2)
    ctx.gls_load_cells(6, tpl, ct, cf, cd)
    ctx.gls_set_input_waveforms(6, st.offsets, st.trans)
    ctx.gls_simulate(2100)
    w = ctx.gls_get_waveforms()
    assert np.array_equal(w.offsets, ref.offsets) and np.array_equal(w.trans, ref.trans)


def test_deep_scratch_retry_on_fresh_context():
    """kErrDeep grow-and-retry: a fresh context with a 1-entry deep scratch per warp and a
    1-entry pending ring (per-lane engine) must overflow the deep scratch, grow it and
    still return the oracle's result; deep_per_warp set after a first run takes effect."""
    nl = W.random_dag(1400, 5, 60, max_delay=40)
    st = W.random_stimuli(3, 5, 80, 800, xz=0.2, max_gap=4)
    ref = run_oracle(nl, st, 900)
    with gls.Context(0) as c:
        s = assert_same(c, nl, st, 900, ref=ref, engine=1, ring_limit=1, chunk_events=9, deep_per_warp=1)
        assert s["deep_chunks"] > 0
        s = assert_same(c, nl, st, 900, ref=ref, engine=0, deep_per_warp=1)
        s = assert_same(c, nl, st, 900, ref=ref, engine=1, ring_limit=1, chunk_events=9, deep_per_warp=2)


def test_auto_arena_regrow():
    """Auto-sized transition store (arena_bytes = 0) smaller than the result: an XOR ladder
    (net k = XOR(net k-2, net k-1)) whose activity grows along the chain outruns the size
    estimate; the kernel aborts, the store grows (given waveforms kept) and the retried run
    equals the oracle."""
    G = 30
    nl = W.netlist_from_gates(2, [(W.XOR, [g, g + 1], [(1, 1, 1, 1)] * 2) for g in range(G)])
    waves = [[(97 * j + 3, j % 2) for j in range(1, 300)], [(131 * j + 5, j % 2) for j in range(1, 200)]]
    st = W.stimuli_from_lists(waves)
    ref = run_oracle(nl, st, 100000)
    est = st.total + 3 * G * (st.total // 2) + 4096   # gls_api.cu ensure_arena's auto estimate
    assert ref.out_trans > est                        # so the retry path runs
    with gls.Context(0) as c:
        for eng in (0, 1, 2):
            assert_same(c, nl, st, 100000, ref=ref, engine=eng)
