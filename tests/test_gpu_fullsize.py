"""Full-size parity (-m gpu) on the bench's configurations, through the C-ABI in the
launch configuration bench.py times (library defaults):

  * C4 (BASELINE configs[3], c4_10m: 10,485,760 gates, 297,203 cycles) — 16 windows spread
    over the whole run, together >= 10 % of it;
  * C3 (configs[2], c3_1m: 1,048,576 gates, 19,999 cycles) — 16 windows, >= 10 %;
  * C5 (configs[4]: the C3 netlist x 64 stimulus sets) — every one of the 64 sets, a
    window of each (at a different place in each set).

The GPU simulates the whole run once per workload; the oracle (oracle/, single-threaded
C) runs each window from the given waveforms clamped `lookback` cycles before it
(reading R17: exact for every net on [window start, ...), pinned on CPU by
test_oracle_pins.py::test_time_window_with_halo_is_exact), the windows in parallel on
the host's cores (ctypes releases the GIL).  Only each window's transitions enter the
compared per-net hashes (tests/winhash.py, pinned by test_winhash.py)."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from oracle import oracle
from paper_2304_13398_b200 import gls, shard
from paper_2304_13398_b200 import workloads as W
from winhash import window_hash

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
DEV = torch.device("cuda", 0)
WORKERS = max(1, min(16, (os.cpu_count() or 2) - 1))


def _oracle_window(nl, spec, H, c_lo, c_hi):
    """Oracle window hashes: the run of the clamped stimuli, hashed on [c_lo, c_hi) cycles."""
    look = shard.lookback_cycles(H)
    o, t = W.window_stimuli(spec, max(0, c_lo - look), c_hi, "cpu")
    s = W.to_stimuli(o, t)
    last = c_hi == spec.ncycles
    dur = spec.duration if last else c_hi * W.PERIOD
    lo, hi = c_lo * W.PERIOD, (dur if last else c_hi * W.PERIOD - 1)
    return s, dur, lo, hi


def _run_oracle(nl, s, dur, lo, hi):
    r = oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay,
                        s.offsets, s.trans, dur)
    return window_hash(r.offsets, r.trans, lo, hi), r.out_trans


def _check_windows(ctx, nl, spec, H, windows):
    """Oracle on every window (in parallel), the GPU's window hashes against them."""
    jobs = []
    with ThreadPoolExecutor(WORKERS) as pool:
        for c_lo, c_hi in windows:
            s, dur, lo, hi = _oracle_window(nl, spec, H, c_lo, c_hi)
            jobs.append((lo, hi, pool.submit(_run_oracle, nl, s, dur, lo, hi)))
        for lo, hi, f in jobs:
            ref, outs = f.result()
            got = ctx.gls_get_net_hashes_window(lo, hi)
            bad = np.flatnonzero(got != ref)
            assert bad.size == 0, f"window [{lo}, {hi}] ps: {bad.size} of {got.size} nets differ (first {bad[:5]})"
            assert outs > 0


def _spread(ncycles, n, frac):
    """n windows spread over [0, ncycles), covering `frac` of the cycles, the last ending at the end."""
    w = max(1, int(np.ceil(frac * ncycles / n)))
    starts = [i * (ncycles - w) // (n - 1) for i in range(n)]
    return [(a, a + w) for a in starts]


def _load_full(cfg, seed=1):
    nl = W.config_netlist(cfg, seed)
    ctx = gls.Context(0, torch.cuda.current_stream(DEV).cuda_stream)
    ctx.gls_set_config()                               # the bench's launch configuration
    ctx.load(nl)
    return nl, ctx


@pytest.mark.parametrize("cfg", ["c4_10m", "c3_1m"])
def test_full_size_windows_cover_ten_percent(cfg):
    nl, ctx = _load_full(cfg)
    spec = W.config_stimspec(cfg, 1)
    H = ctx.gls_get_halo()
    d_off, d_tr = W.window_stimuli(spec, 0, spec.ncycles, DEV)
    torch.cuda.empty_cache()
    ctx.gls_set_input_waveforms_device(nl.num_inputs, d_off.data_ptr(), d_tr.data_ptr(), int(d_tr.numel()))
    ctx.gls_simulate(spec.duration)
    st = ctx.gls_get_stats()
    assert st["gate_evals"] > 2e10 and st["out_transitions"] > 5e9    # the full workload ran
    del d_off, d_tr
    torch.cuda.empty_cache()
    windows = _spread(spec.ncycles, 16, 0.10)
    assert sum(b - a for a, b in windows) >= 0.10 * spec.ncycles
    assert windows[0][0] == 0 and windows[-1][1] == spec.ncycles
    _check_windows(ctx, nl, spec, H, windows)
    ctx.close()


def test_c5_all_sets():
    """C5: the 64 stimulus sets of the bench (seeds 1..64 on the C3 netlist), each
    simulated in full on the GPU and checked on a window at a set-dependent place."""
    cfg = "c5_set"
    nl, ctx = _load_full(cfg)
    H = ctx.gls_get_halo()
    sets = 64
    jobs = []
    with ThreadPoolExecutor(WORKERS) as pool:
        for k in range(sets):
            spec = W.config_stimspec(cfg, 1 + k)
            d_off, d_tr = W.window_stimuli(spec, 0, spec.ncycles, DEV)
            ctx.gls_set_input_waveforms_device(nl.num_inputs, d_off.data_ptr(), d_tr.data_ptr(), int(d_tr.numel()))
            ctx.gls_simulate(spec.duration)
            w = 100
            c_lo = (k * 37) % (spec.ncycles - w) if k != sets - 1 else spec.ncycles - w
            s, dur, lo, hi = _oracle_window(nl, spec, H, c_lo, c_lo + w)
            got = ctx.gls_get_net_hashes_window(lo, hi)
            jobs.append((k, lo, hi, got, pool.submit(_run_oracle, nl, s, dur, lo, hi)))
        for k, lo, hi, got, f in jobs:
            ref, outs = f.result()
            bad = np.flatnonzero(got != ref)
            assert bad.size == 0, f"set {k} window [{lo}, {hi}]: {bad.size} nets differ (first {bad[:5]})"
    ctx.close()
