"""Full-size parity (-m gpu): the bench's workload (BASELINE configs[1] = c4_10m, 10,485,760
gates, 297,203 cycles) simulated once through the C-ABI in the launch configuration
bench.py times (library defaults), then checked bit-exactly against the oracle on sampled
time windows at the start, middle and end of the run.  Each window's oracle run starts
from the given waveforms clamped `lookback` cycles before the window (reading R17: exact
for every net on [window start, ...), pinned on CPU by
test_oracle_pins.py::test_time_window_with_halo_is_exact); only the window's transitions
enter the per-net hashes (tests/winhash.py, pinned by test_winhash.py)."""
import numpy as np
import pytest
import torch

from oracle import oracle
from paper_2304_13398_b200 import gls, shard
from paper_2304_13398_b200 import workloads as W
from winhash import window_hash

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

WINDOW_CYCLES = 150


def test_c4_full_size_sampled_windows():
    cfg = "c4_10m"
    nl = W.config_netlist(cfg, 1)
    spec = W.config_stimspec(cfg, 1)
    dev = torch.device("cuda", 0)
    ctx = gls.Context(0, torch.cuda.current_stream(dev).cuda_stream)
    ctx.gls_set_config()                               # the bench's launch configuration
    ctx.load(nl)
    H = ctx.gls_get_halo()
    d_off, d_tr = W.window_stimuli(spec, 0, spec.ncycles, dev)
    ctx.gls_set_input_waveforms_device(nl.num_inputs, d_off.data_ptr(), d_tr.data_ptr(), int(d_tr.numel()))
    ctx.gls_simulate(spec.duration)
    st = ctx.gls_get_stats()
    assert st["gate_evals"] > 2e10 and st["out_transitions"] > 1e10    # the full workload ran
    del d_off, d_tr
    torch.cuda.empty_cache()
    nc, look = spec.ncycles, shard.lookback_cycles(H)
    mid = nc // 2
    for c_lo, c_hi in [(0, WINDOW_CYCLES), (mid, mid + WINDOW_CYCLES), (nc - WINDOW_CYCLES, nc)]:
        o, t = W.window_stimuli(spec, max(0, c_lo - look), c_hi, "cpu")
        s = W.to_stimuli(o, t)
        last = c_hi == nc
        dur = spec.duration if last else c_hi * W.PERIOD
        r = oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay,
                            s.offsets, s.trans, dur)
        lo, hi = c_lo * W.PERIOD, (dur if last else c_hi * W.PERIOD - 1)
        ref = window_hash(r.offsets, r.trans, lo, hi)
        got = ctx.gls_get_net_hashes_window(lo, hi)
        bad = np.flatnonzero(got != ref)
        assert bad.size == 0, f"window [{lo}, {hi}] ps: {bad.size} of {got.size} nets differ (first {bad[:5]})"
        assert r.out_trans > 0
    ctx.close()
