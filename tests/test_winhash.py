"""Pins for tests/winhash.py (CPU): the vectorised window hash equals the oracle's
own per-net hashes on the full window and a per-net loop on sub-windows."""
import numpy as np

from oracle import oracle
from paper_2304_13398_b200 import workloads as W
from winhash import splitmix64, window_hash


def _loop_hash(offsets, trans, lo, hi):
    M = (1 << 64) - 1

    def sm(x):
        x = (x + 0x9E3779B97F4A7C15) & M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
        return x ^ (x >> 31)
    out = []
    for n in range(len(offsets) - 1):
        es = [int(x) for x in trans[offsets[n]:offsets[n + 1]] if lo <= (int(x) >> 2) <= hi]
        h = sm(0x9E3779B97F4A7C15 ^ len(es))
        for j, x in enumerate(es):
            h ^= sm((x + (j + 1) * 0xD1B54A32D192ED03) & M)
        out.append(h)
    return np.array(out, np.uint64)


def _run():
    nl = W.recipe_netlist(7, 400, 12, 40)
    spec = W.make_stimspec(7, 40, 120, "skewed", mean_trans=30, wcv=4.0)
    o, t = W.generate_stimuli(spec)
    st = W.to_stimuli(o, t)
    r = oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay,
                        st.offsets, st.trans, spec.duration)
    return r, spec


def test_splitmix_known_value():
    # splitmix64 of 0 (the generator's first output from state 0, a published constant)
    with np.errstate(over="ignore"):
        assert int(splitmix64(np.array([0], np.uint64))[0]) == 0xE220A8397B1DCDAF


def test_full_window_equals_oracle_hashes():
    r, spec = _run()
    assert np.array_equal(window_hash(r.offsets, r.trans, 0, spec.duration), r.hashes)


def test_sub_windows_equal_loop():
    r, spec = _run()
    for lo, hi in [(0, 0), (10_000, 350_000), (600_000, spec.duration), (spec.duration + 1, spec.duration + 5)]:
        assert np.array_equal(window_hash(r.offsets, r.trans, lo, hi), _loop_hash(r.offsets, r.trans, lo, hi))


def test_window_terms_split_the_full_hash():
    """The stitching pieces over windows that tile the run XOR to the oracle's own
    full-run per-net checksums; with base 0 and total = count a single window's
    pieces are its window hash."""
    from winhash import window_terms
    nl = W.recipe_netlist(5, 300, 10, 30)
    spec = W.make_stimspec(5, 30, 80, "random")
    o, t = W.generate_stimuli(spec)
    st = W.to_stimuli(o, t)
    r = oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay,
                        st.offsets, st.trans, spec.duration)
    cuts = [0, 123_456, 400_000, 400_001, spec.duration + 1]
    cnts = [window_terms(r.offsets, r.trans, a, b - 1)[0] for a, b in zip(cuts, cuts[1:])]
    total = np.sum(cnts, axis=0)
    h = np.zeros_like(r.hashes)
    base = np.zeros_like(total)
    for k, (a, b) in enumerate(zip(cuts, cuts[1:])):
        _, tt = window_terms(r.offsets, r.trans, a, b - 1, base, total if k == 0 else None)
        h ^= tt
        base = base + cnts[k]
    assert np.array_equal(h, r.hashes)
    c, tt = window_terms(r.offsets, r.trans, 123_456, 399_999, None, cnts[1])
    assert np.array_equal(tt, window_hash(r.offsets, r.trans, 123_456, 399_999))
