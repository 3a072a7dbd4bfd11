"""Offline analysis: how balanced are ref-quantile slices on a workload's gates?"""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from oracle import oracle
from paper_2304_13398_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else 'c4_mini'
cyc = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
nl = W.config_netlist(cfg, 1)
spec = W.config_stimspec(cfg, 1)
o, t = W.window_stimuli(spec, 0, cyc, 'cpu')
st = W.to_stimuli(o, t)
t0 = time.time()
r = oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay,
                    st.offsets, st.trans, cyc * W.PERIOD)
print('oracle', time.time() - t0, 's, gate-evals', r.gate_evals)
times = lambda n: (r.trans[r.offsets[n]:r.offsets[n + 1]] >> np.uint64(2)).astype(np.int64)
rng = np.random.default_rng(0)
ratios, ratios_cb, weights = [], [], []
P = nl.num_inputs
for g in rng.choice(nl.num_gates, 20000, replace=False):
    fin = nl.fanin_net[nl.fanin_offsets[g]:nl.fanin_offsets[g + 1]]
    ts = [times(s) for s in fin]
    n_in = sum(len(x) for x in ts)
    if n_in < 1024:
        continue
    ref = max(range(len(ts)), key=lambda i: len(ts[i]))
    L = len(ts[ref])
    allt = np.sort(np.concatenate(ts))
    # 32 ref-quantile slices
    b = [ts[ref][(L * s) // 32] for s in range(1, 32)]
    cnt = np.diff(np.concatenate([[0], np.searchsorted(allt, b), [len(allt)]]))
    ratios.append(cnt.max() / cnt.mean())
    weights.append(n_in)
print('gates with n_in >= 1024:', len(ratios))
w = np.array(weights)
print('ref-quantile slices: max/mean weighted %.2f  (median %.2f, p90 %.2f)' % (
    np.average(ratios, weights=w), np.median(ratios), np.percentile(ratios, 90)))
