import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2304_13398_b200 import gls, workloads as W
c = gls.Context(0)
def run(nl, st, dur, **cfg):
    c.gls_set_config(**cfg); c.load(nl); c.gls_set_input_waveforms(nl.num_inputs, st.offsets, st.trans); c.gls_simulate(dur)
    s = c.gls_get_stats(); return s
for k, t in [(1, W.BUF), (2, W.AND), (2, W.XOR), (4, W.XOR)]:
    waves = [[(10 * j + p, (j + p) % 2) for j in range(4000)] for p in range(k)]
    nl = W.netlist_from_gates(k, [(t, list(range(k)), [(3, 3, 3, 3)] * k)])
    for M in (4096, 1 << 20):
        s = run(nl, W.stimuli_from_lists(waves), 50000, chunk_events=M)
        print(k, W.TYPE_NAMES[t], M, 'util %.2f' % s['lane_utilization'], 'chunks', s['chunks'], 'fallback', s['deep_chunks'], 'evals', s['gate_evals'])
