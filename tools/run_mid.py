"""Mid-size run through the ABI (for compute-sanitizer / debugging)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2304_13398_b200 import gls, workloads as W
G = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
cyc = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
prof = sys.argv[3] if len(sys.argv) > 3 else 'skewed'
nl = W.recipe_netlist(3, G, 40, G // 10)
spec = W.make_stimspec(3, G // 10, cyc, prof, mean_trans=cyc // 8, wcv=8.0)
o, t = W.generate_stimuli(spec)
st = W.to_stimuli(o, t)
c = gls.Context(0)
c.gls_set_config(arena_bytes=1 << 30)
c.load(nl)
c.gls_set_input_waveforms(nl.num_inputs, st.offsets, st.trans)
c.gls_simulate(spec.duration)
print(c.gls_get_stats())
if len(sys.argv) > 4:
    from oracle import oracle
    r = oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay, st.offsets, st.trans, spec.duration)
    w = c.gls_get_waveforms()
    print('parity', np.array_equal(w.trans, r.trans))
