"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
the worked examples (c17, full adders), the c7552-shaped design and random DAGs / cell
netlists, every engine, checked against the oracle (tools/sanitize.sh)."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import golden_io  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2304_13398_b200 import gls  # noqa: E402
from paper_2304_13398_b200 import workloads as W  # noqa: E402

ndesigns = int(sys.argv[1]) if len(sys.argv) > 1 else 40
bad = 0
with gls.Context(0) as ctx:
    for cfg in [dict(), dict(scheduler=1), dict(engine=1), dict(engine=2), dict(chunk_events=5)]:
        ctx.gls_set_config(**cfg)
        runs = [(ex.build()[:3]) for ex in golden_io.examples()]
        nl = W.config_netlist("c7552")
        spec = W.config_stimspec("c7552", ncycles=200)
        o, t = W.generate_stimuli(spec)
        runs.append((nl, W.Stimuli(o.numpy(), t.numpy().astype(np.uint64)), spec.duration))
        rng = np.random.default_rng(5)
        for d in range(ndesigns):
            P = int(rng.integers(1, 8))
            runs.append((W.random_dag(40_000 + d, P, int(rng.integers(1, 80)), max_delay=int(rng.integers(0, 12))),
                         W.random_stimuli(d, P, 40, 400, xz=0.2), 450))
        for nl, st, dur in runs:
            ctx.load(nl)
            ctx.gls_set_input_waveforms(nl.num_inputs, st.offsets, st.trans)
            ctx.gls_simulate(dur)
            w = ctx.gls_get_waveforms()
            ref = oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay,
                                  st.offsets, st.trans, dur)
            bad += int(not (np.array_equal(w.offsets, ref.offsets) and np.array_equal(w.trans, ref.trans)))
        tpl, ct, cf, cd = W.random_cells(9, 5, 60, p_inf=0.2)
        st = W.random_stimuli(9, 5, 40, 600, xz=0.1)
        ctx.gls_load_cells(5, tpl, ct, cf, cd)
        ctx.gls_set_input_waveforms(5, st.offsets, st.trans)
        ctx.gls_simulate(650)
        w = ctx.gls_get_waveforms()
        ref = oracle.simulate_cells(5, tpl, ct, cf, cd, st.offsets, st.trans, 650)
        bad += int(not np.array_equal(w.trans, ref.trans))
print(f"sanitize_run: {bad} mismatching runs")
sys.exit(1 if bad else 0)
