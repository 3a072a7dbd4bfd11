#!/usr/bin/env python
"""Scheduling trace of one simulation (gls_config.trace): when each topological level's
gates were planned / completed, and how long their chunks took.

    python tools/trace_report.py [config] [seed]
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2304_13398_b200 import gls, workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4_mini"
dev = torch.device("cuda", 0)
nl = W.config_netlist(cfg, 1)
spec = W.config_stimspec(cfg, 1)
ctx = gls.Context(0, torch.cuda.current_stream(dev).cuda_stream)
ctx.load(nl)
d_off, d_tr = W.window_stimuli(spec, 0, spec.ncycles, dev)
torch.cuda.empty_cache()
ctx.gls_set_input_waveforms_device(nl.num_inputs, d_off.data_ptr(), d_tr.data_ptr(), int(d_tr.numel()))
ctx.gls_set_config(trace=1)
ctx.gls_simulate(spec.duration)
ctx.gls_simulate(spec.duration)
s = ctx.gls_get_stats()
tr = ctx.gls_get_trace().astype(np.float64)
# levels (recipe netlists are in topological order)
P, G = nl.num_inputs, nl.num_gates
lev = np.zeros(P + G, np.int64)
for g in range(G):
    a, b = nl.fanin_offsets[g], nl.fanin_offsets[g + 1]
    lev[P + g] = 1 + lev[nl.fanin_net[a:b]].max()
glev = lev[P:]
t0 = tr[:, 0][tr[:, 0] > 0].min()
plan, done = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3          # us
csum = tr[:, 2] / 1e3
cmax = tr[:, 3] / 1e3
crounds, cunits, cmaxit, cmaxsu = (tr[:, q].astype(np.int64) for q in (4, 5, 6, 7))
n_in = np.zeros(G)
counts = ctx.gls_get_net_counts()
for g in range(G):
    a, b = nl.fanin_offsets[g], nl.fanin_offsets[g + 1]
    n_in[g] = counts[nl.fanin_net[a:b]].sum()
print(json.dumps({"config": cfg, "kernel_ms": s["kernel_ms"], "gates": G, "levels": int(glev.max())}))
print(f"{'lvl':>4} {'gates':>7} {'plan p50':>9} {'plan max':>9} {'done p50':>9} {'done max':>9} "
      f"{'chunk us p50':>12} {'p99':>8} {'max':>8} {'n_in p50':>9} {'n_in max':>9}")
L = int(glev.max())
for l in list(range(1, min(L, 12) + 1)) + list(range(15, L + 1, max(1, L // 20))):
    m = glev == l
    if not m.any():
        continue
    print(f"{l:4d} {m.sum():7d} {np.median(plan[m]):9.0f} {plan[m].max():9.0f} {np.median(done[m]):9.0f} "
          f"{done[m].max():9.0f} {np.median(cmax[m]):12.1f} {np.percentile(cmax[m], 99):8.1f} {cmax[m].max():8.1f} "
          f"{np.median(n_in[m]):9.0f} {n_in[m].max():9.0f}")
busy = csum.sum() / 1e3
print(f"sum of chunk durations {busy:.0f} ms over {3552} warps -> {busy / 3552:.1f} ms per warp "
      f"(kernel {s['kernel_ms']:.1f} ms)")
# the gates whose plan time is latest relative to their own level's median: dependency stalls
slow = np.argsort(-cmax)[:10]
for g in slow:
    print(f"slowest chunk: gate {g} level {glev[g]} n_in {n_in[g]:.0f} max chunk {cmax[g]:.0f} us, "
          f"sum {csum[g]:.0f} us, planned {plan[g]:.0f} us, done {done[g]:.0f} us, batch rounds {crounds[g]} "
          f"units {cunits[g]} busiest lane {cmaxit[g]} iterations, most set-ups {cmaxsu[g]}")
# critical path: from the last gate to complete, walk back through the fan-in gate that
# completed last (the one whose completion planned it); per step: wait (plan - that
# fan-in's done) and run (done - plan) of the gate
g = int(np.argmax(done))
path = []
while True:
    path.append(g)
    a, b = nl.fanin_offsets[g], nl.fanin_offsets[g + 1]
    srcs = [int(x) - P for x in nl.fanin_net[a:b] if x >= P]
    if not srcs:
        break
    g = max(srcs, key=lambda x: done[x])
path = path[::-1]
run = sum(done[x] - plan[x] for x in path)
print(f"critical path: {len(path)} gates, levels {glev[path[0]]}..{glev[path[-1]]}, ends at {done[path[-1]]:.0f} us; "
      f"running {run:.0f} us, waiting {done[path[-1]] - run:.0f} us; first planned at {plan[path[0]]:.0f} us")
for x in path[:: max(1, len(path) // 15)]:
    print(f"  gate {x} level {glev[x]} n_in {n_in[x]:.0f} planned {plan[x]:.0f} done {done[x]:.0f} "
          f"(run {done[x] - plan[x]:.0f} us, max chunk {cmax[x]:.0f} us)")
