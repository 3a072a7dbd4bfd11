"""Scheduler A/B across input skew (the paper's WCV claim, Fig. 8/9,
P:601-603): one netlist (c4_mini: 1M gates, depth 100), stimuli with the same mean
activity and growing WCV (Eq. 5), each simulated with the dataflow scheduler (Alg. 1
unlock rule on the device) and with level barriers; prints one JSON line per run."""
import json, sys, time
sys.path.insert(0, '.')
import torch
from paper_2304_13398_b200 import gls, workloads as W

def run(ctx, spec, dev, sched, steps=2, warm=2):
    ctx.gls_set_config(scheduler=sched)
    d_off, d_tr = W.window_stimuli(spec, 0, spec.ncycles, dev)
    lens = (d_off[1:] - d_off[:-1]).double()
    wcv = float(lens.std(unbiased=False) / lens.mean())
    ctx.gls_set_input_waveforms_device(spec.num_inputs, d_off.data_ptr(), d_tr.data_ptr(), int(d_tr.numel()))
    del d_off, d_tr, lens
    torch.cuda.empty_cache()
    for _ in range(warm):
        ctx.gls_simulate(spec.duration)
    ms = []
    for _ in range(steps):
        ctx.gls_simulate(spec.duration)
        ms.append(ctx.gls_get_stats()["kernel_ms"])
    s = ctx.gls_get_stats()
    return wcv, min(ms), s

dev = torch.device("cuda", 0)
nl = W.config_netlist("c4_mini", 1)
c = W.CONFIGS["c4_mini"]
c4_cycles = c["ncycles"]
ncyc = int(sys.argv[1]) if len(sys.argv) > 1 else c4_cycles
ctx = gls.Context(0, torch.cuda.current_stream(dev).cuda_stream)
ctx.load(nl)
mean = max(50, c["mean_trans"] * ncyc // c["ncycles"])   # the same mean activity in every run
for target in [None, 1.0, 4.0, 17.1, 54.5]:   # 17.1, 54.5: NVDLA_c, NVDLA_o
    # "random": every PI toggles with p = 0.5 per cycle, so 2 * mean cycles give the same mean
    spec = (W.make_stimspec(1, c["num_inputs"], 2 * mean, "random") if target is None else
            W.make_stimspec(1, c["num_inputs"], ncyc, "skewed", mean, target))
    row = {}
    for sched, name in [(0, "dataflow"), (1, "levels")]:
        wcv, ms, s = run(ctx, spec, dev, sched)
        row[name] = ms
        row["gate_evals"] = s["gate_evals"]
        row["wcv"] = round(wcv, 2)
    row["target_wcv"] = target
    row["speedup_dataflow"] = row["levels"] / row["dataflow"]
    print(json.dumps(row), flush=True)
