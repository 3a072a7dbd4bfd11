"""Time each public-API call of the e2e step on a config (host pinned inputs)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2304_13398_b200 import gls, workloads as W
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4_10m"
nl = W.config_netlist(cfg, 1); spec = W.config_stimspec(cfg, 1)
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
ctx = gls.Context(0, stream.cuda_stream)
ctx.gls_set_config(); ctx.load(nl)
d_off, d_tr = W.window_stimuli(spec, 0, spec.ncycles, dev)
h_off = torch.empty(d_off.numel(), dtype=torch.int64, pin_memory=True); h_off.copy_(d_off)
h_tr = torch.empty(d_tr.numel(), dtype=torch.int64, pin_memory=True); h_tr.copy_(d_tr)
off_np, tr_np = h_off.numpy(), h_tr.numpy().view(np.uint64)
n = int(d_tr.numel()); del d_off, d_tr; torch.cuda.empty_cache()
def timed(f):
    torch.cuda.synchronize(); t = time.perf_counter(); r = f(); torch.cuda.synchronize(); return r, 1e3 * (time.perf_counter() - t)
for it in range(3):
    _, a = timed(lambda: ctx.gls_set_input_waveforms(nl.num_inputs, off_np, tr_np))
    _, b = timed(lambda: ctx.gls_simulate(spec.duration))
    _, c = timed(lambda: ctx.gls_get_net_hashes())
    s = ctx.gls_get_stats()
    print(f"iter {it}: set_input {a:.1f} ms ({8*(n+len(off_np))/a/1e6:.1f} GB/s), simulate {b:.1f} ms (kernel {s['kernel_ms']:.1f}, simulate_ms {s['simulate_ms']:.1f}), hashes {c:.1f} ms")
