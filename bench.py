#!/usr/bin/env python
"""bench.py — throughput of the gate-level re-simulation hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4_10m] [--impl gls|reference]

A step is one gls_simulate: every gate of the netlist over the whole duration
(all of SURVEY §8(a): plan, k-way merge, LUT, delays, Eq. 1 filter, exact
allocation, levels), with the given waveforms already resident in HBM.  The
value is gate-evaluations per second (metric of BASELINE.json), whole job.

N = 1: the 10M-gate config (c4_10m) on one GPU.  N > 1 (torchrun): the same
workload split into N time windows with a max-path-delay halo (strong scaling,
DESIGN.md §4 / §8); rank 0 prints the JSON line with max-over-ranks timing.

The default run also (rank 0 only) times the CPU oracle on a bounded prefix of
the same workload (cpu_baseline) and checks the GPU's full-size run against it
on that window (parity).  --impl reference times the oracle alone.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2304_13398_b200 import workloads as W  # noqa: E402

FALLBACK_HBM_GBS = 6650.0   # /opt/skills/guides/B200_PROFILING.md fallback
WINDOWS = {}   # N = 1 time windows per launch (--windows; measured slower: off by default)
C5_SETS = int(os.environ.get("GLS_BENCH_C5_SETS", "64"))   # BASELINE configs[4]: 64 independent stimulus sets
# Functional multi-rank runs on ONE GPU (not measurements): GLS_BENCH_BACKEND=gloo stages the
# collectives through host memory and GLS_BENCH_ONE_GPU=1 puts every rank on cuda:0 (NCCL
# refuses two ranks on one device).  The product path is NCCL, one rank per GPU.
BACKEND = os.environ.get("GLS_BENCH_BACKEND", "nccl")
ONE_GPU = os.environ.get("GLS_BENCH_ONE_GPU", "0") == "1"

# prefix of the workload the oracle runs (cycles), sized for ~10-30 s of one core
SAMPLE_CYCLES = {"c4_10m": 3000, "c3_1m": 60, "c7552": 1999, "c5_set": 150, "c4_mini": 3000}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4_10m", choices=sorted(W.CONFIGS))
    ap.add_argument("--impl", default="gls", choices=["gls", "reference"])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sample-cycles", type=int, default=0)
    ap.add_argument("--chunk-events", type=int, default=0)
    ap.add_argument("--blocks-per-sm", type=int, default=0)
    ap.add_argument("--arena-gb", type=float, default=0.0)
    ap.add_argument("--engine", type=int, default=0)
    ap.add_argument("--scheduler", type=int, default=0)
    ap.add_argument("--windows", type=int, default=0,
                    help="N=1: time windows with the max-path-delay halo simulated as disjoint netlist "
                         "copies in one launch (0: the config's default)")
    ap.add_argument("--c5-union", type=int, default=8,
                    help="C5: stimulus sets per launch (k disjoint netlist copies, one set each)")
    ap.add_argument("--ncycles", type=int, default=0,
                    help="A/B / profiling only: override the config's number of clock cycles")
    ap.add_argument("--wcv", type=float, default=0.0,
                    help="A/B only: override the skewed profile's WCV target (Eq. 5) of the config")
    return ap.parse_args()


def _shard_ag(out, t):
    from paper_2304_13398_b200 import shard
    shard.all_gather_t(out, t)


def log(*a):
    print("[bench]", *a, file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy-based)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(self.dev)], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) == 6:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def build_netlist(cfg, seed):
    t = time.perf_counter()
    nl = W.config_netlist(cfg, seed)
    log(f"netlist {cfg}: {nl.num_gates} gates, {nl.num_inputs} PIs, {nl.num_pins} pins "
        f"({time.perf_counter() - t:.1f}s)")
    return nl


def host_cpu():
    """CPU model and logical core count of the host (the oracle timings' machine)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def oracle_sample(nl, spec, cycles):
    """The oracle as it stands on the workload's first `cycles` clock cycles."""
    from oracle import oracle
    o, t = W.window_stimuli(spec, 0, cycles, "cpu")
    st = W.to_stimuli(o, t)
    dur = cycles * W.PERIOD
    t0 = time.perf_counter()
    r = oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay,
                        st.offsets, st.trans, dur, want_waves=False)
    dt = time.perf_counter() - t0
    return r, dt, dur


def _oracle_set_worker(args):
    """(spawned process) the oracle as it stands on one stimulus set's first `cycles` cycles"""
    cfg, seed, cycles = args
    nl = W.config_netlist(cfg, 1)
    spec = W.config_stimspec(cfg, seed)
    r, dt, _ = oracle_sample(nl, spec, cycles)
    return r.gate_evals, dt


def oracle_sets_concurrent(cfg, seeds, cycles):
    """C5's CPU baseline: min(64, nproc) single-thread oracle processes, one per
    stimulus set, run concurrently; aggregate gate-evals / the slowest process's time."""
    import concurrent.futures as cf
    import multiprocessing as mp
    with cf.ProcessPoolExecutor(max_workers=len(seeds), mp_context=mp.get_context("spawn")) as ex:
        res = list(ex.map(_oracle_set_worker, [(cfg, s, cycles) for s in seeds]))
    evals = sum(r[0] for r in res)
    return evals, max(r[1] for r in res)


def run_reference(a):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cfg = a.config
    nl = build_netlist(cfg, a.seed)
    # C5 (independent stimulus sets): one set per rank, replicas; otherwise one workload
    # split into time windows
    replicas = cfg == "c5_set" and world > 1
    spec = W.config_stimspec(cfg, a.seed + (rank if replicas else 0))
    # the cpu_baseline leg's sample when K + W = 8 (the default run), shorter for longer
    # runs so that the whole reference arm stays within a few minutes
    base = a.sample_cycles or SAMPLE_CYCLES[cfg]
    cyc = max(1, base * 8 // max(8, a.steps + a.warmup))
    for _ in range(a.warmup):
        oracle_sample(nl, spec, cyc)
    evals, secs, outs = 0, 0.0, 0
    for _ in range(a.steps):
        r, dt, dur = oracle_sample(nl, spec, cyc)
        evals += r.gate_evals
        outs += r.out_trans
        secs += dt
    v = evals / secs
    sample = (f"{cfg} netlist ({nl.num_gates} gates), first {cyc} of {spec.ncycles} clock cycles "
              f"(t <= {cyc * W.PERIOD} ps), {r.gate_evals} gate-evals per step")
    line = {"impl": "reference", "metric": "gate-evals/s", "value": v, "unit": "gate-evals/s",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * secs / a.steps,
            "higher_is_better": True, "scaling": "strong" if world > 1 and not replicas else "weak", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic",
            "config": {"workload": cfg, "gates": nl.num_gates, "pis": nl.num_inputs},
            "output_transitions_per_s": outs / secs,
            "cpu_baseline": {"value": v, "unit": "gate-evals/s", "cores": 1, "kind": "oracle", "sample": sample,
                             **host_cpu()},
            "e2e": {"value": v, "unit": "gate-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def balance_str(s):
    """engine-0 counters (gls_stats.balance): static units, units split off while running,
    re-balancing rounds, fallback units, per batch"""
    b = s.get("balance") or [0] * 8
    nb = max(1, s.get("batches") or 1)
    return (f"[units/batch {b[0] / nb:.1f}, splits/batch {b[1] / nb:.2f}, rounds/batch {b[2] / nb:.1f}, "
            f"fallback units {int(b[3])}, set-up/end/re-balance clocks of the sweep "
            f"{[round(x / max(1.0, (s.get('phase_cycles') or [0] * 6)[2]), 3) for x in b[4:7]]}]")


def post_timing_stitch(ctx, nl, plan, dev, stream, world, rank, replicas, set_hashes, stims):
    """N > 1, after the timed region: the §8(e) stitch of the ranks' results:
    time windows — full-run per-net checksums and the waveforms of 1/16 of the nets
    gathered on rank 0; stimulus sets — every set's per-net checksums on every rank."""
    stitch = None
    if world > 1 and not replicas:
        from paper_2304_13398_b200 import shard as _shard
        lo, hi = plan["own"]
        torch.distributed.barrier()
        torch.cuda.synchronize(dev)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        stitched = _shard.gls_window_stitch(ctx, lo, hi, dev)
        s1.record(stream)
        torch.cuda.synchronize(dev)
        st_ms = s0.elapsed_time(s1)
        tt = torch.tensor([st_ms], dtype=torch.float64, device=dev)
        allv = [torch.zeros_like(tt) for _ in range(world)]
        _shard_ag(allv, tt)
        stitch = {"ms": float(torch.stack(allv).max()), "nets": int(stitched.numel()),
                  "bytes_per_rank": int(16 * stitched.numel()),
                  "what": "full-run per-net checksums from the time windows (all_gather of counts and "
                          f"position-keyed terms over {BACKEND})"}
        del stitched
        # the waveforms themselves (§8(e) stitch): every rank's owned-window CSR of the first
        # 1/16 of the nets to rank 0 (the whole result, ~90 GB, would not fit beside rank 0's
        # own arena), assembled there into the canonical CSR of the full run
        n_sub = max(1, nl.num_nets // 16)
        torch.distributed.barrier()
        torch.cuda.synchronize(dev)
        s0.record(stream)
        res = _shard.gls_gather_waveforms(ctx, lo, hi, dev, dst=0, net_lo=0, net_hi=n_sub)
        s1.record(stream)
        torch.cuda.synchronize(dev)
        g_ms = s0.elapsed_time(s1)
        tt = torch.tensor([g_ms], dtype=torch.float64, device=dev)
        allv = [torch.zeros_like(tt) for _ in range(world)]
        _shard_ag(allv, tt)
        if rank == 0:
            g_bytes = 8 * int(res[0][-1])
            stitch["waveforms"] = {"ms": float(torch.stack(allv).max()), "nets": [0, n_sub], "bytes": g_bytes,
                                   "gbs": g_bytes / (float(torch.stack(allv).max()) / 1e3) / 1e9,
                                   "what": f"owned-window CSRs (gls_get_waveforms_range_device) -> {BACKEND} "
                                           "send/recv to rank 0 -> gls_scatter_segments into the full-run CSR"}
        del res
    if world > 1 and replicas:
        # C5: every set's per-net checksums (computed on the device in the step) to every rank
        torch.distributed.barrier()
        torch.cuda.synchronize(dev)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        per = (C5_SETS + world - 1) // world
        mine = torch.zeros((per, nl.num_nets), dtype=torch.int64, device=dev)
        mine[:set_hashes.shape[0]] = set_hashes
        allh = [torch.empty_like(mine) for _ in range(world)]
        _shard_ag(allh, mine)
        s1.record(stream)
        torch.cuda.synchronize(dev)
        # set k lives on rank k % world at row k // world
        h0 = allh[0][0].cpu()
        stitch = {"ms": s0.elapsed_time(s1), "sets": C5_SETS, "bytes": int(8 * per * world * nl.num_nets),
                  "what": f"per-set per-net checksums (device, in the step) all_gathered over {BACKEND}",
                  "set0_matches_rank0": bool(torch.equal(h0, set_hashes[0].cpu()))}
        del allh, mine
    return stitch


def run_gls(a):
    from paper_2304_13398_b200 import gls
    rank, world, local = dist_env()
    if ONE_GPU:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        if BACKEND == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(BACKEND)
    cfg = a.config
    nl = build_netlist(cfg, a.seed)
    # C5 (BASELINE configs[4]): C5_SETS independent stimulus sets on one netlist, dealt
    # round-robin to the ranks (replicas, no exchange); otherwise one workload split into
    # time windows
    sets = list(range(rank, C5_SETS, world)) if cfg == "c5_set" else [0]
    replicas = cfg == "c5_set"
    spec = W.config_stimspec(cfg, a.seed + sets[0])
    # C5: UK sets per launch, as UK disjoint copies of the netlist (independent problems in
    # one launch fill the warps a single set's critical path leaves idle; each copy's result
    # is exactly its set's, tests/test_stitch.py::test_union_netlist_is_its_copies)
    UK = 1
    if replicas:
        UK = max(1, min(a.c5_union, len(sets)))
        while len(sets) % UK:
            UK -= 1
    # N = 1 time windows (reading R17): the run split into KW windows with the max-path-delay
    # halo, simulated as KW disjoint netlist copies in one launch — every copy's outputs are
    # exact on its window, and a hot gate's work is split KW ways, which shortens the
    # dependency chain through the hot cone that bounds C4
    KW = 1
    if not replicas and world == 1:
        KW = a.windows if a.windows > 0 else WINDOWS.get(cfg, 1)
    copies = UK if replicas else KW
    unl = W.union_netlist(nl, copies)
    stream = torch.cuda.current_stream(dev)
    ctx = gls.Context(local, stream.cuda_stream)
    ctx.gls_set_config(chunk_events=a.chunk_events, blocks_per_sm=a.blocks_per_sm,
                       arena_bytes=int(a.arena_gb * (1 << 30)), engine=a.engine, scheduler=a.scheduler)
    t = time.perf_counter()
    ctx.load(unl)
    L = ctx.gls_get_levels()
    H = ctx.gls_get_halo()
    log(f"loaded: {L} levels, halo {H} ps ({time.perf_counter() - t:.1f}s)")

    # this rank's time window (strong scaling over the time axis; one window at N=1)
    from paper_2304_13398_b200 import shard
    nc = spec.ncycles
    plan = shard.rank_plan(0 if replicas else rank, 1 if replicas else world, nc, H, spec.duration)
    k_hi = plan["gen_cycles"][1]
    duration = plan["duration"]
    t = time.perf_counter()
    stims = []                       # this rank's given waveforms, resident in HBM: one per launch
    halo_stim = None
    if KW > 1:
        offs, trs, hoffs, htrs, base, hbase = [], [], [], [], 0, 0
        for k in range(KW):
            pk = shard.rank_plan(k, KW, nc, H, spec.duration)
            d_off, d_tr = W.window_stimuli(spec, *pk["gen_cycles"], dev)
            offs.append(d_off if not offs else d_off[1:] + base)
            base += int(d_tr.numel())
            trs.append(d_tr)
            # the same window's halo alone (cycles before its own): its evaluations are the
            # ones the window repeats from its predecessor; counted once, then subtracted
            k_lo = shard.time_window(k, KW, nc)[0]
            if k == 0:
                h_off, h_tr = torch.zeros(nl.num_inputs + 1, dtype=torch.int64, device=dev), d_tr[:0]
            else:
                h_off, h_tr = W.window_stimuli(spec, pk["gen_cycles"][0], k_lo, dev)
            hoffs.append(h_off if not hoffs else h_off[1:] + hbase)
            hbase += int(h_tr.numel())
            htrs.append(h_tr)
        stims.append((torch.cat(offs), torch.cat(trs), base))
        halo_stim = (torch.cat(hoffs), torch.cat(htrs), hbase)
        del offs, trs, hoffs, htrs
        duration = spec.duration
    for g0 in (range(0, len(sets), UK) if KW == 1 else []):
        offs, trs, base = [], [], 0
        for k in sets[g0:g0 + UK]:
            sp = W.config_stimspec(cfg, a.seed + k) if replicas else spec
            d_off, d_tr = W.window_stimuli(sp, *plan["gen_cycles"], dev)
            offs.append(d_off if not offs else d_off[1:] + base)
            base += int(d_tr.numel())
            trs.append(d_tr)
        d_off = offs[0] if UK == 1 else torch.cat(offs)
        d_tr = trs[0] if UK == 1 else torch.cat(trs)
        del offs, trs
        stims.append((d_off, d_tr, int(d_tr.numel())))
    torch.cuda.synchronize(dev)
    torch.cuda.empty_cache()            # the generator's temporaries: leave the HBM to the library's arena
    d_off, d_tr, n_in = stims[0]
    P_ = nl.num_inputs
    lens = (d_off[1:P_ + 1] - d_off[:P_]).double()                              # (set 0)
    for k in range(1, KW):                                                    # (windows: the whole run)
        lens = lens + (d_off[k * P_ + 1:(k + 1) * P_ + 1] - d_off[k * P_:(k + 1) * P_]).double()
    wcv = float(lens.std(unbiased=False) / lens.mean()) if n_in else 0.0
    n_in_all = sum(x[2] for x in stims)
    log(f"stimuli: {len(stims)} set(s), {n_in_all} transitions on {spec.num_inputs} PIs, WCV {wcv:.2f} "
        f"({time.perf_counter() - t:.1f}s)")
    if not replicas:
        ctx.gls_set_input_waveforms_device(unl.num_inputs, d_off.data_ptr(), d_tr.data_ptr(), n_in)
    # per launch: the checksums of every net of the (union) netlist, kept on the device
    launch_hashes = torch.zeros((len(stims), unl.num_nets), dtype=torch.int64, device=dev) if replicas else None

    def step():
        """One pass of the hot path over the rank's batch of input: its time window, or each
        of its stimulus sets (set the device-resident inputs, simulate).  Returns the
        per-simulation stats of the step (kernel time, counts)."""
        if not replicas:
            ctx.gls_simulate(duration)
            return [ctx.gls_get_stats()]
        out = []
        for k_, (o_, t_, n_) in enumerate(stims):
            ctx.gls_set_input_waveforms_device(unl.num_inputs, o_.data_ptr(), t_.data_ptr(), n_)
            ctx.gls_simulate(duration)
            ctx.gls_get_net_hashes_device(launch_hashes[k_].data_ptr())  # a10 per launch, on the device
            out.append(ctx.gls_get_stats())
        return out

    halo_evals = halo_outs = 0
    if halo_stim is not None:
        ctx.gls_set_input_waveforms_device(unl.num_inputs, halo_stim[0].data_ptr(), halo_stim[1].data_ptr(), halo_stim[2])
        ctx.gls_simulate(duration)
        hs = ctx.gls_get_stats()
        halo_evals, halo_outs = int(hs["gate_evals"]), int(hs["out_transitions"])
        ctx.gls_set_input_waveforms_device(unl.num_inputs, d_off.data_ptr(), d_tr.data_ptr(), n_in)
        log(f"{KW} windows: halo re-evaluations {halo_evals} gate-evals, {halo_outs} outputs (subtracted)")
        del halo_stim
    for i in range(a.warmup):
        t = time.perf_counter()
        s = step()[0]
        log(f"warmup {i}: kernel {s['kernel_ms']:.1f} ms, {s['gate_evals']} gate-evals, "
            f"{s['out_transitions']} outputs, {s['chunks']} chunks ({s['deep_chunks']} fallback), "
            f"lane util {s['lane_utilization']:.2f}, batches {s['batches']} x {s['batch_lanes']:.1f} lanes / "
            f"{s['batch_est']:.0f} est, phases {[round(x / max(1.0, sum(s['phase_cycles'][:5])), 3) for x in s['phase_cycles']]}, "
            f"arena {s['arena_used_bytes'] / 1e9:.1f} GB, balance {balance_str(s)} "
            f"(wall {time.perf_counter() - t:.2f}s)")
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kernel_ms = []
    ev0.record(stream)
    for _ in range(a.steps):
        st_ = step()
        kernel_ms.extend(x["kernel_ms"] for x in st_)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    ck = clocks.stop()
    ms = ev0.elapsed_time(ev1) / a.steps
    s = st_[-1]
    units = sum(x["gate_evals"] for x in st_) - halo_evals  # per step, this rank (halo evaluations not counted)
    outs = sum(x["out_transitions"] for x in st_) - halo_outs
    alg = statistics.mean(x["alg_bytes"] for x in st_)      # per kernel launch
    kms = statistics.mean(kernel_ms)                        # per kernel launch
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([ms, kms, units, outs, alg], dtype=torch.float64, device=dev)
        allv = [torch.zeros_like(tt) for _ in range(world)]
        _shard_ag(allv, tt)
        allv = torch.stack(allv).cpu().numpy()
        ms, kms = float(allv[:, 0].max()), float(allv[:, 1].max())
        units, outs = float(allv[:, 2].sum()), float(allv[:, 3].sum())
        alg = float(allv[:, 4].mean())                      # per launch on one GPU (roofline is per GPU)

    # per-set checksums (each set's nets inside its launch's union netlist), after the timing
    set_hashes = None
    if launch_hashes is not None:
        idx = [torch.as_tensor(W.union_nets(nl, UK, c), device=dev) for c in range(UK)]
        set_hashes = torch.stack([launch_hashes[j][idx[c]] for j in range(len(stims)) for c in range(UK)])

    # N > 1 time windows: stitch the full-run per-net checksums from the ranks' windows
    # (NCCL all_gather of per-net counts, then of position-keyed terms; shard.stitch_hashes),
    # timed on the device after the timed region, max over ranks
    stitch = None
    try:
        stitch = post_timing_stitch(ctx, nl, plan, dev, stream, world, rank, replicas, set_hashes, stims)
    except Exception as e:                      # the measured line must still be printed
        log(f"stitch failed: {e!r}")
        stitch = {"error": repr(e)}

    # e2e through the public API with host buffers (pinned), every step:
    # H2D of the given waveforms, simulate, D2H of the per-net hashes
    e2e = None
    if not a.no_e2e:
        e_sets = stims[:min(len(stims), 8)]     # C5: the first (up to) 8 of the rank's sets
        pinned = []
        for o_, t_, n_ in e_sets:
            h_off = torch.empty(o_.numel(), dtype=torch.int64, pin_memory=True)
            h_tr = torch.empty(n_, dtype=torch.int64, pin_memory=True)
            h_off.copy_(o_)
            h_tr.copy_(t_)
            pinned.append((h_off, h_tr))
        n_e2e = max(1, min(a.steps, 3))
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n_e2e):
            for h_off, h_tr in pinned:
                ctx.gls_set_input_waveforms(unl.num_inputs, h_off.numpy(), h_tr.numpy().view(np.uint64))
                ctx.gls_simulate(duration)
                hashes = ctx.gls_get_net_hashes()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e_ms = e0.elapsed_time(e1) / n_e2e
        e_units = sum(x["gate_evals"] for x in st_[:len(e_sets)]) - halo_evals
        if world > 1:
            import torch.distributed as dist
            tt = torch.tensor([e_ms, e_units], dtype=torch.float64, device=dev)
            allv = [torch.zeros_like(tt) for _ in range(world)]
            _shard_ag(allv, tt)
            allv = torch.stack(allv).cpu().numpy()
            e_ms, e_units = float(allv[:, 0].max()), float(allv[:, 1].sum())
        e2e = {"value": e_units / (e_ms / 1e3), "unit": "gate-evals/s",
               "h2d_bytes_per_step": int(sum(8 * (o_.numel() + n_) for o_, _, n_ in e_sets)),
               "d2h_bytes_per_step": int(8 * hashes.size * len(e_sets)), "ms_per_step": e_ms,
               "api": "gls_set_input_waveforms(host pinned) + gls_simulate + gls_get_net_hashes" +
                      (f", first {len(e_sets)} of the rank's {len(stims)} launches of {UK} stimulus sets" if replicas else "")}
        del pinned

    # e2e with a WAVEFORM readback (a10): each step H2D of the given waveforms (pinned), simulate,
    # then the canonical CSR of every net restricted to the first 1/32 of the duration
    # gathered on the device (gls_get_waveforms_range_device) and read back into pinned host
    # memory — the transitions themselves, not their checksums
    e2e_w = None
    if not a.no_e2e and not replicas and world == 1:
        try:
            o_, t_, n_ = stims[0]
            h_off = torch.empty(o_.numel(), dtype=torch.int64, pin_memory=True)
            h_tr = torch.empty(n_, dtype=torch.int64, pin_memory=True)
            h_off.copy_(o_)
            h_tr.copy_(t_)
            t_hi = duration // 32
            nn = unl.num_nets
            d_o = torch.empty(nn + 1, dtype=torch.int64, device=dev)
            tot = ctx.gls_get_waveforms_range_device(0, nn, 0, t_hi, d_o.data_ptr())
            d_w = torch.empty(max(1, int(tot * 1.05) + 1024), dtype=torch.int64, device=dev)
            h_w = torch.empty(d_w.numel(), dtype=torch.int64, pin_memory=True)
            h_o = torch.empty(nn + 1, dtype=torch.int64, pin_memory=True)
            n_e = max(1, min(a.steps, 2))
            torch.cuda.synchronize(dev)
            w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            w0.record(stream)
            d2h = 0
            for _ in range(n_e):
                ctx.gls_set_input_waveforms(unl.num_inputs, h_off.numpy(), h_tr.numpy().view(np.uint64))
                ctx.gls_simulate(duration)
                tot = ctx.gls_get_waveforms_range_device(0, nn, 0, t_hi, d_o.data_ptr(), d_w.data_ptr(), d_w.numel())
                h_o.copy_(d_o, non_blocking=True)
                h_w[:tot].copy_(d_w[:tot], non_blocking=True)
                d2h = 8 * (nn + 1 + tot)
            w1.record(stream)
            torch.cuda.synchronize(dev)
            w_ms = w0.elapsed_time(w1) / n_e
            e2e_w = {"value": units / (w_ms / 1e3), "unit": "gate-evals/s", "ms_per_step": w_ms,
                     "h2d_bytes_per_step": int(8 * (o_.numel() + n_)), "d2h_bytes_per_step": int(d2h),
                     "window_ps": [0, int(t_hi)], "transitions_read_back": int(tot),
                     "api": "gls_set_input_waveforms(host pinned) + gls_simulate + gls_get_waveforms_range_device "
                            "(all nets, first 1/32 of the duration) + D2H into pinned host memory"}
            del d_o, d_w, h_w, h_o, h_off, h_tr
        except Exception as e:                  # (a device buffer that does not fit beside the arena)
            e2e_w = {"error": repr(e)[:200]}

    # a10 at full size: the canonical CSR of the whole result through the public host API
    # (device gather in net order, batch by batch through a staging buffer, one D2H each),
    # timed once on rank 0 when it fits comfortably in host memory
    readback = None
    if rank == 0 and not a.no_e2e:
        import psutil
        rb_total = int(ctx.gls_get_net_counts().sum())
        need = 8 * rb_total
        avail = psutil.virtual_memory().available
        if need < 0.4 * avail:
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            w = ctx.gls_get_waveforms()
            dt = time.perf_counter() - t0
            readback = {"ms": 1e3 * dt, "bytes": need, "gbs": need / dt / 1e9, "transitions": rb_total,
                        "api": "gls_get_waveforms (host, pageable numpy buffer)"}
            del w
        else:
            readback = {"skipped": f"{need / 1e9:.0f} GB result > 40 % of the host's available memory"}

    if replicas:                # the parity check below is on the first set: simulate it again
        ctx.gls_set_input_waveforms_device(unl.num_inputs, stims[0][0].data_ptr(), stims[0][1].data_ptr(), stims[0][2])
        ctx.gls_simulate(duration)

    # CPU oracle on a bounded prefix of the same workload + full-size parity there
    cpu = parity = None
    if rank == 0 and not a.no_cpu_baseline:
        cyc = min(a.sample_cycles or SAMPLE_CYCLES[cfg], k_hi)
        r, dt, tmax = oracle_sample(nl, spec, cyc)
        cpu = {"value": r.gate_evals / dt, "unit": "gate-evals/s", "cores": 1, "kind": "oracle",
               "sample": f"{cfg} netlist ({nl.num_gates} gates), first {cyc} of {nc} clock cycles "
                         f"(t <= {tmax} ps): {r.gate_evals} gate-evals in {dt:.2f} s, single thread",
               **host_cpu()}
        gh = ctx.gls_get_net_hashes_window(0, tmax)[W.union_nets(nl, copies, 0)]   # (set 0 / window 0: copy 0)
        mism = int((gh != r.hashes).sum())
        parity = {"window_ps": [0, tmax], "nets": int(gh.size), "hash_mismatches": mism,
                  "bit_exact": mism == 0}
        log(f"oracle sample: {r.gate_evals} gate-evals in {dt:.2f}s; parity mismatches {mism}")
        if replicas:
            # independent stimulus sets: one single-thread oracle process per set, concurrently
            k = max(1, min(C5_SETS, os.cpu_count() or 1))
            try:
                ev, wall = oracle_sets_concurrent(cfg, [a.seed + j for j in range(k)], cyc)
                cpu.update({"value": ev / wall, "cores": k,
                            "sample": f"{cfg}: {k} stimulus sets (seeds {a.seed}..{a.seed + k - 1}) in {k} concurrent "
                                      f"single-thread oracle processes, first {cyc} of {nc} clock cycles each: "
                                      f"{ev} gate-evals, slowest process {wall:.2f} s",
                            "single_process_value": r.gate_evals / dt})
            except Exception as e:
                log(f"concurrent oracle failed: {e!r}")

    if rank == 0:
        peak, peak_src = load_peaks()
        achieved = alg / (kms / 1e3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic_r02.json")
        if os.path.exists(tp):
            try:
                with open(tp) as f:
                    traffic = json.load(f).get(cfg)
            except Exception:
                traffic = None
        line = {
            "metric": "gate-evals/s", "value": units / (ms / 1e3), "unit": "gate-evals/s",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": cfg + (f"@wcv{a.wcv:g}" if a.wcv > 0 else "") + (f"@{a.ncycles}cyc" if a.ncycles > 0 else ""), "gates": nl.num_gates,
                       "pis": nl.num_inputs, "pins": nl.num_pins,
                       "levels": L, "duration_ps": spec.duration, "stimulus_transitions": n_in,
                       "stimulus_wcv": round(wcv, 2), "halo_ps": H,
                       **({"stimulus_sets": C5_SETS, "sets_per_rank": len(sets), "sets_per_launch": UK,
                           "stimulus_transitions_per_rank": n_in_all} if replicas else {}),
                       **({"time_windows": KW, "halo_gate_evals_subtracted": halo_evals} if KW > 1 else {}),
                       "parallelism": (f"stimulus sets round-robin over {world} rank(s), no exchange" if replicas else
                                       f"{KW} time windows with the max-path-delay halo as disjoint netlist copies in one launch"
                                       if KW > 1 else
                                       f"time-windows x{world}" if world > 1 else "single GPU"),
                       "cache": "working set (given + computed waveforms) >> 126 MB L2; no flush needed"},
            "output_transitions_per_s": outs / (ms / 1e3),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": "gls::sim_kernel", "kernel_ms": kms, "alg_bytes_per_launch": alg},
            "cpu_baseline": cpu, "parity": parity, "e2e": e2e, "e2e_waveforms": e2e_w, "stitch": stitch,
            "readback": readback,
            # per step: init_given_kernel + sim_kernel (gls_simulate) and fanin_reads_kernel
            # (gls_get_stats' algorithmic-bytes count, read after every step for kernel_ms)
            # (C5: + validate_kernel of gls_set_input_waveforms_device per set)
            "gpu_launches": a.steps * len(stims) * (3 + (1 if replicas else 0)),   # (per launch)
            "clocks": ck,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    a = parse()
    if a.wcv > 0:                          # (A/B of the kernel across input skew; not a bench line)
        W.CONFIGS[a.config] = dict(W.CONFIGS[a.config], profile="skewed", wcv=a.wcv,
                                   mean_trans=W.CONFIGS[a.config].get("mean_trans") or 1000)
    if a.ncycles > 0:
        W.CONFIGS[a.config] = dict(W.CONFIGS[a.config], ncycles=a.ncycles)
    if a.impl == "reference":
        return run_reference(a)
    return run_gls(a)


if __name__ == "__main__":
    sys.exit(main())
