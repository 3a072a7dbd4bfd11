"""Results stitching on CPU: the owner-side assembly of the
canonical CSR from per-window CSRs (shard.assemble) against the oracle's full run, in
one process, and end to end over gloo with 2 and 3 ranks (shard.stitch_waveforms:
all_gather of counts, point-to-point segments to the owner, scatter) — each rank's window
simulated by the oracle exactly as bench.py's ranks do with the GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from csr_util import cpu_alloc, numpy_scatter, window_csr
from oracle import oracle
from paper_2304_13398_b200 import shard
from paper_2304_13398_b200 import workloads as W


def _setup():
    nl = W.recipe_netlist(17, 500, 10, 30)
    spec = W.make_stimspec(17, 30, 50, "skewed", mean_trans=16, wcv=3.0)
    return nl, spec


def _halo(nl):
    P, G = nl.num_inputs, nl.num_gates
    A = np.zeros(P + G, np.int64)
    for g in range(G):
        a, b = nl.fanin_offsets[g], nl.fanin_offsets[g + 1]
        A[P + g] = max(A[s] for s in nl.fanin_net[a:b]) + int(nl.pin_delay[a:b].max())
    return int(A.max()) + 1


def _full(nl, spec):
    o, t = W.generate_stimuli(spec)
    st = W.to_stimuli(o, t)
    return oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay,
                           st.offsets, st.trans, spec.duration)


def _rank_window(nl, spec, rank, world):
    """The rank's owned window of its own (halo-clamped) oracle run: (counts, transitions)."""
    plan = shard.rank_plan(rank, world, spec.ncycles, _halo(nl), spec.duration)
    o, t = W.window_stimuli(spec, *plan["gen_cycles"], "cpu")
    st = W.to_stimuli(o, t)
    r = oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay,
                        st.offsets, st.trans, plan["duration"])
    return window_csr(r.offsets, r.trans, *plan["own"])


@pytest.mark.parametrize("world", [1, 2, 4])
def test_assemble_windows_equals_full_run(world):
    nl, spec = _setup()
    full = _full(nl, spec)
    parts = [_rank_window(nl, spec, r, world) for r in range(world)]
    allc = torch.as_tensor(np.stack([c for c, _ in parts]))
    bufs = [torch.as_tensor(tr.view(np.int64)) for _, tr in parts]
    off, out = shard.assemble(allc, bufs, numpy_scatter, cpu_alloc)
    assert np.array_equal(off.numpy(), full.offsets)
    assert np.array_equal(out.numpy()[:off[-1]].view(np.uint64), full.trans)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nl, spec = _setup()
    cnt, tr = _rank_window(nl, spec, rank, world)
    res = shard.stitch_waveforms(torch.as_tensor(cnt), torch.as_tensor(tr.view(np.int64)), numpy_scatter,
                                 cpu_alloc, dst=world - 1)
    if rank == world - 1:
        off, out = res
        q.put((off.numpy().copy(), out.numpy()[:int(off[-1])].view(np.uint64).copy()))
    else:
        assert res is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_stitch_waveforms_gloo(world):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    off, tr = q.get(timeout=300)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    nl, spec = _setup()
    full = _full(nl, spec)
    assert np.array_equal(off, full.offsets)
    assert np.array_equal(tr, full.trans)


def test_union_netlist_is_its_copies():
    """C5's batching of independent stimulus sets (bench.py --c5-union): k disjoint copies of
    a netlist simulated as one, each copy driven by its own set, give every copy exactly the
    single-set result (oracle on both sides)."""
    nl = W.recipe_netlist(5, 300, 12, 20)
    k = 3
    u = W.union_netlist(nl, k)
    sts = [W.random_stimuli(40 + c, nl.num_inputs, 30, 600, xz=0.1) for c in range(k)]
    off = [np.zeros(1, np.int64)]
    tr, base = [], 0
    for st in sts:
        off.append(st.offsets[1:] + base)
        base += int(st.offsets[-1])
        tr.append(st.trans)
    ust = W.Stimuli(np.concatenate(off), np.concatenate(tr).astype(np.uint64))
    ref = oracle.simulate(u.num_inputs, u.gate_type, u.fanin_offsets, u.fanin_net, u.pin_delay,
                          ust.offsets, ust.trans, 650)
    for c, st in enumerate(sts):
        one = oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay,
                              st.offsets, st.trans, 650)
        assert np.array_equal(ref.hashes[W.union_nets(nl, k, c)], one.hashes)
