"""World-size-2 and -3 gloo tests of the time-window sharding, on CPU.

Each rank simulates its window with the ORACLE (CPU) exactly as bench.py's
ranks do with the GPU (same rank_plan, same window generator), computes the
per-net hashes of its owned output window, and rank 0 checks them against a
single full run restricted to each window.  This exercises the partitioning,
halo and gather logic without a GPU, and the checksum stitching
(shard.stitch_hashes): the XOR of the ranks' position-keyed window terms equals the
oracle's full-run per-net checksums.
"""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import winhash
from oracle import oracle
from paper_2304_13398_b200 import shard
from paper_2304_13398_b200 import workloads as W


def window_hash(offsets, trans, lo, hi):
    M = (1 << 64) - 1

    def sm(x):
        x = (x + 0x9E3779B97F4A7C15) & M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
        return x ^ (x >> 31)
    out = []
    for n in range(len(offsets) - 1):
        e = trans[offsets[n]:offsets[n + 1]]
        t = (e >> np.uint64(2)).astype(np.int64)
        e = e[(t >= lo) & (t <= hi)]
        h = sm(0x9E3779B97F4A7C15 ^ len(e))
        for j, x in enumerate(e):
            h ^= sm((int(x) + (j + 1) * 0xD1B54A32D192ED03) & M)
        out.append(h)
    return np.array(out, dtype=np.uint64)


def _setup():
    nl = W.recipe_netlist(11, 600, 12, 40)
    spec = W.make_stimspec(11, 40, 60, "skewed", mean_trans=20, wcv=3.0)
    return nl, spec


def _halo(nl):
    P, G = nl.num_inputs, nl.num_gates
    A = np.zeros(P + G, np.int64)
    for g in range(G):   # recipe netlists are generated in topological order
        a, b = nl.fanin_offsets[g], nl.fanin_offsets[g + 1]
        A[P + g] = max(A[s] for s in nl.fanin_net[a:b]) + int(nl.pin_delay[a:b].max())
    return int(A.max()) + 1


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nl, spec = _setup()
    H = _halo(nl)
    plan = shard.rank_plan(rank, world, spec.ncycles, H, spec.duration)
    o, t = W.window_stimuli(spec, *plan["gen_cycles"], "cpu")
    st = W.to_stimuli(o, t)
    r = oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay,
                        st.offsets, st.trans, plan["duration"])
    lo, hi = plan["own"]
    h = window_hash(r.offsets, r.trans, lo, hi)
    ht = torch.as_tensor(h.view(np.int64))
    allh = [torch.zeros_like(ht) for _ in range(world)]
    dist.all_gather(allh, ht)
    rows = shard.all_gather_rows([float(r.gate_evals), float(lo), float(hi)], "cpu")
    # stitch the full-run per-net checksums from the windows (shard.stitch_hashes)
    cnt, _ = winhash.window_terms(r.offsets, r.trans, lo, hi)

    def terms_fn(base, total):
        _, tt = winhash.window_terms(r.offsets, r.trans, lo, hi, base.numpy(),
                                     None if total is None else total.numpy())
        return torch.as_tensor(tt.view(np.int64))

    stitched = shard.stitch_hashes(torch.as_tensor(cnt), terms_fn)
    if rank == 0:
        q.put(([x.numpy().view(np.uint64).copy() for x in allh], rows.numpy(),
               stitched.numpy().view(np.uint64).copy()))
    dist.barrier()
    dist.destroy_process_group()


import pytest


@pytest.mark.parametrize("world", [2, 3])
def test_time_windows_ranks(world):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, rows, stitched = q.get(timeout=300)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    nl, spec = _setup()
    o, t = W.generate_stimuli(spec)
    st = W.to_stimuli(o, t)
    full = oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay,
                           st.offsets, st.trans, spec.duration)
    covered = []
    for r in range(world):
        lo, hi = int(rows[r, 1]), int(rows[r, 2])
        covered.append((lo, hi))
        ref = window_hash(full.offsets, full.trans, lo, hi)
        assert np.array_equal(got[r], ref), f"rank {r} window [{lo},{hi}] differs"
    # windows tile [0, duration] exactly once
    assert covered[0][0] == 0 and covered[-1][1] == spec.duration
    for (a, b), (c, d) in zip(covered, covered[1:]):
        assert c == b + 1
    # the stitched checksums are the full run's (every net, whole duration)
    assert np.array_equal(stitched, full.hashes)
    # gate-evals of the ranks cover the full run's (halo re-evaluation may add a few)
    assert rows[:, 0].sum() >= full.gate_evals
