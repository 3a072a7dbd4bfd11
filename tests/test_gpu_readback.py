"""a10 readback and the §8(e) results stitch on the GPU, through the C ABI, against the
oracle: the device-built canonical CSR (gls_get_waveforms_range_device) over net and
time ranges, gls_get_waveforms through a small staging buffer (many batches), time
windows simulated one after the other as the ranks would and assembled into the full
run's CSR with gls_scatter_segments, and shard.gls_gather_waveforms over a one-rank
NCCL group."""
import numpy as np
import pytest
import torch

from csr_util import window_csr
from oracle import oracle
from paper_2304_13398_b200 import gls, shard
from paper_2304_13398_b200 import workloads as W

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module")
def ctx():
    c = gls.Context(0, torch.cuda.current_stream(DEV).cuda_stream)
    yield c
    c.close()


def _design(seed=31, G=1500, P=90, cycles=300):
    nl = W.recipe_netlist(seed, G, 16, P, shuffle=True)
    spec = W.make_stimspec(seed, P, cycles, "skewed", mean_trans=60, wcv=3.0)
    o, t = W.generate_stimuli(spec)
    st = W.to_stimuli(o, t)
    ref = oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay,
                          st.offsets, st.trans, spec.duration)
    return nl, st, spec.duration, ref


def _range(ctx, n0, n1, lo, hi):
    offs = torch.empty(n1 - n0 + 1, dtype=torch.int64, device=DEV)
    total = ctx.gls_get_waveforms_range_device(n0, n1, lo, hi, offs.data_ptr())
    tr = torch.empty(max(1, total), dtype=torch.int64, device=DEV)
    assert ctx.gls_get_waveforms_range_device(n0, n1, lo, hi, offs.data_ptr(), tr.data_ptr(), tr.numel()) == total
    return offs.cpu().numpy(), tr[:total].cpu().numpy().view(np.uint64)


def test_range_readback_matches_oracle(ctx):
    nl, st, dur, ref = _design()
    ctx.gls_set_config(chunk_events=64)                 # many chunks per net
    ctx.load(nl)
    ctx.gls_set_input_waveforms(nl.num_inputs, st.offsets, st.trans)
    ctx.gls_simulate(dur)
    N = nl.num_nets
    I64 = np.iinfo(np.int64)
    off, tr = _range(ctx, 0, N, I64.min, I64.max)       # the whole run
    assert np.array_equal(off, ref.offsets) and np.array_equal(tr, ref.trans)
    rng = np.random.default_rng(5)
    for _ in range(12):
        n0 = int(rng.integers(0, N))
        n1 = int(rng.integers(n0, N + 1))
        lo = int(rng.integers(-5, dur))
        hi = int(rng.integers(lo, dur + 10))
        off, tr = _range(ctx, n0, n1, lo, hi)
        sub = ref.offsets[n0:n1 + 1]
        c, e = window_csr(sub - sub[0], ref.trans[sub[0]:sub[-1]], lo, hi)
        assert np.array_equal(np.diff(off), c) and np.array_equal(tr, e)
    # size query, errors
    offs = torch.empty(N + 1, dtype=torch.int64, device=DEV)
    total = ctx.gls_get_waveforms_range_device(0, N, 0, dur, offs.data_ptr())
    small = torch.empty(max(1, total - 1), dtype=torch.int64, device=DEV)
    with pytest.raises(gls.GlsError) as e:
        ctx.gls_get_waveforms_range_device(0, N, 0, dur, offs.data_ptr(), small.data_ptr(), total - 1)
    assert e.value.code == gls.GLS_ERANGE
    for bad in [(-1, N, 0, 1), (0, N + 1, 0, 1), (5, 4, 0, 1), (0, N, 5, 4)]:
        with pytest.raises(gls.GlsError) as e:
            ctx.gls_get_waveforms_range_device(*bad, offs.data_ptr())
        assert e.value.code == gls.GLS_EINVAL


def test_host_readback_in_small_batches(ctx):
    """gls_get_waveforms through a 1 MiB staging buffer: the canonical CSR arrives in many
    batches of nets, bit-exact."""
    nl, st, dur, ref = _design(33, 4000, 200, 400)
    ctx.gls_set_config(readback_mib=1)
    ctx.load(nl)
    ctx.gls_set_input_waveforms(nl.num_inputs, st.offsets, st.trans)
    ctx.gls_simulate(dur)
    assert ref.trans.size > (1 << 17)                     # > 1 batch of 1 MiB
    w = ctx.gls_get_waveforms()
    assert np.array_equal(w.offsets, ref.offsets) and np.array_equal(w.trans, ref.trans)


@pytest.mark.parametrize("windows", [2, 3, 5])
def test_windows_assembled_on_device_equal_full_run(ctx, windows):
    """The ranks' work done one after the other on one GPU: each window simulated with its
    halo (gls_simulate_window), its owned part read back as a device CSR, then the owner's
    assembly (shard.assemble with gls_scatter_segments) = the oracle's full CSR."""
    nl, st, dur, ref = _design(35)
    ctx.gls_set_config(chunk_events=128)
    ctx.load(nl)
    ctx.gls_set_input_waveforms(nl.num_inputs, st.offsets, st.trans)
    cuts = [dur * k // windows for k in range(windows)] + [dur + 1]
    counts, bufs = [], []
    for a, b in zip(cuts, cuts[1:]):
        ctx.gls_simulate_window(a, b, dur)
        c, tr = shard.gls_window_csr(ctx, a, b - 1, DEV)
        counts.append(c)
        bufs.append(tr)
    off, out = shard.assemble(torch.stack(counts), bufs, shard.gls_scatter(ctx),
                              lambda k: torch.empty(max(1, k), dtype=torch.int64, device=DEV))
    assert np.array_equal(off.cpu().numpy(), ref.offsets)
    assert np.array_equal(out[:int(off[-1])].cpu().numpy().view(np.uint64), ref.trans)


def test_gather_waveforms_over_nccl_single_rank(ctx):
    import os
    import socket
    import torch.distributed as dist
    nl, st, dur, ref = _design(37, 900, 60, 200)
    ctx.gls_set_config()
    ctx.load(nl)
    ctx.gls_set_input_waveforms(nl.num_inputs, st.offsets, st.trans)
    ctx.gls_simulate(dur)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    try:
        off, out = shard.gls_gather_waveforms(ctx, 0, dur, DEV)
        torch.cuda.synchronize(DEV)
    finally:
        dist.destroy_process_group()
    assert np.array_equal(off.cpu().numpy(), ref.offsets)
    assert np.array_equal(out[:int(off[-1])].cpu().numpy().view(np.uint64), ref.trans)


def test_union_netlist_on_gpu_is_its_copies():
    """bench.py's C5 batching on the GPU: k disjoint netlist copies, one stimulus set each,
    in one gls_simulate give every copy the oracle's single-set result (whole CSR)."""
    nl = W.recipe_netlist(8, 400, 15, 24, shuffle=True)
    k = 4
    u = W.union_netlist(nl, k)
    sts = [W.random_stimuli(60 + c, nl.num_inputs, 40, 900, xz=0.1) for c in range(k)]
    off, tr, base = [np.zeros(1, np.int64)], [], 0
    for st in sts:
        off.append(st.offsets[1:] + base)
        base += int(st.offsets[-1])
        tr.append(st.trans)
    with gls.Context(0) as c:
        c.load(u)
        c.gls_set_input_waveforms(u.num_inputs, np.concatenate(off), np.concatenate(tr).astype(np.uint64))
        c.gls_simulate(950)
        w = c.gls_get_waveforms()
    for ci, st in enumerate(sts):
        ref = oracle.simulate(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay,
                              st.offsets, st.trans, 950)
        got = np.concatenate([w.trans[w.offsets[n]:w.offsets[n + 1]] for n in W.union_nets(nl, k, ci)])
        assert np.array_equal(got, ref.trans)
