// gls_kernels.cu — sm_100a kernels of the gate-level re-simulation hot path.
//
// One persistent cooperative kernel (sim_kernel) evaluates the whole netlist in
// one pass with no host round trip (the paper's one-pass property, P:100,
// P:254).  Work items are (gate, time-chunk) pairs: Algorithm 2
// over the chunk's time range with an exact halo, the Eq. 1 glitch filter
// with a streaming-finality rule, and an exact output segment per
// chunk (bump allocation without page waste, cf. the atomic page iterator of
// P:499).  Two schedulers:
//   * dataflow (default): Alg. 1's unlock rule on the device —
//     a gate's chunks are planned and published the moment its last fan-in
//     gate completes (per-gate ready counters); warps pull published chunks
//     from one queue, so no warp ever waits for a level to drain;
//   * level barriers: plan a topological level, device-wide barrier, evaluate
//     it, barrier (kept for A/B and for the per-lane engine).
// Two evaluation engines (gls_config.engine): 0 a warp's lanes on time-slice units
// of a batch of chunks, re-balanced while they run (gls_lanes.cuh), 1 one chunk per
// lane (below; also the exact fallback of engine 0).  DESIGN.md §4-§5 give the derivations;
// every engine / scheduler is checked bit-exactly against oracle/ by
// tests/test_gpu_parity.py.
#include <climits>

#include <cub/device/device_scan.cuh>

#include "gls_internal.cuh"

namespace gls {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
#ifndef GLS_NOFENCE
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
#else
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
#endif
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Counters whose last arriver reads what every earlier arriver wrote (gate completion,
// the Alg. 1 ready counters): each arrival is a release RMW; only the last arriver then
// issues an acquire fence (the fence-based acquire pattern of the PTX memory model), so
// the L1 invalidation an acquire implies happens once per gate, not once per arrival.
__device__ __forceinline__ unsigned atom_add_release(unsigned* p, unsigned v) {
    unsigned r;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
    return r;
}
#ifndef GLS_NOFENCE
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
#else   // A/B only: no acquire (relaxed + L2 loads, control dependency)
__device__ __forceinline__ void fence_acquire() {}
#endif
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u32(unsigned* p, unsigned v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// release fence without the L1 invalidation a full __threadfence() implies
__device__ __forceinline__ void fence_release() { asm volatile("fence.release.gpu;" ::: "memory"); }

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned warp_global_id() { return blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); }

// Device-wide barrier for a co-resident (cooperative) grid.  The last block to
// arrive publishes the abort decision (any error raised before the barrier),
// so every block takes the same branch afterwards.
__device__ bool grid_barrier(Ctl* ctl, unsigned nblocks, unsigned& gen) {
    __shared__ unsigned s_abort;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned arrived = atomicAdd(&ctl->bar_count, 1u);
        if (arrived == nblocks - 1) {
            ctl->bar_count = 0;
            ctl->bar_abort = (*(volatile unsigned*)&ctl->error) != 0u;
            __threadfence();
            st_release_u32(&ctl->bar_gen, gen + 1);
        } else {
            while (ld_acquire_u32(&ctl->bar_gen) == gen) __nanosleep(40);
        }
        __threadfence();  // gpu-scope fence also invalidates this SM's L1
        s_abort = *(volatile unsigned*)&ctl->bar_abort;
        gen = gen + 1;
    }
    __syncthreads();
    return s_abort != 0u;
}

__device__ __forceinline__ unsigned warp_incl_scan(unsigned x) {
    const unsigned lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (unsigned)o) x += y;
    }
    return x;
}
__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}
__device__ __forceinline__ unsigned long long warp_max64(unsigned long long x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = max(x, (unsigned long long)__shfl_xor_sync(0xffffffffu, x, o));
    return x;
}

// Z is read as X: code 3 -> 2.
__device__ __forceinline__ uint32_t norm_code(uint32_t v) { return v ^ ((v >> 1) & v & 1u); }
// rank in the order 0 < X < 1 (reading R2): 0->0, 2(X)->1, 1->2
__device__ __forceinline__ uint32_t rank_code(uint32_t f) { return ((f & 1u) << 1) | (f >> 1); }

__device__ __forceinline__ long long etime(uint64_t e) { return (long long)(e >> 2); }

// ------------------------------------------------------------------ allocation
// Output segments start on 128-byte lines (16 entries): no L1 line ever mixes
// a finished segment with one still being written, so reads of published
// segments need no L1 invalidation (dataflow scheduler).
constexpr unsigned long long kSegAlign = 16;
__device__ __forceinline__ unsigned long long seg_round(unsigned long long n) {
    return (n + kSegAlign - 1) & ~(kSegAlign - 1);
}
// whole warp: exact (rounded) space for `total` entries; ~0 on overflow (flag raised)
__device__ unsigned long long arena_alloc(const SimParams& p, uint32_t total) {
    const int lane = threadIdx.x & 31;
    unsigned long long at = 0;
    if (lane == 0 && total) at = atomicAdd(&p.ctl->arena_top, seg_round(total));
    at = __shfl_sync(0xffffffffu, at, 0);
    if (at + total > p.arena_cap) {
        if (lane == 0) {
            atomicOr(&p.ctl->error, kErrArena);
            atomicMax(&p.ctl->need_arena, at + total);
        }
        return ~0ull;
    }
    return at;
}
// one lane: space in this warp's private deep-scratch region (reset per chunk); ~0 on overflow
__device__ unsigned long long deep_alloc(const SimParams& p, unsigned long long n) {
    const unsigned w = warp_global_id();
    const unsigned long long at = atomicAdd(&p.deep_wtop[w], n);
    if (at + n > p.deep_per_warp) {
        atomicOr(&p.ctl->error, kErrDeep);
        atomicMax(&p.ctl->need_deep, at + n);
        return ~0ull;
    }
    return (unsigned long long)w * p.deep_per_warp + at;
}

// ------------------------------------------------------------------ net access
// time of the idx-th transition of a net (idx < net_len)
__device__ long long time_at(const SimParams& p, uint32_t net, unsigned long long idx) {
    uint32_t cb = __ldcg(&p.net_ck[net]), n = __ldcg(&p.net_nck[net]);
    uint32_t lo = 0, hi = n;  // largest j with cum[cb+j] <= idx
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (__ldcg(&p.ck_cum[cb + mid]) <= idx) lo = mid; else hi = mid;
    }
    uint32_t j = cb + lo;
    GLS_ASSERT(j < p.ck_cap && __ldcg(&p.ck_off[j]) + (idx - __ldcg(&p.ck_cum[j])) < p.arena_cap);
    return etime(p.arena[__ldcg(&p.ck_off[j]) + (idx - __ldcg(&p.ck_cum[j]))]);
}

// number of transitions of `net` with t < T (chunk start times, then inside the segment)
__device__ unsigned long long count_before(const SimParams& p, uint32_t net, long long T) {
    const uint32_t cb = __ldcg(&p.net_ck[net]), n = __ldcg(&p.net_nck[net]);
    uint32_t lo = 0, hi = n;  // largest j with ck_T[j] <= T (default 0)
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldcg(&p.ck_T[cb + mid]) <= T) lo = mid; else hi = mid;
    }
    const uint32_t j = cb + lo;
    const uint64_t* seg = p.arena + __ldcg(&p.ck_off[j]);
    uint32_t a = 0, b = __ldcg(&p.ck_cnt[j]);
    while (a < b) {
        const uint32_t m = (a + b) >> 1;
        if (etime(seg[m]) < T) a = m + 1; else b = m;
    }
    return __ldcg(&p.ck_cum[j]) + a;
}

// Cursor over one fan-in net's transitions (across its chunk segments).
struct Cursor {
    const uint64_t* ptr;
    const uint64_t* end;
    uint32_t ck, ck_end;
};

__device__ __forceinline__ void refill(const SimParams& p, Cursor& c) {
    while (c.ptr == c.end && c.ck + 1 < c.ck_end) {
        ++c.ck;
        unsigned long long off = __ldcg(&p.ck_off[c.ck]);
        uint32_t cnt = __ldcg(&p.ck_cnt[c.ck]);
        c.ptr = p.arena + off;
        c.end = c.ptr + cnt;
    }
}
__device__ __forceinline__ uint64_t head(const Cursor& c) { return c.ptr < c.end ? *c.ptr : kInfEntry; }

// Position a cursor at the first transition with t > tau0; *init = the net's
// value at tau0 (X if none).  Uses the chunk start times and each chunk's
// value-before (ck_vb) so no backward walk is needed.
__device__ void locate(const SimParams& p, uint32_t net, long long tau0, Cursor& c, uint32_t& init) {
    uint32_t cb = __ldcg(&p.net_ck[net]), n = __ldcg(&p.net_nck[net]);
    uint32_t lo = 0, hi = n;  // largest j with ck_T[j] <= tau0 + 1 (default 0)
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (__ldcg(&p.ck_T[cb + mid]) <= tau0 + 1) lo = mid; else hi = mid;
    }
    uint32_t j = cb + lo;
    const uint64_t* seg = p.arena + __ldcg(&p.ck_off[j]);
    uint32_t cnt = __ldcg(&p.ck_cnt[j]);
    uint32_t a = 0, b = cnt;  // first index with t > tau0
    while (a < b) {
        uint32_t m = (a + b) >> 1;
        if (etime(seg[m]) <= tau0) a = m + 1; else b = m;
    }
    init = a > 0 ? (uint32_t)(seg[a - 1] & 3u) : (uint32_t)__ldcg(&p.ck_vb[j]);
    c.ptr = seg + a;
    c.end = seg + cnt;
    c.ck = j;
    c.ck_end = cb + n;
    refill(p, c);
}

struct ChunkSetup {
    uint32_t src[4];
    uint4 d[4];
    uint32_t k, lut_base, dmin, dmax, pin_off;
    bool inf;                   // some delay is GLS_DELAY_INF: the gate is one chunk (no halo starts)
    long long T0, T1, tau0;
};

struct ChunkOut {
    uint32_t cnt;       // output transitions in [T0, min(T1-1, duration)]
    uint32_t evals;     // distinct input timestamps in [T0, T1)
    uint32_t events;    // zero-delay output changes at timestamps in [T0, T1)
    uint32_t vb;        // output value just before T0
    bool overflow;      // pending ring overflow (local ring only)
};

// Count input transitions of the chunk window (tau0, T1): bound for the deep ring.
__device__ unsigned long long window_bound(const SimParams& p, const ChunkSetup& s) {
    unsigned long long n = 2;
    for (uint32_t i = 0; i < s.k; ++i) {
        Cursor c;
        uint32_t init;
        locate(p, s.src[i], s.tau0, c, init);
        for (;;) {
            uint64_t h = head(c);
            if (h == kInfEntry || etime(h) >= s.T1) break;
            ++n;
            ++c.ptr;
            if (c.ptr == c.end) refill(p, c);
        }
    }
    return n;
}

// One pass of Algorithm 2 over a chunk.  DEEP selects the pending-schedule
// storage: a 32-entry ring in local memory, or a linear array in global
// scratch sized by window_bound (exact for any backtrace depth, reading R13).
template <bool WRITE, bool DEEP>
__device__ __noinline__ void run_chunk(const SimParams& p, const ChunkSetup& s, const uint8_t* lut,
                          uint64_t* out, uint64_t* dbuf, unsigned long long dcap, ChunkOut& r) {
    uint64_t lring[DEEP ? 1 : kRing];
    uint64_t* ring = DEEP ? dbuf : lring;
    const unsigned long long cap = DEEP ? dcap : (unsigned long long)p.ring_cap;
    const unsigned long long mask = DEEP ? ~0ull : (unsigned long long)(kRing - 1);

    Cursor cur[4];
    uint64_t h[4];
    uint32_t xn = 0, x0 = 0;  // packed normalised input codes, 2 bits per pin
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        h[i] = kInfEntry;
        if ((uint32_t)i < s.k) {
            uint32_t init;
            locate(p, s.src[i], s.tau0, cur[i], init);
            h[i] = head(cur[i]);
            xn |= 2u << (2 * i);                      // all inputs start at X
            x0 |= norm_code(init) << (2 * i);         // values in effect at tau0
        }
    }
    uint32_t Eprev = 2;          // previous zero-delay evaluation, X
    unsigned long long lo = 0, hi = 0;
    uint32_t lastv = 2;          // value of the last finalised schedule (X before any)
    uint32_t vb = 2, cnt = 0, evals = 0, events = 0;
    bool overflow = false;
    const long long T0 = s.T0, T1 = s.T1, dur = p.duration;
    const long long dmin = (long long)s.dmin;

    auto emit = [&](uint64_t e) {
        long long rr = etime(e);
        if (rr < T0) {
            vb = (uint32_t)(e & 3u);
        } else if (rr < T1 && rr <= dur) {
            GLS_ASSERT(!WRITE || (out + cnt >= p.arena && out + cnt < p.arena + p.arena_cap));
            if (WRITE) out[cnt] = e;
            ++cnt;
        }
        lastv = (uint32_t)(e & 3u);
    };

    // one distinct timestamp t with post-update input vector nx (Alg. 2 body)
    auto step = [&](long long t, uint32_t nx) {
        if (nx != xn) {
            uint32_t E = lut[s.lut_base + nx];                   // calculateSignals
            if (E != Eprev) {                                    // "o_k.v is changed" (R4a)
                uint32_t del = 0xffffffffu;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    uint32_t fo = (xn >> (2 * i)) & 3u, fn = (nx >> (2 * i)) & 3u;
                    if (fo != fn) {                              // changed inputs only (R3)
                        bool rise = rank_code(fn) > rank_code(fo);
                        uint32_t a = rise ? s.d[i].x : s.d[i].z;  // -> 0
                        uint32_t b = rise ? s.d[i].y : s.d[i].w;  // -> 1
                        uint32_t dd = E == 0u ? a : (E == 1u ? b : min(a, b));   // R1
                        del = min(del, dd);                      // min rule
                    }
                }
                long long rr = t + (long long)del;               // o_k.t = t + del
                if (del != kDelayInf) {                          // reading R9: unrelated pins -> no schedule
                    // addSignalChange with Eq. 1: deny pending schedules at >= rr
                    while (hi != lo && etime(ring[(hi - 1) & mask]) >= rr) --hi;
                    uint32_t tv = hi != lo ? (uint32_t)(ring[(hi - 1) & mask] & 3u) : lastv;
                    if (tv != E) {
                        if (hi - lo >= cap) {
                            overflow = true;
                        } else {
                            GLS_ASSERT(!DEEP || (dbuf + (hi & mask) >= p.deep && dbuf + (hi & mask) < p.deep + p.deep_cap));
                            ring[hi & mask] = ((uint64_t)rr << 2) | E;
                            ++hi;
                        }
                    }
                }
                if (t >= T0) ++events;
                Eprev = E;
            }
            xn = nx;
        }
        // streaming finality: later schedules appear after t + dmin, so they
        // can only deny entries beyond it
        const long long lim = t + dmin;
        while (hi != lo && etime(ring[lo & mask]) <= lim) {
            emit(ring[lo & mask]);
            ++lo;
        }
    };

    step(s.tau0, x0);  // the halo start: inputs take their values at tau0
    for (;;) {
        if (overflow) break;
        uint64_t m = min(min(h[0], h[1]), min(h[2], h[3]));
        long long t = etime(m);
        if (m == kInfEntry || t >= T1) break;
        uint32_t nx = xn;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (etime(h[i]) == t && h[i] != kInfEntry) {
                nx = (nx & ~(3u << (2 * i))) | (norm_code((uint32_t)(h[i] & 3u)) << (2 * i));
                ++cur[i].ptr;
                if (cur[i].ptr == cur[i].end) refill(p, cur[i]);
                h[i] = head(cur[i]);
            }
        }
        if (t >= T0) ++evals;
        step(t, nx);
    }
    // everything pending that appears before T1 is final for this chunk
    while (hi != lo && etime(ring[lo & mask]) < T1) {
        emit(ring[lo & mask]);
        ++lo;
    }
    r.cnt = cnt;
    r.evals = evals;
    r.events = events;
    r.vb = vb;
    r.overflow = overflow;
}

// ------------------------------------------------------------------ phase A
// Plan level l: every gate gets ceil(n_in / M) chunks (n_in = Σ fan-in lengths,
// at most len(ref)+1 where ref = longest fan-in); chunk ids are bump-allocated
// per warp and each chunk records its gate.

__device__ void plan_level(const SimParams& p, int l, unsigned gwarp, unsigned nwarps) {
    const unsigned lane = threadIdx.x & 31;
    const int g0 = p.level_off[l - 1], g1 = p.level_off[l];
    const int n = g1 - g0;
    for (int base = (int)gwarp * 32; base < n; base += (int)nwarps * 32) {
        const int gi = g0 + base + (int)lane;
        const bool v = base + (int)lane < n;
        unsigned nch = 0;
        if (v) {
            GateInfo g = p.gate[gi];
            unsigned long long n_in = 0, lenref = 0;
            for (uint32_t i = 0; i < g.k; ++i) {
                unsigned long long len = p.net_len[p.pin_src[g.pin_off + i]];
                n_in += len;
                if (len > lenref) lenref = len;
            }
            unsigned long long c = (n_in + (unsigned long long)p.M - 1) / (unsigned long long)p.M;
            if (c < 1) c = 1;
            if (c > lenref + 1) c = lenref + 1;
            if (g.flags & kGateInf) c = 1;              // no halo starts with unrelated pins (reading R9)
            nch = (unsigned)c;
            p.gate_nin[gi] = n_in;
        }
        unsigned incl = warp_incl_scan(nch);
        unsigned total = __shfl_sync(0xffffffffu, incl, 31);
        unsigned long long wb = 0;
        if (lane == 31) wb = atomicAdd(&p.ctl->chunk_top, (unsigned long long)total);
        wb = __shfl_sync(0xffffffffu, wb, 31);
        if (wb + total > p.ck_cap) {
            if (lane == 0) {
                atomicOr(&p.ctl->error, kErrChunks);
                atomicMax(&p.ctl->need_chunks, wb + total);
            }
            continue;
        }
        unsigned long long my = wb + incl - nch;
        if (v) {
            p.net_ck[p.P + gi] = (uint32_t)my;
            p.net_nck[p.P + gi] = nch;
            p.gate_done[gi] = 0;
            // chunk start times: quantiles of the longest fan-in's transition times
            const GateInfo g = p.gate[gi];
            unsigned long long lenref = 0;
            uint32_t ref = 0;
            for (uint32_t i = 0; i < g.k; ++i) {
                const uint32_t src = p.pin_src[g.pin_off + i];
                const unsigned long long len = p.net_len[src];
                if (len > lenref) { lenref = len; ref = src; }
            }
            for (unsigned c = 0; c < nch; ++c) {
                const unsigned long long q = lenref / nch, rm = lenref % nch;
                p.ck_T[my + c] = c == 0 ? 0 : time_at(p, ref, (unsigned long long)c * q + ((unsigned long long)c * rm) / nch);
            }
        }
        // the warp writes the chunk -> gate map of its 32 gates cooperatively
        for (int j = 0; j < 32; ++j) {
            unsigned nj = __shfl_sync(0xffffffffu, nch, j);
            unsigned long long bj = __shfl_sync(0xffffffffu, my, j);
            for (unsigned c = lane; c < nj; c += 32) p.ck_gate[bj + c] = (uint32_t)(g0 + base + j);
        }
    }
}

// ------------------------------------------------------------------ phase B
__device__ void setup_chunk(const SimParams& p, unsigned long long id, ChunkSetup& s,
                            uint32_t& g_out, uint32_t& c_out, uint32_t& nch_out,
                            unsigned long long* q0_out = nullptr, unsigned long long* q1_out = nullptr,
                            uint32_t* ref_out = nullptr, unsigned long long* nin_out = nullptr) {
    const uint32_t gi = __ldcg(&p.ck_gate[id]);
    const GateInfo g = p.gate[gi];
    const uint32_t base = __ldcg(&p.net_ck[p.P + gi]), nch = __ldcg(&p.net_nck[p.P + gi]);
    const uint32_t c = (uint32_t)(id - base);
    s.k = g.k;
    s.lut_base = g.lut_base;
    s.pin_off = g.pin_off;
    unsigned long long lenref = 0, n_in = 0;
    uint32_t ref = 0;
    uint32_t dmin = 0xffffffffu, dmax = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if ((uint32_t)i < g.k) {
            uint32_t src = p.pin_src[g.pin_off + i];
            s.src[i] = src;
            uint4 d = p.pin_delay[g.pin_off + i];
            s.d[i] = d;
            const uint32_t f[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)                   // finite delays only (GLS_DELAY_INF: no relation)
                if (f[q] != kDelayInf) {
                    dmin = min(dmin, f[q]);
                    dmax = max(dmax, f[q]);
                }
            unsigned long long len = __ldcg(&p.net_len[src]);
            n_in += len;
            if (len > lenref) { lenref = len; ref = src; }
        } else {
            s.src[i] = 0;
            s.d[i] = make_uint4(0, 0, 0, 0);
        }
    }
    s.dmin = dmin == 0xffffffffu ? 0u : dmin;
    s.dmax = dmax;
    s.inf = (g.flags & kGateInf) != 0;
    // chunk boundaries: quantiles of the longest fan-in's transition times
    auto qidx = [&](uint32_t cc) -> unsigned long long {
        unsigned long long q = lenref / nch, rm = lenref % nch;
        return (unsigned long long)cc * q + ((unsigned long long)cc * rm) / nch;
    };
    // chunk start times are written when the gate is planned (plan_gate / plan_level)
    s.T0 = __ldcg(&p.ck_T[id]);
    s.T1 = c + 1 == nch ? p.duration + 1 : __ldcg(&p.ck_T[id + 1]);
    if (q0_out) *q0_out = qidx(c);
    if (q1_out) *q1_out = c + 1 == nch ? lenref : qidx(c + 1);
    if (ref_out) *ref_out = ref;
    if (nin_out) *nin_out = n_in;
    // halo: H = dmax + 1 (reading R17 for one gate); tau0 may be negative
    s.tau0 = s.T0 - (long long)dmax - 1;
    g_out = gi;
    c_out = c;
    nch_out = nch;
}

__device__ void process_level(const SimParams& p, unsigned long long ck_begin, unsigned long long ck_end,
                              unsigned long long* work, const uint8_t* lut) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned long long n = ck_end - ck_begin;
    for (;;) {
        if (lane == 0) p.deep_wtop[warp_global_id()] = 0;   // per-warp deep scratch, reused per batch
        __syncwarp();
        unsigned long long wb = 0;
        if (lane == 0) wb = atomicAdd(work, 32ull);
        wb = __shfl_sync(0xffffffffu, wb, 0);
        if (wb >= n) break;
        const unsigned long long id = ck_begin + wb + lane;
        const bool active = wb + lane < n;

        ChunkSetup s;
        ChunkOut r{0, 0, 0, 2, false};
        uint32_t gi = 0, c = 0, nch = 1;
        bool deep = false;
        uint64_t* dbuf = nullptr;
        unsigned long long dcap = 0;
        if (active) {
            setup_chunk(p, id, s, gi, c, nch);
            run_chunk<false, false>(p, s, lut, nullptr, nullptr, 0, r);
            if (r.overflow) {
                // deep backtrace: exact path with a scratch ring sized by the window
                deep = true;
                dcap = window_bound(p, s);
                const unsigned long long at = deep_alloc(p, dcap);
                atomicAdd(&p.ctl->deep_chunks, 1ull);
                if (at == ~0ull) {
                    deep = false;
                    r.cnt = 0;
                } else {
                    dbuf = p.deep + at;
                    run_chunk<false, true>(p, s, lut, nullptr, dbuf, dcap, r);
                    if (r.overflow) atomicOr(&p.ctl->error, kErrBug);
                }
            }
        }
        // exact output allocation: warp scan + one bump per warp (no page waste)
        unsigned incl = warp_incl_scan(r.cnt);
        unsigned total = __shfl_sync(0xffffffffu, incl, 31);
        unsigned long long ab = 0;
        if (lane == 31) ab = atomicAdd(&p.ctl->arena_top, (unsigned long long)total);
        ab = __shfl_sync(0xffffffffu, ab, 31);
        const bool fits = ab + total <= p.arena_cap;
        if (!fits && lane == 0) {
            atomicOr(&p.ctl->error, kErrArena);
            atomicMax(&p.ctl->need_arena, ab + total);
        }
        const unsigned long long my = ab + incl - r.cnt;
        if (active && fits) {
            ChunkOut r2{0, 0, 0, 2, false};
            if (deep)
                run_chunk<true, true>(p, s, lut, p.arena + my, dbuf, dcap, r2);
            else
                run_chunk<true, false>(p, s, lut, p.arena + my, nullptr, 0, r2);
            if (r2.cnt != r.cnt) atomicOr(&p.ctl->error, kErrBug);
            p.ck_T[id] = s.T0;
            p.ck_off[id] = my;
            p.ck_cnt[id] = r.cnt;
            p.ck_vb[id] = (uint8_t)r.vb;
            // release (no L1 invalidation, unlike __threadfence): this chunk's
            // descriptor is visible before the gate's done counter moves
            const unsigned prev = atom_add_release(&p.gate_done[gi], 1u);
            if (prev == nch - 1) {
                fence_acquire();
                // last chunk of the gate: prefix counts + net length (strong loads
                // read L2, never a stale L1 line)
                const uint32_t base = __ldcg(&p.net_ck[p.P + gi]);
                unsigned long long cum = 0;
                for (uint32_t j = 0; j < nch; ++j) {
                    p.ck_cum[base + j] = cum;
                    cum += ld_relaxed_u32(&p.ck_cnt[base + j]);
                }
                p.net_len[p.P + gi] = cum;
            }
        }
        unsigned long long se = warp_sum64(active ? r.evals : 0u);
        unsigned long long sv = warp_sum64(active ? r.events : 0u);
        unsigned long long sc = warp_sum64(active ? 1ull : 0ull);
        if (lane == 0) {
            atomicAdd(&p.ctl->gate_evals, se);
            atomicAdd(&p.ctl->events, sv);
            atomicAdd(&p.ctl->out_trans, (unsigned long long)total);
            atomicAdd(&p.ctl->chunks, sc);
        }
    }
}

// ------------------------------------------------------------------ chunk results, gates, dataflow
struct ChunkResult {
    ChunkSetup s;
    uint32_t gi, nch;
    unsigned long long off, evals, events;
    uint32_t total, vb;
    bool fits;
};

// The per-lane engine on one lane: count pass, exact allocation, write pass
// (deep ring if the 32-entry ring overflows).  Used when a chunk defeats an
// engine's bounded on-chip state.
__device__ __noinline__ void lane_chunk(const SimParams& p, const ChunkSetup& s, const uint8_t* lut,
                                        unsigned long long& off, uint32_t& cnt, uint32_t& vb,
                                        unsigned long long& evals, unsigned long long& events, bool& fits) {
    ChunkOut r{0, 0, 0, 2, false};
    run_chunk<false, false>(p, s, lut, nullptr, nullptr, 0, r);
    bool deep = false;
    uint64_t* dbuf = nullptr;
    unsigned long long dcap = 0;
    if (r.overflow) {
        deep = true;
        dcap = window_bound(p, s);
        const unsigned long long at = deep_alloc(p, dcap);
        if (at == ~0ull) {
            fits = false;
            cnt = 0;
            return;
        }
        dbuf = p.deep + at;
        run_chunk<false, true>(p, s, lut, nullptr, dbuf, dcap, r);
        if (r.overflow) atomicOr(&p.ctl->error, kErrBug);
    }
    off = r.cnt ? atomicAdd(&p.ctl->arena_top, seg_round(r.cnt)) : 0ull;
    fits = off + r.cnt <= p.arena_cap;
    if (!fits) {
        atomicOr(&p.ctl->error, kErrArena);
        atomicMax(&p.ctl->need_arena, off + r.cnt);
    } else {
        ChunkOut r2{0, 0, 0, 2, false};
        if (deep)
            run_chunk<true, true>(p, s, lut, p.arena + off, dbuf, dcap, r2);
        else
            run_chunk<true, false>(p, s, lut, p.arena + off, nullptr, 0, r2);
        if (r2.cnt != r.cnt) atomicOr(&p.ctl->error, kErrBug);
    }
    cnt = r.cnt;
    vb = r.vb;
    evals = r.evals;
    events = r.events;
}

// Whole warp: make gate c schedulable — nch = ceil(n_in / M) chunks (at most
// len(longest fan-in) + 1), chunk ids from the shared queue, chunk -> gate map
// written last (publication; consumers spin on it).
__device__ void plan_gate(const SimParams& p, uint32_t c) {
    const int lane = threadIdx.x & 31;
    const GateInfo g = p.gate[c];
    const uint32_t my_src = (uint32_t)lane < g.k ? p.pin_src[g.pin_off + lane] : 0u;
    const unsigned long long len = (uint32_t)lane < g.k ? __ldcg(&p.net_len[my_src]) : 0ull;
    const unsigned long long n_in = warp_sum64(len), lenref = warp_max64(len);
    // longest fan-in (first such pin): its quantiles are the chunk boundaries
    const unsigned bm = __ballot_sync(0xffffffffu, (uint32_t)lane < g.k && len == lenref);
    const uint32_t ref = __shfl_sync(0xffffffffu, my_src, __ffs(bm) - 1);
    unsigned long long nch = (n_in + (unsigned long long)p.M - 1) / (unsigned long long)p.M;
    if (nch < 1) nch = 1;
    if (nch > lenref + 1) nch = lenref + 1;
    if (g.flags & kGateInf) nch = 1;                    // no halo starts with unrelated pins (reading R9)
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&p.ctl->chunk_top, nch);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base + nch > p.ck_cap) {
        if (lane == 0) {
            atomicOr(&p.ctl->error, kErrChunks);
            atomicMax(&p.ctl->need_chunks, base + nch);
        }
        return;
    }
    if (lane == 0) {
        if (p.trace) p.trace[8ull * c] = gtimer();
        p.net_ck[p.P + c] = (uint32_t)base;
        p.net_nck[p.P + c] = (uint32_t)nch;
        p.gate_nin[c] = n_in;
        p.gate_done[c] = 0;
        fence_release();
    }
    // chunk start times: quantiles of the longest fan-in's transition times
    GLS_ASSERT(base + nch <= p.ck_cap);
    for (unsigned long long j = lane; j < nch; j += 32) {
        const unsigned long long q = lenref / nch, rm = lenref % nch;
        p.ck_T[base + j] = j == 0 ? 0 : time_at(p, ref, j * q + (j * rm) / nch);
    }
    fence_release();
    __syncwarp();
    for (unsigned long long j = lane; j < nch; j += 32) st_relaxed_u32(&p.ck_gate[base + j], c);
}

// Whole warp: the last chunk of gate gi finished — prefix counts, net length,
// and (dataflow) unlock the consumers whose last fan-in this was (Alg. 1).
template <bool DATAFLOW>
__device__ void gate_complete(const SimParams& p, uint32_t gi, uint32_t base, uint32_t nch) {
    const int lane = threadIdx.x & 31;
    unsigned long long cum = 0;
    for (uint32_t j0 = 0; j0 < nch; j0 += 32) {
        const uint32_t j = j0 + lane;
        const unsigned long long c = j < nch ? ld_relaxed_u32(&p.ck_cnt[base + j]) : 0ull;
        unsigned long long x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (j < nch) p.ck_cum[base + j] = cum + x - c;
        cum += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) {
        p.net_len[p.P + gi] = cum;
        if (p.trace) p.trace[8ull * gi + 1] = gtimer();
    }
    if (!DATAFLOW) return;
    fence_release();
    __syncwarp();
    const uint32_t net = (uint32_t)p.P + gi;
    const uint32_t f0 = p.fo_off[net], f1 = p.fo_off[net + 1];
    for (uint32_t e0 = f0; e0 < f1; e0 += 32) {
        const uint32_t e = e0 + (uint32_t)lane;
        uint32_t cg = 0;
        bool ready = false;
        if (e < f1) {
            cg = p.fo_gate[e];
            ready = atom_add_release(&p.pend[cg], 0xffffffffu) == 1u;   // decrement; the last one plans cg
        }
        const unsigned rdy = __ballot_sync(0xffffffffu, ready);
        if (rdy) fence_acquire();                       // (every lane: plan_gate reads the fan-ins' lengths)
        for (unsigned rb = rdy; rb; rb &= rb - 1) {
            const int src = __ffs(rb) - 1;
            plan_gate(p, __shfl_sync(0xffffffffu, cg, src));
        }
    }
    __syncwarp();
    if (lane == 0) atomicAdd(&p.ctl->done_gates, 1ull);
}

// Whole warp: record a finished chunk (descriptor, stats); the gate's last
// chunk completes the gate.
template <bool DATAFLOW>
__device__ void chunk_done(const SimParams& p, unsigned long long id, const ChunkResult& R,
                           unsigned long long* acc = nullptr) {
    const int lane = threadIdx.x & 31;
    unsigned prev = 0;
    if (lane == 0) {
        GLS_ASSERT(id < p.ck_cap && R.gi < (uint32_t)p.G);
        GLS_ASSERT(!R.fits || R.off + R.total <= p.arena_cap);
        if (R.fits) {
            p.ck_T[id] = R.s.T0;
            p.ck_off[id] = R.off;
            p.ck_cnt[id] = R.total;
            p.ck_vb[id] = (uint8_t)R.vb;
            prev = atom_add_release(&p.gate_done[R.gi], 1u);
        }
        if (acc) {                                      // per-warp statistics (slice engine)
            acc[0] += R.evals;
            acc[1] += R.events;
            acc[2] += (unsigned long long)R.total;
            acc[3] += 1ull;
        } else {
            atomicAdd(&p.ctl->gate_evals, R.evals);
            atomicAdd(&p.ctl->events, R.events);
            atomicAdd(&p.ctl->out_trans, (unsigned long long)R.total);
            atomicAdd(&p.ctl->chunks, 1ull);
        }
    }
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (R.fits && prev == R.nch - 1) {
        if (R.nch > 1) fence_acquire();                 // (every lane: the last chunk reads the others' counts)
        gate_complete<DATAFLOW>(p, R.gi, __ldcg(&p.net_ck[p.P + R.gi]), R.nch);
    }
    __syncwarp();
}


}  // namespace gls
#include "gls_lanes.cuh"
namespace gls {
constexpr int kCsrpStack = 1024;    // engine 2: a thread's individual memory (entries)
}
#include "gls_csrp.cuh"
namespace gls {

#ifndef GLS_MINB
#define GLS_MINB 3
#endif
template <int ENGINE, bool DATAFLOW>
__global__ void __launch_bounds__(kThreads, GLS_MINB) sim_kernel(const __grid_constant__ SimParams p) {
    uint8_t* const s_lut = ln::g_lut;
    for (int i = threadIdx.x; i < kLutCap; i += blockDim.x) s_lut[i] = p.lut[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned warps_per_block = blockDim.x >> 5;
    const unsigned gwarp = blockIdx.x * warps_per_block + (threadIdx.x >> 5);
    const unsigned nwarps = gridDim.x * warps_per_block;
    if (DATAFLOW) {
        // seed: gates fed only by given nets (topological level 1) are ready now
        for (int g = (int)gwarp; g < p.level_off[1]; g += (int)nwarps) plan_gate(p, (uint32_t)g);
        // pull published chunks until every gate is complete (Alg. 1 loop)
        unsigned long long carry = ~0ull;
        if (lane == 0) ln::acc_zero(ln::warp_batch());
        while (ln::lane_batch<true>(p, carry, 0, 0, nullptr)) {
        }
        if (lane == 0) ln::acc_flush(p, ln::warp_batch());
    } else {
        unsigned gen = 0;
        unsigned long long ck_begin = (unsigned long long)p.P;
        if (ENGINE == 0 && lane == 0) ln::acc_zero(ln::warp_batch());
        for (int l = 1; l <= p.L; ++l) {
            plan_level(p, l, gwarp, nwarps);
            if (grid_barrier(p.ctl, p.nblocks, gen)) return;
            const unsigned long long ck_end = *(volatile unsigned long long*)&p.ctl->chunk_top;
            if (ENGINE == 1) {
                process_level(p, ck_begin, ck_end, &p.work[l], s_lut);
            } else {
                unsigned long long carry = ~0ull;
                while (ln::lane_batch<false>(p, carry, ck_begin, ck_end - ck_begin, &p.work[l])) {
                }
                if (lane == 0) ln::acc_flush(p, ln::warp_batch());   // (before the barrier: counts are read after it)
            }
            if (grid_barrier(p.ctl, p.nblocks, gen)) return;
            ck_begin = ck_end;
        }
    }
}

// given nets: one chunk each, covering the whole duration
__global__ void init_given_kernel(SimParams p, const long long* in_off) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.P; i += gridDim.x * blockDim.x) {
        long long a = in_off[i], b = in_off[i + 1];
        p.net_ck[i] = (uint32_t)i;
        p.net_nck[i] = 1;
        p.net_len[i] = (unsigned long long)(b - a);
        p.ck_T[i] = 0;
        p.ck_off[i] = (unsigned long long)a;
        p.ck_cnt[i] = (uint32_t)(b - a);
        p.ck_cum[i] = 0;
        p.ck_vb[i] = 2;
        p.ck_gate[i] = 0xffffffffu;
    }
}

// ------------------------------------------------------------------ time windows
// One net's slice for a window: [ia, ib) = the transitions with t_clamp < t < t_end;
// the earlier ones collapse into one at t_clamp carrying the last value (kept unless X,
// which every net starts at — reading R6/R17).
__device__ __forceinline__ void window_range(const long long* off, const uint64_t* tr, int i, long long t_clamp,
                                             long long t_end, long long& ia, long long& ib, int& collapse,
                                             uint64_t& ce) {
    const long long a = off[i], b = off[i + 1];
    long long lo = a, hi = b;                          // first index with t > t_clamp
    while (lo < hi) {
        const long long m = (lo + hi) >> 1;
        if ((long long)(tr[m] >> 2) <= t_clamp) lo = m + 1; else hi = m;
    }
    ia = lo;
    hi = b;                                            // first index with t >= t_end
    while (lo < hi) {
        const long long m = (lo + hi) >> 1;
        if ((long long)(tr[m] >> 2) < t_end) lo = m + 1; else hi = m;
    }
    ib = lo;
    collapse = 0;
    ce = 0;
    if (ia > a && (tr[ia - 1] & 3u) != 2u) {
        collapse = 1;
        ce = ((uint64_t)t_clamp << 2) | (tr[ia - 1] & 3u);
    }
}
__global__ void window_count_kernel(int32_t P, const long long* off, const uint64_t* tr, long long t_clamp,
                                    long long t_end, long long* cnt) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
        long long ia, ib;
        int c;
        uint64_t ce;
        window_range(off, tr, i, t_clamp, t_end, ia, ib, c, ce);
        cnt[i] = c + (ib - ia);
    }
}
// one warp per net: coalesced copy of the kept range
__global__ void window_fill_kernel(int32_t P, const long long* off, const uint64_t* tr, long long t_clamp,
                                   long long t_end, const long long* new_off, uint64_t* out) {
    const int lane = threadIdx.x & 31;
    const int nw = (int)((gridDim.x * blockDim.x) >> 5);
    for (int i = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < P; i += nw) {
        long long ia = 0, ib = 0;
        int c = 0;
        uint64_t ce = 0;
        if (lane == 0) window_range(off, tr, i, t_clamp, t_end, ia, ib, c, ce);
        ia = __shfl_sync(0xffffffffu, ia, 0);
        ib = __shfl_sync(0xffffffffu, ib, 0);
        c = __shfl_sync(0xffffffffu, c, 0);
        ce = __shfl_sync(0xffffffffu, ce, 0);
        uint64_t* dst = out + new_off[i];
        if (lane == 0 && c) dst[0] = ce;
        for (long long j = ia + lane; j < ib; j += 32) dst[c + (j - ia)] = tr[j];
    }
}

// validation of device-resident given waveforms (same rules as the host path):
// one warp per net, each lane checks consecutive pairs (coalesced): strictly
// increasing times < 2^61, every transition changes the value, the first one
// is not X (R6: every net starts at X).
__global__ void validate_kernel(int32_t P, const long long* off, const uint64_t* tr, long long total,
                                unsigned* err, unsigned long long* maxt) {
    const int lane = threadIdx.x & 31;
    const int nw = (int)((gridDim.x * blockDim.x) >> 5);
    unsigned long long mx = 0;
    for (int i = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < P; i += nw) {
        const long long a = off[i], b = off[i + 1];
        if (a < 0 || b < a || b > total) {
            if (lane == 0) atomicOr(err, 1u);
            continue;
        }
        bool bad = false;
        for (long long j = a + lane; j < b; j += 32) {
            const uint64_t e = tr[j];
            const long long t = (long long)(e >> 2);
            const uint32_t v = (uint32_t)(e & 3u);
            uint64_t pe = 2;                            // the value before the first transition: X
            long long pt = -1;
            if (j > a) {
                pe = tr[j - 1];
                pt = (long long)(pe >> 2);
            }
            bad |= t <= pt || v == (uint32_t)(pe & 3u) || t >= (1ll << 61);
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, 2u);
        if (lane == 0 && b > a) mx = max(mx, (unsigned long long)(tr[b - 1] >> 2));
    }
    if (lane == 0 && mx) atomicMax(maxt, mx);          // one same-address atomic per warp, not per net
    if (blockIdx.x == 0 && threadIdx.x == 0 && off[0] != 0) atomicOr(err, 1u);
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// Per-net results checksum, written in user net order: one warp per
// net, coalesced loads of its chunk segments, position-keyed terms XOR-reduced.
constexpr uint64_t kHashC = 0x9E3779B97F4A7C15ull, kHashK = 0xD1B54A32D192ED03ull;
__global__ void hash_kernel(SimParams p, const uint32_t* perm, uint64_t* out) {
    const int N = p.P + p.G;
    const int lane = threadIdx.x & 31;
    const int nw = (int)((gridDim.x * blockDim.x) >> 5);
    for (int n = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); n < N; n += nw) {
        const uint32_t cb = p.net_ck[n], nck = p.net_nck[n];
        uint64_t h = 0, pos = 0;                       // pos: index of the chunk's first entry
        for (uint32_t j = cb; j < cb + nck; ++j) {
            const uint64_t* s = p.arena + p.ck_off[j];
            const uint32_t c = p.ck_cnt[j];
            uint32_t q = lane;
            for (; q + 96 < c; q += 128) {             // 4 independent loads in flight per lane
                const uint64_t e0 = __ldcs(s + q), e1 = __ldcs(s + q + 32), e2 = __ldcs(s + q + 64),
                               e3 = __ldcs(s + q + 96);
                h ^= splitmix64(e0 + (pos + q + 1) * kHashK) ^ splitmix64(e1 + (pos + q + 33) * kHashK) ^
                     splitmix64(e2 + (pos + q + 65) * kHashK) ^ splitmix64(e3 + (pos + q + 97) * kHashK);
            }
            for (; q < c; q += 32) h ^= splitmix64(__ldcs(s + q) + (pos + q + 1) * kHashK);
            pos += c;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) h ^= __shfl_xor_sync(0xffffffffu, h, o);
        if (lane == 0) {
            const int user = n < p.P ? n : p.P + (int)perm[n - p.P];
            out[user] = h ^ splitmix64(kHashC ^ (uint64_t)p.net_len[n]);
        }
    }
}

// Same checksum over the transitions with t_lo <= t <= t_hi (contiguous in each net:
// positions counted from the first of them, found with count_before).
__global__ void hash_window_kernel(SimParams p, const uint32_t* perm, long long t_lo, long long t_hi, uint64_t* out) {
    const int N = p.P + p.G;
    const int lane = threadIdx.x & 31;
    const int nw = (int)((gridDim.x * blockDim.x) >> 5);
    for (int n = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); n < N; n += nw) {
        const uint32_t cb = p.net_ck[n], nck = p.net_nck[n];
        const unsigned long long i0 = count_before(p, (uint32_t)n, t_lo);
        const unsigned long long i1 = t_hi == LLONG_MAX ? (unsigned long long)p.net_len[n]
                                                         : count_before(p, (uint32_t)n, t_hi + 1);
        uint64_t h = 0;
        for (uint32_t j = cb; j < cb + nck && i1 > i0; ++j) {
            const unsigned long long c0 = p.ck_cum[j], c = p.ck_cnt[j];
            if (c0 + c <= i0 || c0 >= i1) continue;    // chunk outside the window
            const uint64_t* s = p.arena + p.ck_off[j];
            const unsigned long long qa = i0 > c0 ? i0 - c0 : 0ull, qb = min(c, i1 - c0);
            for (unsigned long long q = qa + lane; q < qb; q += 32) h ^= splitmix64(s[q] + (c0 + q - i0 + 1) * kHashK);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) h ^= __shfl_xor_sync(0xffffffffu, h, o);
        if (lane == 0) {
            const int user = n < p.P ? n : p.P + (int)perm[n - p.P];
            out[user] = h ^ splitmix64(kHashC ^ (uint64_t)(i1 > i0 ? i1 - i0 : 0ull));
        }
    }
}

// time-window stitching pieces: one warp per net (user order out), like hash_window_kernel
// but with the window's position keyed from base[user] and the length term optional
__global__ void hash_terms_kernel(SimParams p, const uint32_t* perm, long long t_lo, long long t_hi,
                                  const long long* base, const long long* total, long long* counts,
                                  uint64_t* terms) {
    const int N = p.P + p.G;
    const int lane = threadIdx.x & 31;
    const int nw = (int)((gridDim.x * blockDim.x) >> 5);
    for (int n = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); n < N; n += nw) {
        const int user = n < p.P ? n : p.P + (int)perm[n - p.P];
        const unsigned long long i0 = count_before(p, (uint32_t)n, t_lo);
        const unsigned long long i1 = t_hi == LLONG_MAX ? (unsigned long long)p.net_len[n]
                                                         : count_before(p, (uint32_t)n, t_hi + 1);
        const unsigned long long cnt = i1 > i0 ? i1 - i0 : 0ull;
        if (terms) {
            const unsigned long long b = base ? (unsigned long long)base[user] : 0ull;
            const uint32_t cb = p.net_ck[n], nck = p.net_nck[n];
            uint64_t h = 0;
            for (uint32_t j = cb; j < cb + nck && cnt; ++j) {
                const unsigned long long c0 = p.ck_cum[j], c = p.ck_cnt[j];
                if (c0 + c <= i0 || c0 >= i1) continue;    // chunk outside the window
                const uint64_t* s = p.arena + p.ck_off[j];
                const unsigned long long qa = i0 > c0 ? i0 - c0 : 0ull, qb = min(c, i1 - c0);
                for (unsigned long long q = qa + lane; q < qb; q += 32)
                    h ^= splitmix64(s[q] + (b + c0 + q - i0 + 1) * kHashK);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) h ^= __shfl_xor_sync(0xffffffffu, h, o);
            if (lane == 0) terms[user] = total ? h ^ splitmix64(kHashC ^ (uint64_t)total[user]) : h;
        }
        if (lane == 0) counts[user] = (long long)cnt;
    }
}


// ------------------------------------------------------------------ result readback (a10, GK3)
// Canonical CSR on the device: user nets [u0, u1) in net order, each net's transitions
// with t_lo <= t <= t_hi (the whole run: LLONG_MIN, LLONG_MAX), gathered from its chunk
// segments.  The paper transfers the finished store to the CPU as the output;
// here the store is permuted into the caller's order on the device first, so the host
// receives one contiguous CSR (or a device consumer — NCCL stitching — reads it).
__device__ __forceinline__ uint32_t internal_net(const SimParams& p, const uint32_t* inv, long long u) {
    return u < p.P ? (uint32_t)u : (uint32_t)p.P + inv[u - p.P];
}
__device__ __forceinline__ void net_range(const SimParams& p, uint32_t n, long long t_lo, long long t_hi,
                                          unsigned long long& i0, unsigned long long& i1) {
    i0 = t_lo == LLONG_MIN ? 0ull : count_before(p, n, t_lo);
    i1 = t_hi == LLONG_MAX ? (unsigned long long)p.net_len[n] : count_before(p, n, t_hi + 1);
    if (i1 < i0) i1 = i0;
}
__global__ void range_counts_kernel(SimParams p, const uint32_t* inv, long long u0, long long u1, long long t_lo,
                                    long long t_hi, long long* cnt) {
    for (long long u = u0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; u < u1;
         u += (long long)gridDim.x * blockDim.x) {
        unsigned long long i0, i1;
        net_range(p, internal_net(p, inv, u), t_lo, t_hi, i0, i1);
        cnt[u - u0] = (long long)(i1 - i0);
    }
}
// one warp per net: coalesced copy of the net's [i0, i1) across its chunk segments
__global__ void range_gather_kernel(SimParams p, const uint32_t* inv, long long u0, long long u1, long long t_lo,
                                    long long t_hi, const long long* off, uint64_t* dst) {
    const int lane = threadIdx.x & 31;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long u = u0 + (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5); u < u1; u += nw) {
        const uint32_t n = internal_net(p, inv, u);
        unsigned long long i0, i1;
        net_range(p, n, t_lo, t_hi, i0, i1);
        uint64_t* d = dst + off[u - u0];
        const uint32_t cb = p.net_ck[n], nck = p.net_nck[n];
        for (uint32_t j = cb; j < cb + nck && i1 > i0; ++j) {
            const unsigned long long c0 = p.ck_cum[j], c = p.ck_cnt[j];
            if (c0 + c <= i0 || c0 >= i1) continue;    // chunk outside the range
            const uint64_t* s = p.arena + p.ck_off[j];
            const unsigned long long qa = i0 > c0 ? i0 - c0 : 0ull, qb = min(c, i1 - c0);
            for (unsigned long long q = qa + lane; q < qb; q += 32) d[c0 + q - i0] = __ldcs(s + q);
        }
    }
}
// segment i (src_off[i] .. src_off[i+1]) -> dst + dst_off[i]; one warp per segment
__global__ void scatter_segments_kernel(long long nseg, const long long* src_off, const uint64_t* src,
                                        const long long* dst_off, uint64_t* dst) {
    const int lane = threadIdx.x & 31;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nseg; i += nw) {
        const long long a = src_off[i], b = src_off[i + 1], o = dst_off[i];
        for (long long q = a + lane; q < b; q += 32) dst[o + (q - a)] = src[q];
    }
}

// sum over nets of len x fan-out (measurement only)
__global__ void fanin_reads_kernel(const unsigned long long* len, const uint32_t* fo, long long n,
                                   unsigned long long* out) {
    unsigned long long acc = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        acc += len[i] * (unsigned long long)fo[i];
    acc = warp_sum64(acc);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// ------------------------------------------------------------------ launchers
static size_t dyn_smem(int engine) {
    return engine == 0 ? ln::kDynBytes : 0;
}
static const void* kernel_for(int engine, int sched) {
    if (engine == 1) return (const void*)sim_kernel<1, false>;
    return sched == 1 ? (const void*)sim_kernel<0, false> : (const void*)sim_kernel<0, true>;
}

size_t warp_aux_bytes(int blocks) { return (size_t)blocks * (kThreads / 32) * sizeof(ln::WarpAux); }

size_t warp_scratch_entries(int blocks) {
    return (size_t)blocks * (kThreads / 32) * ln::kScratchPerWarp;
}

int max_coresident_blocks(int device, int engine, int sched, int* per_sm) {
    int nb = 0, sms = 0;
    const void* k = kernel_for(engine, sched);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_smem(engine));
    // shared-memory carveout: just what the resident CTAs need (the rest stays L1, which
    // caches the fan-in entries the sweep reads: engine 0 at 3 CTAs/SM keeps ~92 KB)
    if (engine == 0) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, k);
        int maxsm = 0, want = 3;
        cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
        const size_t per = fa.sharedSizeBytes + dyn_smem(engine) + 1024;      // + the per-CTA reservation
        if (maxsm > 0) {
            const int pct = (int)((want * per * 100 + (size_t)maxsm - 1) / (size_t)maxsm);
            cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct > 100 ? 100 : pct);
        }
    }
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, kThreads, dyn_smem(engine));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (per_sm) *per_sm = nb;
    return nb * sms;
}


// ---- engine 2 (the paper's CSRP store and Alg. 1, gls_csrp.cuh)
constexpr int kCsrpThreads = 128;
int csrp_coresident_threads(int device) {
    int nb = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)cp::csrp_kernel, kCsrpThreads, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return nb * sms * kCsrpThreads;
}
size_t csrp_scratch_entries(int threads) { return (size_t)threads * kCsrpStack; }
cudaError_t launch_csrp(const SimParams& p, uint64_t* pages, unsigned long long* page_top,
                        unsigned long long page_cap, uint32_t pagelen, unsigned long long* first_page,
                        uint32_t* known, unsigned long long* out_cnt, const long long* in_off, int threads,
                        cudaStream_t s) {
    cp::CsrpParams c{pages, page_top, page_cap, pagelen, first_page, known, out_cnt};
    if (p.P > 0) {
        int blocks = (p.P + 255) / 256;
        if (blocks > 4096) blocks = 4096;
        cp::csrp_given_kernel<<<blocks, 256, 0, s>>>(p, c, in_off);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (p.G == 0) return cudaSuccess;
    SimParams q = p;
    void* args[] = {&q, &c};
    return cudaLaunchCooperativeKernel((const void*)cp::csrp_kernel, dim3(threads / kCsrpThreads), dim3(kCsrpThreads),
                                       args, 0, s);
}
cudaError_t launch_csrp_collect(const SimParams& p, uint64_t* pages, uint32_t pagelen, unsigned long long* first_page,
                                unsigned long long* out_cnt, const unsigned long long* seg_off, cudaStream_t s) {
    if (p.G == 0) return cudaSuccess;
    cp::CsrpParams c{pages, nullptr, 0, pagelen, first_page, nullptr, out_cnt};
    long long blocks = ((long long)p.G + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    cp::csrp_collect_kernel<<<(unsigned)blocks, 256, 0, s>>>(p, c, seg_off);
    return cudaGetLastError();
}

cudaError_t launch_simulate(const SimParams& p, int blocks, cudaStream_t s) {
    SimParams q = p;
    q.nblocks = (uint32_t)blocks;
    void* args[] = {&q};
    return cudaLaunchCooperativeKernel(kernel_for(p.engine, p.sched), dim3(blocks), dim3(kThreads), args,
                                       dyn_smem(p.engine), s);
}

cudaError_t launch_init_given(const SimParams& p, const long long* in_off, cudaStream_t s) {
    if (p.P == 0) return cudaSuccess;
    int blocks = (p.P + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    init_given_kernel<<<blocks, 256, 0, s>>>(p, in_off);
    return cudaGetLastError();
}

cudaError_t launch_window_count(int32_t P, const long long* off, const uint64_t* tr, long long t_clamp,
                                long long t_end, long long* cnt, cudaStream_t s) {
    if (P == 0) return cudaSuccess;
    int blocks = (P + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    window_count_kernel<<<blocks, 256, 0, s>>>(P, off, tr, t_clamp, t_end, cnt);
    return cudaGetLastError();
}

cudaError_t launch_window_fill(int32_t P, const long long* off, const uint64_t* tr, long long t_clamp,
                               long long t_end, const long long* new_off, uint64_t* out, cudaStream_t s) {
    if (P == 0) return cudaSuccess;
    int blocks = (P + 7) / 8;                          // one warp per net
    if (blocks > 148 * 16) blocks = 148 * 16;
    window_fill_kernel<<<blocks, 256, 0, s>>>(P, off, tr, t_clamp, t_end, new_off, out);
    return cudaGetLastError();
}

cudaError_t launch_validate_inputs(int32_t P, const long long* off, const uint64_t* tr, long long total,
                                   unsigned* d_err, unsigned long long* d_maxt, cudaStream_t s) {
    int blocks = (P + 7) / 8;                          // one warp per net
    if (blocks < 1) blocks = 1;
    if (blocks > 148 * 16) blocks = 148 * 16;
    validate_kernel<<<blocks, 256, 0, s>>>(P, off, tr, total, d_err, d_maxt);
    return cudaGetLastError();
}

cudaError_t launch_hash_terms(const SimParams& p, const uint32_t* perm, long long t_lo, long long t_hi,
                              const long long* base, const long long* total, long long* counts, uint64_t* terms,
                              cudaStream_t s) {
    const int N = p.P + p.G;
    if (N == 0) return cudaSuccess;
    int blocks = (N + 7) / 8;                          // one warp per net
    if (blocks > 148 * 16) blocks = 148 * 16;
    hash_terms_kernel<<<blocks, 256, 0, s>>>(p, perm, t_lo, t_hi, base, total, counts, terms);
    return cudaGetLastError();
}

cudaError_t launch_range_counts(const SimParams& p, const uint32_t* inv, long long u0, long long u1, long long t_lo,
                                long long t_hi, long long* cnt, cudaStream_t s) {
    if (u1 <= u0) return cudaSuccess;
    long long blocks = (u1 - u0 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    range_counts_kernel<<<(unsigned)blocks, 256, 0, s>>>(p, inv, u0, u1, t_lo, t_hi, cnt);
    return cudaGetLastError();
}
cudaError_t launch_range_gather(const SimParams& p, const uint32_t* inv, long long u0, long long u1, long long t_lo,
                                long long t_hi, const long long* off, uint64_t* dst, cudaStream_t s) {
    if (u1 <= u0) return cudaSuccess;
    long long blocks = (u1 - u0 + 7) / 8;              // one warp per net
    if (blocks > 148 * 16) blocks = 148 * 16;
    range_gather_kernel<<<(unsigned)blocks, 256, 0, s>>>(p, inv, u0, u1, t_lo, t_hi, off, dst);
    return cudaGetLastError();
}
cudaError_t launch_scatter_segments(long long nseg, const long long* src_off, const uint64_t* src,
                                    const long long* dst_off, uint64_t* dst, cudaStream_t s) {
    if (nseg <= 0) return cudaSuccess;
    long long blocks = (nseg + 7) / 8;                 // one warp per segment
    if (blocks > 148 * 16) blocks = 148 * 16;
    scatter_segments_kernel<<<(unsigned)blocks, 256, 0, s>>>(nseg, src_off, src, dst_off, dst);
    return cudaGetLastError();
}

// inclusive prefix sum (CUB); tmp == NULL: *tmp_bytes = the scratch it needs
cudaError_t launch_inclusive_scan(const long long* in, long long* out, long long n, void* tmp, size_t* tmp_bytes,
                                  cudaStream_t s) {
    return cub::DeviceScan::InclusiveSum(tmp, *tmp_bytes, in, out, (int64_t)n, s);
}
cudaError_t launch_fanin_reads(const unsigned long long* len, const uint32_t* fanout, long long n,
                               unsigned long long* out, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    fanin_reads_kernel<<<148 * 4, 256, 0, s>>>(len, fanout, n, out);
    return cudaGetLastError();
}

cudaError_t launch_hashes(const SimParams& p, const uint32_t* perm, uint64_t* out, cudaStream_t s) {
    int N = p.P + p.G;
    if (N == 0) return cudaSuccess;
    int blocks = (N + 7) / 8;                          // one warp per net
    if (blocks > 148 * 16) blocks = 148 * 16;
    hash_kernel<<<blocks, 256, 0, s>>>(p, perm, out);
    return cudaGetLastError();
}

cudaError_t launch_hashes_window(const SimParams& p, const uint32_t* perm, long long t_lo, long long t_hi,
                                 uint64_t* out, cudaStream_t s) {
    int N = p.P + p.G;
    if (N == 0) return cudaSuccess;
    int blocks = (N + 7) / 8;                          // one warp per net
    if (blocks > 148 * 16) blocks = 148 * 16;
    hash_window_kernel<<<blocks, 256, 0, s>>>(p, perm, t_lo, t_hi, out);
    return cudaGetLastError();
}

}  // namespace gls