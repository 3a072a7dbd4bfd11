// gls_slice.cuh — engine 0 (default): one warp per (gate, time-chunk) work item, its
// lanes on balanced time slices of it.  Included by gls_kernels.cu.
//
// A chunk [T0, T1) of gate g is cut into nl <= 32 slices at quantiles of the
// longest fan-in's transition times, so every lane gets about the same number
// of merged input transitions.  A slice is itself an exact time chunk (DESIGN.md
// §4): the lane starts at tau = T_l - (dmax + 1) with the inputs' values there,
// runs Algorithm 2 sequentially over the merged fan-in lists, keeps
// the pending schedules of Eq. 1 in a 4-entry register ring
// (streaming finality: entries with r <= t + dmin are final) and writes the
// change points in [T_l, T_{l+1}) to its output scratch.  The slices' outputs,
// concatenated in lane order, are exactly the chunk's outputs: one prefix sum,
// one atomic for the chunk's exact segment, and a coalesced copy-out.  A lane
// whose ring or scratch overflows sends the whole chunk to the per-lane
// engine's exact deep path.
#pragma once

namespace gls {
namespace sl {

#ifndef GLS_DISCARD
#define GLS_DISCARD 0          // 1: drop the staged output lines from L2 after the copy-out (fewer DRAM
                               // write-backs, but measured 5 % slower on C4 at 3 CTAs/SM)
#endif
#ifndef GLS_PF
#define GLS_PF 1
#endif
#ifndef GLS_MAXSLEEP
#define GLS_MAXSLEEP 8192      // ns: longest back-off of a warp waiting for published work
#endif
#ifndef GLS_ADAPT
#define GLS_ADAPT 1            // batch fill adapts to the queue depth (dataflow scheduler)
#endif
constexpr int RD = 4;                  // register pending ring depth
#ifndef GLS_LCAP
#define GLS_LCAP 2048
#endif
constexpr int LCAP = GLS_LCAP;            // per-lane output scratch entries
constexpr int E_MIN = 32;              // fewest expected transitions per lane
constexpr unsigned FULL = 0xffffffffu;
constexpr size_t kScratchPerWarp = 32u * LCAP;

struct Cur {
    const uint64_t* ptr;
    uint32_t rem, ck, ckend;
};

// next non-empty segment of a net (chunk boundary crossing; by value so the
// cursors stay in registers)
struct Seg {
    const uint64_t* ptr;
    uint32_t rem, ck;
};
__device__ __noinline__ Seg next_segment(const SimParams& p, uint32_t ck, uint32_t ckend) {
    Seg r{nullptr, 0u, ck};
    while (r.rem == 0 && r.ck + 1 < ckend) {
        ++r.ck;
        r.ptr = p.arena + __ldcg(&p.ck_off[r.ck]);
        r.rem = __ldcg(&p.ck_cnt[r.ck]);
    }
    return r;
}

// Sequential Algorithm 2 over one slice.  dtab: this lane's delay table in
// shared memory, [pin*6 + (rise ? 3 : 0) + out value][stride] (R1 for X).
// Returns 0, or 1 on ring overflow, 2 on scratch overflow.
template <bool DIRECT>
__device__ __forceinline__ int run_slice(const SimParams& p, const ChunkSetup& s, const uint8_t* lut,
                                         const uint32_t* dtab, int dstride, uint64_t* out, uint32_t& cnt,
                                         uint32_t& vb, uint32_t& evals, uint32_t& events, uint32_t& iters,
                                         uint32_t cap, long long& c_loc) {
    const long long c_l0 = clock64();
    Cur c[4];
    uint64_t h[4];
    uint32_t xn = 0, x0 = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        h[i] = kInfEntry;
        c[i].ptr = nullptr;
        c[i].rem = 0;
        c[i].ck = c[i].ckend = 0;
        if ((uint32_t)i < s.k) {
            Cursor cc;
            uint32_t init;
            locate(p, s.src[i], s.tau0, cc, init);
            c[i].ptr = cc.ptr;
            c[i].rem = (uint32_t)(cc.end - cc.ptr);
            c[i].ck = cc.ck;
            c[i].ckend = cc.ck_end;
            if (c[i].rem) h[i] = *c[i].ptr;
            xn |= 2u << (2 * i);                       // inputs start at X
            x0 |= norm_code(init) << (2 * i);          // values in effect at tau
        }
    }
    c_loc += clock64() - c_l0;
    const uint32_t lb = s.lut_base;
    const long long T0 = s.T0, T1 = s.T1, dmin = (long long)s.dmin;
    const long long T1e = min(T1, p.duration + 1);     // outputs in [T0, T1) and <= duration (R7)
    uint64_t lim1 = (uint64_t)T1 << 2;                 // entry time >= T1  <=>  entry >= lim1
    uint64_t rg0 = 0, rg1 = 0, rg2 = 0, rg3 = 0;       // pending ring: rg0 newest, rg[rn-1] oldest
    int rn = 0;
    long long ft = LLONG_MAX;                          // time of the oldest pending entry (none: max)
    uint32_t Eprev = 2, lastv = 2;
    uint32_t n_out = 0, n_ev = 0, n_evals = 0;
    vb = 2;
    int status = 0;

    auto emit = [&](uint64_t e) {
        const long long r = etime(e);
        if (r < T0) {
            vb = (uint32_t)(e & 3u);
        } else if (r < T1e) {
            if (DIRECT || n_out < cap) out[n_out] = e;
            ++n_out;
        }
        lastv = (uint32_t)(e & 3u);
    };
    auto front = [&]() -> uint64_t { return rn == 1 ? rg0 : rn == 2 ? rg1 : rn == 3 ? rg2 : rg3; };
    // emit the pending entries with time <= lim (oldest first); keeps ft
    auto drain = [&](long long lim) {
        while (rn > 0) {
            const uint64_t f = front();
            if (etime(f) > lim) {
                ft = etime(f);
                return;
            }
            emit(f);
            --rn;
        }
        ft = LLONG_MAX;
    };
    auto step = [&](long long t, uint32_t nx) {
        if (nx != xn) {
            const uint32_t E = lut[lb + nx];            // calculateSignals
            if (E != Eprev) {                           // "o_k.v is changed" (R4a)
                uint32_t del = 0xffffffffu;
                const uint32_t d = nx ^ xn;
                for (uint32_t cm = (d | (d >> 1)) & 0x55u; cm; cm &= cm - 1) {   // changed pins (R3)
                    const int b = __ffs(cm) - 1;
                    const uint32_t fo = (xn >> b) & 3u, fn = (nx >> b) & 3u;
                    const int q = (b >> 1) * 6 + (rank_code(fn) > rank_code(fo) ? 3 : 0) + (int)E;
                    del = min(del, dtab[q * dstride]);   // min rule
                }
                const long long rr = t + (long long)del;
                // addSignalChange with Eq. 1: deny pending schedules at >= rr
                while (rn > 0 && etime(rg0) >= rr) {
                    rg0 = rg1; rg1 = rg2; rg2 = rg3;
                    --rn;
                }
                if (rn == 0) ft = LLONG_MAX;
                const uint32_t tv = rn > 0 ? (uint32_t)(rg0 & 3u) : lastv;
                if (tv != E) {
                    if (rn == RD) {
                        status = 1;
                        lim1 = 0;                       // stop at the next iteration
                    } else {
                        rg3 = rg2; rg2 = rg1; rg1 = rg0;
                        rg0 = ((uint64_t)rr << 2) | E;
                        if (rn == 0) ft = rr;
                        ++rn;
                    }
                }
                if (t >= T0) ++n_ev;
                Eprev = E;
            }
            xn = nx;
        }
        if (ft <= t + dmin) drain(t + dmin);           // streaming finality
    };

    step(s.tau0, x0);                                   // the slice's halo start
    uint32_t n_it = 0;
    for (;;) {
        ++n_it;
        const uint64_t m = min(min(h[0], h[1]), min(h[2], h[3]));
        if (m >= lim1) break;
        const uint64_t mt = m | 3ull;                  // h[i] <= mt  <=>  pin i changes at t
        const long long t = etime(m);
        uint32_t nx = xn;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (h[i] <= mt) {                          // pin i changes at t
                nx = (nx & ~(3u << (2 * i))) | (norm_code((uint32_t)(h[i] & 3u)) << (2 * i));
                ++c[i].ptr;
                if (--c[i].rem == 0) {
                    const Seg g = next_segment(p, c[i].ck, c[i].ckend);
                    if (g.rem) { c[i].ptr = g.ptr; c[i].rem = g.rem; c[i].ck = g.ck; }
                }
                h[i] = c[i].rem ? *c[i].ptr : kInfEntry;
#if GLS_PF
                if ((((uintptr_t)c[i].ptr) & 127u) == 0 && c[i].rem > 32)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(c[i].ptr + 32));
#endif
            }
        }
        n_evals += (t >= T0);
        step(t, nx);
    }
    drain(T1 - 1);                                      // final for this slice below T1
    cnt = n_out;
    evals = n_evals;
    events = n_ev;
    iters = n_it;
    if (!DIRECT && status == 0 && n_out > cap) status = 2;
    return status;
}

}  // namespace sl
}  // namespace gls
#include "gls_sweep.cuh"
namespace gls {
namespace sl {

// Per-warp batch (lane 0 assembles it from the chunk queue): published chunks
// are claimed until the batch holds about 32 x W_LANE expected transitions;
// then the 32 lanes are spread in proportion to the expected work w = total/32:
// a chunk with at least w gets about est/w lanes, one time slice each (cut at
// quantiles of its longest fan-in); smaller chunks are packed whole, several
// per lane.  Units are assigned in lane order, so the slices of a chunk sit on
// consecutive lanes and a lane's units are contiguous.
#ifndef GLS_WLANE
#define GLS_WLANE 256
#endif
constexpr int W_LANE = GLS_WLANE;           // a batch is filled up to 32 x W_LANE expected transitions
constexpr int W_MIN = 32;              // fewest expected transitions per lane (slice setup cost)
#ifndef GLS_MAXC
#define GLS_MAXC 16
#define GLS_MAXU 48
#endif
constexpr int MAXC = GLS_MAXC;         // chunks per batch
constexpr int MAXU = GLS_MAXU;         // units per batch
// per-warp statistics, accumulated in shared memory and added to Ctl once when the
// warp runs out of work (instead of ~25 same-address atomics per batch)
enum Acc { A_EVALS, A_EVENTS, A_OUTS, A_CHUNKS, A_LANE_IT, A_WARP_IT, A_BATCHES, A_BLANES, A_BEST, A_CYC, A_BAL = A_CYC + 6,
           A_N = A_BAL + 8 };
struct Batch {
    unsigned long long acc[A_N];
    unsigned long long id[MAXC];
    uint8_t nsl[MAXC];                     // slices of the chunk
    uint8_t first_unit[MAXC];
    uint8_t u_chunk[MAXU], u_slice[MAXU];  // unit -> (chunk, slice)
    uint8_t lane_u0[32], lane_nu[32];      // lane -> its units [u0, u0 + nu)
    uint32_t u_cnt[MAXU], u_ev[MAXU], u_evt[MAXU];
    uint16_t u_soff[MAXU];                 // offset of the unit's outputs in its lane scratch
    uint32_t u_pre[MAXU];                  // offset of the unit's outputs inside its chunk
    uint8_t u_vb[MAXU], u_st[MAXU], u_lane[MAXU];
    unsigned long long c_off[MAXC];
    long long c_T0[MAXC];                  // chunk start time (recorded by its slice 0)
    uint32_t c_total[MAXC];
};
constexpr size_t kBatchBytes = sizeof(Batch);

// this unit's time range: the chunk, or one slice of it (quantiles of the
// longest fan-in inside the chunk); each slice is an exact chunk
// (the slice's end is the next slice's start: computed by the next lane when it
// is that slice's lane, else here)
__device__ __forceinline__ long long slice_start(const SimParams& p, uint32_t ref, unsigned long long q0,
                                                 unsigned long long q1, int sidx, int nsl, long long T0) {
    return sidx == 0 ? T0 : time_at(p, ref, q0 + ((q1 - q0) * (unsigned long long)sidx) / nsl);
}
__device__ __forceinline__ void unit_setup(const SimParams& p, unsigned long long id, int sidx, int nsl,
                                           ChunkSetup& s, uint32_t& gi, uint32_t& nch, const long long* next_start) {
    uint32_t cidx, ref;
    unsigned long long q0, q1, n_in;
    setup_chunk(p, id, s, gi, cidx, nch, &q0, &q1, &ref, &n_in);
    if (nsl > 1) {
        const long long t0 = slice_start(p, ref, q0, q1, sidx, nsl, s.T0);
        const long long t1 = sidx + 1 == nsl ? s.T1
                             : next_start ? *next_start
                                          : slice_start(p, ref, q0, q1, sidx + 1, nsl, s.T0);
        s.T0 = t0;
        s.T1 = t1;
        s.tau0 = t0 - (long long)s.dmax - 1;
    }
}
template <class T>
__device__ __forceinline__ void fill_dtab(T* dtab, int dstride, const ChunkSetup& s) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {                       // R1: output X takes the smaller delay
        const uint4 d = s.d[i];
        dtab[(i * 6 + 0) * dstride] = (T)d.z;
        dtab[(i * 6 + 1) * dstride] = (T)d.w;
        dtab[(i * 6 + 2) * dstride] = (T)min(d.z, d.w);
        dtab[(i * 6 + 3) * dstride] = (T)d.x;
        dtab[(i * 6 + 4) * dstride] = (T)d.y;
        dtab[(i * 6 + 5) * dstride] = (T)min(d.x, d.y);
    }
}

// lane 0: zero / flush this warp's statistics
__device__ __forceinline__ void acc_zero(Batch& B) {
    for (int k = 0; k < A_N; ++k) B.acc[k] = 0;
}
__device__ void acc_flush(const SimParams& p, Batch& B) {
    unsigned long long* const dst[A_N] = {
        &p.ctl->gate_evals, &p.ctl->events, &p.ctl->out_trans, &p.ctl->chunks, &p.ctl->lane_iters, &p.ctl->warp_iters,
        &p.ctl->batches, &p.ctl->batch_lanes, &p.ctl->batch_est, &p.ctl->cyc[0], &p.ctl->cyc[1], &p.ctl->cyc[2],
        &p.ctl->cyc[3], &p.ctl->cyc[4], &p.ctl->cyc[5], &p.ctl->bal[0], &p.ctl->bal[1], &p.ctl->bal[2],
        &p.ctl->bal[3], &p.ctl->bal[4], &p.ctl->bal[5], &p.ctl->bal[6], &p.ctl->bal[7]};
    for (int k = 0; k < A_N; ++k)
        if (B.acc[k]) atomicAdd(dst[k], B.acc[k]);
    acc_zero(B);
}

// Whole warp: evaluate one batch.  Returns false when there is no more work
// (dataflow: every gate done or an error; levels: the level is exhausted).
// `carry` (lane 0) holds a claimed chunk id that did not fit the last batch.
template <bool DATAFLOW>
__device__ bool slice_batch(const SimParams& p, const uint8_t* lut, uint16_t* s_dtab, Batch& B,
                            unsigned long long& carry, unsigned long long lvl_begin, unsigned long long lvl_n,
                            unsigned long long* lvl_work, PinSm cs) {
    const int lane = threadIdx.x & 31;
    constexpr unsigned long long NONE = ~0ull;
    int nc = 0, nu = 0;
    bool more = true;
    const long long c_start = clock64();
    if (lane == 0) {
        // phase 1: claim published chunks until the batch holds about 32 x W_LANE transitions
        unsigned long long est[MAXC];
        unsigned long long total = 0;
        // shallow queue (fewer published chunks than warps): one chunk per batch, so its
        // slices spread over all 32 lanes and the critical path through the netlist shortens
        unsigned long long fill = 32ull * W_LANE;
        if (DATAFLOW && GLS_ADAPT) {
            const unsigned long long pub = ld_relaxed_u64(&p.ctl->chunk_top), head = ld_relaxed_u64(&p.ctl->work_head);
            if (pub < head + (unsigned long long)gridDim.x * (blockDim.x >> 5)) fill = 1;
        }
        while (nc < MAXC && total < fill) {
            unsigned long long id;
            if (carry != NONE) {
                id = carry;
                carry = NONE;
            } else if (DATAFLOW) {
                id = atomicAdd(&p.ctl->work_head, 1ull);
            } else {
                const unsigned long long w = atomicAdd(lvl_work, 1ull);
                if (w >= lvl_n) break;
                id = lvl_begin + w;
            }
            uint32_t g;
            if (DATAFLOW) {
                g = id < p.ck_cap ? ld_relaxed_u32(&p.ck_gate[id]) : 0xffffffffu;
                if (g == 0xffffffffu) {
                    if (nc > 0) {                           // never wait while holding work
                        carry = id;
                        break;
                    }
                    unsigned ns = 32;
                    unsigned long long t_start = 0, seen = ~0ull;
                    for (;;) {
                        if (id < p.ck_cap) {
                            g = ld_relaxed_u32(&p.ck_gate[id]);
                            if (g != 0xffffffffu) break;
                        }
                        const unsigned long long done = ld_relaxed_u64(&p.ctl->done_gates);
                        if (done >= (unsigned long long)p.G || ld_relaxed_u32(&p.ctl->error) != 0u) break;
                        unsigned long long now;             // watchdog (10 s without progress)
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                        if (done != seen) {
                            seen = done;
                            t_start = now;
                        } else if (now - t_start > 10000000000ull) {
                            atomicOr(&p.ctl->error, kErrWatchdog);
                            break;
                        }
                        __nanosleep(ns);
                        if (ns < GLS_MAXSLEEP) ns <<= 1;
                    }
                    if (g == 0xffffffffu) {
                        more = false;
                        break;
                    }
                }
            } else {
                g = __ldcg(&p.ck_gate[id]);
            }
            const unsigned long long nch = __ldcg(&p.net_nck[p.P + g]);
            const unsigned long long e = __ldcg(&p.gate_nin[g]) / (nch ? nch : 1ull);
            B.id[nc] = id;
            est[nc] = e;
            total += e;
            ++nc;
        }
        if (nc > 0) {
            B.acc[A_BATCHES] += 1ull;
            B.acc[A_BEST] += total;
        }
        // phase 2: spread the 32 lanes in proportion to the expected work (w per lane)
        const unsigned long long w = max((unsigned long long)W_MIN, (total + 31) / 32);
        int next_lane = 0, shared = -1;
        unsigned long long shared_load = 0;
        for (int q = 0; q < 32; ++q) B.lane_nu[q] = 0;
        for (int j = 0; j < nc; ++j) {
            const unsigned long long e = est[j];
            const int left = 32 - next_lane;
            B.first_unit[j] = (uint8_t)nu;
            if (e >= w && left > 0 && nu + left <= MAXU) {
                const int ns = (int)min((unsigned long long)left, max(1ull, (e + w / 2) / w));
                B.nsl[j] = (uint8_t)ns;
                for (int q = 0; q < ns; ++q) {
                    B.u_chunk[nu] = (uint8_t)j;
                    B.u_slice[nu] = (uint8_t)q;
                    B.u_lane[nu] = (uint8_t)next_lane;
                    B.lane_u0[next_lane] = (uint8_t)nu;
                    B.lane_nu[next_lane] = 1;
                    ++next_lane;
                    ++nu;
                }
                shared = -1;                        // a lane's units must stay contiguous
            } else {
                if (shared < 0 || (shared_load + e > w && left > 0)) {
                    if (left > 0) {
                        shared = next_lane++;
                        shared_load = 0;
                        B.lane_u0[shared] = (uint8_t)nu;
                    } else {
                        shared = 31;                // out of lanes: the last lane takes the rest
                    }
                }
                B.nsl[j] = 1;
                B.u_chunk[nu] = (uint8_t)j;
                B.u_slice[nu] = 0;
                B.u_lane[nu] = (uint8_t)shared;
                B.lane_nu[shared]++;
                shared_load += e;
                ++nu;
            }
        }
        if (nc > 0) {
            int busy = 0;
            for (int q = 0; q < 32; ++q) busy += B.lane_nu[q] > 0;
            B.acc[A_BLANES] += (unsigned long long)busy;
        }
        p.deep_wtop[warp_global_id()] = 0;          // this warp's deep scratch, reused per batch
    }
    nc = __shfl_sync(FULL, nc, 0);
    more = __shfl_sync(FULL, (int)more, 0) != 0;
    __syncwarp();
    if (nc == 0) return DATAFLOW ? more : false;
    nu = __shfl_sync(FULL, nu, 0);

    uint64_t* const wscr = p.wscr + (size_t)warp_global_id() * kScratchPerWarp;
    uint64_t* scr = wscr + (size_t)lane * LCAP;
    uint16_t* dtab = s_dtab + threadIdx.x;                // [q * blockDim.x + tid] (gates with dmax < 2^16)
    const int dstride = (int)blockDim.x;
    const uint32_t lut_sa = (uint32_t)__cvta_generic_to_shared(lut);
    const uint32_t dtab_sa = (uint32_t)__cvta_generic_to_shared(dtab);
    // ---- each lane: its units, in order
    const int u0 = B.lane_u0[lane], nun = B.lane_nu[lane];
    uint32_t used = 0, its_sum = 0;
    const long long c_asm = clock64();
    long long c_setup = 0, c_locate = 0;
    // a slice lane (one unit, of a chunk with several slices) publishes its start time to
    // the previous lane, whose slice ends there
    long long my_start = 0;
    bool slice_lane = false;
    if (nun == 1 && B.nsl[B.u_chunk[u0]] > 1) {
        const int j = B.u_chunk[u0];
        ChunkSetup s0;
        uint32_t gi0, cidx0, nch0, ref0;
        unsigned long long q0, q1, nin0;
        setup_chunk(p, B.id[j], s0, gi0, cidx0, nch0, &q0, &q1, &ref0, &nin0);
        my_start = slice_start(p, ref0, q0, q1, B.u_slice[u0], B.nsl[j], s0.T0);
        slice_lane = true;
    }
    const long long nb_start = __shfl_down_sync(FULL, my_start, 1);
    const bool nb_same = __shfl_down_sync(FULL, (int)(slice_lane ? (int)B.u_chunk[u0] : -1), 1) ==
                         (slice_lane ? (int)B.u_chunk[u0] : -2);
    for (int u = u0; u < u0 + nun; ++u) {
        const long long c_us = clock64();
        const int j = B.u_chunk[u];
        ChunkSetup s;
        uint32_t gi, nch;
        unit_setup(p, B.id[j], B.u_slice[u], B.nsl[j], s, gi, nch,
                   (slice_lane && nb_same && lane < 31) ? &nb_start : nullptr);
        if (B.u_slice[u] == 0) B.c_T0[j] = s.T0;
        if (s.dmax < kFastDelay) fill_dtab(dtab, dstride, s);
        c_setup += clock64() - c_us;
        uint32_t cnt = 0, vb = 2, ev = 0, evt = 0, its = 0;
        const uint32_t cap = used < (uint32_t)LCAP ? (uint32_t)LCAP - used : 0u;
        int st;
        if (s.dmax < kFastDelay) {
            uint32_t res[5];
            st = run_slice32<false>(p, s, lut_sa, dtab_sa, cs, scr + (used < (uint32_t)LCAP ? used : 0u), cap,
                                    res, &c_locate);
            cnt = res[0];
            vb = res[1];
            ev = res[2];
            evt = res[3];
            its = res[4];
        } else {
            uint32_t dl[24];                                // long delays: 64-bit sweep, table in local memory
            fill_dtab(dl, 1, s);
            st = run_slice<false>(p, s, lut, dl, 1, scr + (used < (uint32_t)LCAP ? used : 0u), cnt, vb,
                                  ev, evt, its, cap, c_locate);
        }
        if (st == 1) {
            // pending ring overflow: exact count by the per-lane engine (deep ring if needed)
            ChunkOut r{0, 0, 0, 2, false};
            run_chunk<false, false>(p, s, lut, nullptr, nullptr, 0, r);
            if (r.overflow) {
                const unsigned long long dcap = window_bound(p, s);
                const unsigned long long at = deep_alloc(p, dcap);
                if (at != ~0ull) {
                    r = ChunkOut{0, 0, 0, 2, false};
                    run_chunk<false, true>(p, s, lut, nullptr, p.deep + at, dcap, r);
                }
            }
            cnt = r.cnt;
            vb = r.vb;
            ev = r.evals;
            evt = r.events;
        }
        if (st != 0) atomicAdd(&p.ctl->deep_chunks, 1ull);
        B.u_cnt[u] = cnt;
        B.u_ev[u] = ev;
        B.u_evt[u] = evt;
        B.u_vb[u] = (uint8_t)vb;
        B.u_st[u] = (uint8_t)st;
        B.u_soff[u] = (uint16_t)(used < (uint32_t)LCAP ? used : 0u);
        if (st == 0) used += cnt;
        its_sum += its;
    }
    __syncwarp();
    const long long c_run = clock64();
    {   // lane utilisation counters
        const unsigned long long sum_it = warp_sum64(its_sum);
        unsigned long long mx = its_sum;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = max(mx, (unsigned long long)__shfl_xor_sync(FULL, mx, o));
        if (lane == 0) {
            B.acc[A_LANE_IT] += sum_it;
            B.acc[A_WARP_IT] += 32ull * mx;
        }
        // balance counters: slice lanes against their group's longest lane, packed lanes, idle lanes
        const unsigned gid = slice_lane ? (unsigned)B.u_chunk[u0] : (nun > 0 ? 1000u : 2000u);
        const unsigned gm = __match_any_sync(FULL, gid);
        const unsigned gmax = __reduce_max_sync(gm, its_sum);
        const unsigned long long b0 = warp_sum64(slice_lane ? its_sum : 0u);
        const unsigned long long b1 = warp_sum64(slice_lane ? gmax : 0u);
        const unsigned long long b2 = warp_sum64(!slice_lane && nun > 0 ? its_sum : 0u);
        const unsigned n_sl = __popc(__ballot_sync(FULL, slice_lane));
        const unsigned n_pk = __popc(__ballot_sync(FULL, !slice_lane && nun > 0));
        if (lane == 0) {
            B.acc[A_BAL + 0] += b0;
            B.acc[A_BAL + 1] += b1;
            B.acc[A_BAL + 2] += b2;
            B.acc[A_BAL + 3] += (unsigned long long)n_pk * mx;
            B.acc[A_BAL + 4] += (unsigned long long)n_sl * mx;
            B.acc[A_BAL + 5] += (unsigned long long)(32u - n_sl - n_pk) * mx;
            B.acc[A_BAL + 6] += (unsigned long long)n_sl;
            B.acc[A_BAL + 7] += (unsigned long long)n_pk;
        }
    }
    __syncwarp();
    // ---- per chunk: unit offsets, total and one exact segment
    for (int j = lane; j < nc; j += 32) {
        uint32_t tot = 0;
        for (int u = B.first_unit[j]; u < B.first_unit[j] + B.nsl[j]; ++u) {
            B.u_pre[u] = tot;
            tot += B.u_cnt[u];
        }
        unsigned long long off = tot ? atomicAdd(&p.ctl->arena_top, seg_round(tot)) : 0ull;
        if (off + tot > p.arena_cap) {
            atomicOr(&p.ctl->error, kErrArena);
            atomicMax(&p.ctl->need_arena, off + tot);
            off = ~0ull;
        }
        B.c_off[j] = off;
        B.c_total[j] = tot;
    }
    __syncwarp();
    // ---- each lane moves its clean units into place (independent loads, overlapped latency)
    for (int u = u0; u < u0 + nun; ++u) {
        const unsigned long long off = B.c_off[B.u_chunk[u]];
        const uint32_t cu = B.u_cnt[u];
        if (off == ~0ull || B.u_st[u] != 0 || cu == 0) continue;
        const uint64_t* src = scr + B.u_soff[u];
        uint64_t* dst = p.arena + off + B.u_pre[u];
        uint32_t e = 0;
        for (; e + 4 <= cu; e += 4) {
            const uint64_t a0 = src[e], a1 = src[e + 1], a2 = src[e + 2], a3 = src[e + 3];
            dst[e] = a0;
            dst[e + 1] = a1;
            dst[e + 2] = a2;
            dst[e + 3] = a3;
        }
        for (; e < cu; ++e) dst[e] = src[e];
    }
#if GLS_DISCARD
    // the staged outputs are dead: drop their L2 lines without writing them back to DRAM
    for (uint32_t q = 0; q < min(used, (uint32_t)LCAP); q += 16)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(scr + q) : "memory");
#endif
    // ---- units whose scratch or ring overflowed: the owning lane writes them in place
    for (int u = u0; u < u0 + nun; ++u) {
        const int st = B.u_st[u];
        if (st == 0) continue;
        const int j = B.u_chunk[u];
        const unsigned long long off = B.c_off[j];
        if (off == ~0ull) continue;
        ChunkSetup s;
        uint32_t gi, nch;
        unit_setup(p, B.id[j], B.u_slice[u], B.nsl[j], s, gi, nch, nullptr);
        if (s.dmax < kFastDelay) fill_dtab(dtab, dstride, s);
        uint64_t* dst = p.arena + off + B.u_pre[u];
        if (st == 2) {                                  // scratch overflow: re-run straight into place
            uint32_t c2, v2, e2, t2, i2;
            long long c_dummy = 0;
            if (s.dmax < kFastDelay) {
                uint32_t res[5];
                run_slice32<true>(p, s, lut_sa, dtab_sa, cs, dst, 0u, res, &c_dummy);
                c2 = res[0];
            } else {
                uint32_t dl[24];
                fill_dtab(dl, 1, s);
                run_slice<true>(p, s, lut, dl, 1, dst, c2, v2, e2, t2, i2, 0u, c_dummy);
            }
            if (c2 != B.u_cnt[u]) atomicOr(&p.ctl->error, kErrBug);
        } else {                                        // ring overflow: per-lane engine in place
            ChunkOut r2{0, 0, 0, 2, false};
            run_chunk<true, false>(p, s, lut, dst, nullptr, 0, r2);
            if (r2.overflow) {
                const unsigned long long dcap = window_bound(p, s);
                const unsigned long long at = deep_alloc(p, dcap);
                if (at != ~0ull) {
                    r2 = ChunkOut{0, 0, 0, 2, false};
                    run_chunk<true, true>(p, s, lut, dst, p.deep + at, dcap, r2);
                }
            }
            if (r2.cnt != B.u_cnt[u]) atomicOr(&p.ctl->error, kErrBug);
        }
    }
    __syncwarp();
    const long long c_out = clock64();
    // ---- complete the chunks (whole warp, one after the other)
    for (int j = 0; j < nc; ++j) {
        const int ufirst = B.first_unit[j];
        const unsigned long long id = B.id[j];
        ChunkResult R;
        R.gi = __ldcg(&p.ck_gate[id]);
        R.nch = __ldcg(&p.net_nck[p.P + R.gi]);
        R.s.T0 = B.c_T0[j];
        R.off = B.c_off[j];
        R.fits = R.off != ~0ull;
        R.total = B.c_total[j];
        R.vb = B.u_vb[ufirst];
        unsigned long long e1 = 0, e2 = 0;
        for (int u = ufirst; u < ufirst + B.nsl[j]; ++u) {
            e1 += B.u_ev[u];
            e2 += B.u_evt[u];
        }
        R.evals = e1;
        R.events = e2;
        chunk_done<DATAFLOW>(p, id, R, B.acc);
    }
    const long long c_end = clock64();
    const unsigned long long setup_max = warp_max64((unsigned long long)c_setup);
    const unsigned long long loc_max = warp_max64((unsigned long long)c_locate);
    if (lane == 0) {
        B.acc[A_CYC + 0] += (unsigned long long)(c_asm - c_start);
        B.acc[A_CYC + 1] += setup_max;
        B.acc[A_CYC + 2] += loc_max;
        B.acc[A_CYC + 3] += (unsigned long long)(c_run - c_asm) - setup_max - loc_max;
        B.acc[A_CYC + 4] += (unsigned long long)(c_out - c_run);
        B.acc[A_CYC + 5] += (unsigned long long)(c_end - c_out);
    }
    return true;
}

}  // namespace sl
}  // namespace gls
