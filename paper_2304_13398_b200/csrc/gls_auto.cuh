// gls_auto.cuh — engine 3: autonomous lanes writing in place.  Included by
// gls_kernels.cu after gls_lanes.cuh (it reuses that file's sweep helpers).
// DESIGN.md §7.
//
// Every lane of a persistent warp runs its own (gate, time-chunk) work item from
// start to end: the dataflow scheduler (Alg. 1's unlock rule) plans a
// gate into chunks of about M merged input entries as soon as its fan-in gates are
// complete, and idle lanes pull published chunk ids from one device queue.  A chunk
// is an exact time chunk (halo start at tau0 = T0 - dmax - 1), swept
// by the same 32-bit Algorithm 2 loop as engine 0 (one fan-in entry per
// iteration, LUT in shared memory, min-rule delay, Eq. 1 as the addSignalChange
// stack).  Differences from engine 0:
//   * no warp batches, static slices or re-balancing rounds: a lane that finishes
//     takes the next chunk at the warp's next service point (every AROUND
//     iterations), so lanes stay busy whatever the activity skew;
//   * the Eq. 1 stack lives in the ARENA, in a page owned by the lane: the chunk's
//     outputs are a contiguous run of that stack (entries >= T0, < T1), so they are
//     published where they were written — no scratch, no copy, one exact segment per
//     chunk, 128-byte aligned.  The next chunk of the lane starts its stack
//     on the next 128-byte line after the run.  A stack that outgrows the page
//     restarts the chunk on a fresh page twice as large (rare).
//   * the service point is warp-uniform: the warp publishes each finished lane's
//     chunk (descriptor, gate completion, consumers unlocked and planned —
//     chunk_done / gate_complete / plan_gate, whole warp), claims ids for idle
//     lanes with one atomicAdd, and newly published lanes set up (locate their pins
//     at tau0: lockstep binary searches).
//   * the sweep state of a lane lives in shared memory between rounds (loaded into
//     registers for a round of AROUND iterations, stored back after it), so no
//     register is live across the service point and the set-up: the round function
//     has the whole register file.
// Gates with a delay >= 2^16 run the per-lane ring engine (lane_chunk) inside the
// set-up, synchronously.
#pragma once

namespace gls {
namespace au {

using namespace ln;

#ifndef GLS_APAGE
#define GLS_APAGE 8192
#endif
constexpr uint32_t APAGE = GLS_APAGE;            // entries of a lane's output page (64 KB)
#ifndef GLS_AROUND
#define GLS_AROUND 32
#endif
constexpr int AROUND = GLS_AROUND;               // sweep iterations between service points
#ifndef GLS_PF
#define GLS_PF 0                                 // L2 prefetch distance in 128-byte lines (0: none)
#endif
#ifndef GLS_RING
#define GLS_RING 4                               // lookahead ring entries per pin (power of 2, >= 2)
#endif
#ifndef GLS_ACQ_CLAIM
#define GLS_ACQ_CLAIM 1                          // acquire on the claimed chunk's publication
#endif

enum : uint32_t { S_IDLE = 0, S_CLAIMED = 1, S_RUN = 2, S_DONE = 3, S_READY = 4 };

// a lane's chunk record (global memory, one per lane of the grid; read by the whole
// warp at the service point)
struct LaneRec {
    unsigned long long id;                 // chunk id
    long long T0, T1;                      // its time range
    unsigned long long sb;                 // arena offset of its Eq. 1 stack
    unsigned long long top, end;           // the lane's page: next free entry, end
    uint32_t ev, evt;                      // gate-evals / events counted so far
    uint32_t lo, hi;                       // done: outputs = stack entries [lo, hi)
    uint32_t need;                         // room the next set-up must find (restart: 2 x the stack)
    uint32_t st, vb, pad;
};
__device__ __forceinline__ LaneRec* lane_recs(const SimParams& p) {
    return reinterpret_cast<LaneRec*>(p.waux) + (size_t)warp_global_id() * 32u;
}

// sweep state columns in shared memory, [field][kThreads]
struct StateCols {
    unsigned long long b4[kThreads];       // base B in entry form
    unsigned long long scr[kThreads];      // &arena[sb]
    uint32_t h[4][kThreads];               // pin heads, entry form relative to B
    uint32_t nr[kThreads], xn[kThreads], eprev[kThreads], lutb[kThreads];
    uint32_t t0q[kThreads], lim[kThreads], n[kThreads], cap[kThreads];
    uint32_t nfl[kThreads], top[kThreads];
};
struct WarpAcc {
    unsigned long long acc[A_N];
};
__device__ void acc_flush(const SimParams& p, WarpAcc& A) {
    unsigned long long* const dst[A_N] = {
        &p.ctl->gate_evals, &p.ctl->events, &p.ctl->out_trans, &p.ctl->chunks, &p.ctl->lane_iters, &p.ctl->warp_iters,
        &p.ctl->batches, &p.ctl->batch_lanes, &p.ctl->batch_est, &p.ctl->cyc[0], &p.ctl->cyc[1], &p.ctl->cyc[2],
        &p.ctl->cyc[3], &p.ctl->cyc[4], &p.ctl->cyc[5], &p.ctl->bal[0], &p.ctl->bal[1], &p.ctl->bal[2],
        &p.ctl->bal[3], &p.ctl->bal[4], &p.ctl->bal[5], &p.ctl->bal[6], &p.ctl->bal[7]};
    for (int k = 0; k < A_N; ++k)
        if (A.acc[k]) atomicAdd(dst[k], A.acc[k]);
}
constexpr size_t kDtabBytes = (size_t)kDtabWords * kThreads * 2;
constexpr size_t kDynBytes = kDtabBytes + sizeof(StateCols) + sizeof(WarpAcc) * (kThreads / 32) + 4 * kThreads * (8 + 4 + 4 + 8 * GLS_RING);

__device__ __forceinline__ StateCols& state() { return *reinterpret_cast<StateCols*>(g_dyn + kDtabBytes); }
__device__ __forceinline__ WarpAcc& wacc() {
    return reinterpret_cast<WarpAcc*>(g_dyn + kDtabBytes + sizeof(StateCols))[threadIdx.x >> 5];
}
// per-thread pin cursors and lookahead rings in shared memory: head address, entries from
// the head on, chunk of the segment, and a ring of RING entries mirroring the entries
// after the head (slot = (entry address / 8) mod RING, so a slot is refilled with the
// entry RING positions ahead the moment its entry becomes the head)
constexpr int RING = GLS_RING;
struct PinCols {
    uint32_t b;
    __device__ __forceinline__ uint32_t ptr(int ci) const { return b + (uint32_t)ci * 8u; }
    __device__ __forceinline__ uint32_t rem(int ci) const { return b + 4u * kThreads * 8u + (uint32_t)ci * 4u; }
    __device__ __forceinline__ uint32_t ck(int ci) const { return b + 4u * kThreads * 12u + (uint32_t)ci * 4u; }
    // ring slot of entry address a for pin i (ci = i * kThreads + tid)
    __device__ __forceinline__ uint32_t slot(int ci, const uint64_t* a) const {
        return b + 4u * kThreads * 16u + ((uint32_t)ci + (((uint32_t)(uintptr_t)a >> 3) & (RING - 1)) * 4u * kThreads) * 8u;
    }
};
constexpr size_t kPinColsBytes = (size_t)4 * kThreads * (8 + 4 + 4 + 8 * RING);
__device__ __forceinline__ PinCols pins() {
    return PinCols{(uint32_t)__cvta_generic_to_shared(g_dyn + kDtabBytes + sizeof(StateCols) +
                                                      sizeof(WarpAcc) * (kThreads / 32))};
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
// request entry a into smem address sa if go (predicated; no commit)
__device__ __forceinline__ void cp_req8_if(bool go, uint32_t sa, const void* a) {
    asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %0, 0;\n @p cp.async.ca.shared.global [%1], [%2], 8;\n}\n" ::"r"((uint32_t)go),
                 "r"(sa), "l"(a) : "memory");
}
// the ring entries after the head (entries 1 .. RING-1 of a cursor with rem entries)
__device__ __forceinline__ void ring_fill(const PinCols& cs, int ci, const uint64_t* head, uint32_t rem) {
#pragma unroll
    for (int j = 1; j < RING; ++j) cp_req8_if((uint32_t)j < rem, cs.slot(ci, head + j), head + j);
}

// Set up the lane's claimed chunk (published): its record, page room, delay table,
// cursors at tau0 and the halo-start evaluation; the sweep state goes to the shared
// columns.  Returns S_RUN, S_DONE when the chunk was finished here (per-lane ring engine
// for long delays), S_IDLE when the arena is full (error raised; the run aborts).
__device__ __noinline__ uint32_t begin(const SimParams& p) {
    LaneRec& R = lane_recs(p)[threadIdx.x & 31];
    StateCols& S = state();
    const PinCols cs = pins();
    const int tid = threadIdx.x;
    const unsigned long long id = R.id;
    ChunkSetup s;
    uint32_t gi, cidx, nch;
    setup_chunk(p, id, s, gi, cidx, nch);
    R.T0 = s.T0;
    R.T1 = s.T1;
    R.ev = R.evt = 0;
    if (s.dmax >= kFastDelay) {                                   // long delays: 64-bit ring engine
        unsigned long long off = 0, ev = 0, evt = 0;
        uint32_t cnt = 0, vb = 2;
        bool fits = true;
        lane_chunk(p, s, g_lut, off, cnt, vb, ev, evt, fits);
        if (!fits) return S_IDLE;
        R.sb = off;
        R.lo = 0;
        R.hi = cnt;
        R.vb = vb;
        R.ev = (uint32_t)ev;
        R.evt = (uint32_t)evt;
        return S_DONE;
    }
    // the stack starts on the next 128-byte line of the lane's page; a fresh page when the
    // room left is below the expected merged entries of the chunk (or what a restart asks)
    const unsigned long long nin = __ldcg(&p.gate_nin[gi]);
    const unsigned long long want = max((unsigned long long)R.need, nin / max(1u, nch) + 64ull);
    unsigned long long sb = (R.top + 15ull) & ~15ull;
    if (sb + want > R.end) {
        const unsigned long long sz = (max((unsigned long long)APAGE, 2ull * want) + 15ull) & ~15ull;
        const unsigned long long at = atomicAdd(&p.ctl->arena_top, sz);
        if (at + sz > p.arena_cap) {
            atomicOr(&p.ctl->error, kErrArena);
            atomicMax(&p.ctl->need_arena, at + sz);
            R.top = R.end = 0;
            return S_IDLE;
        }
        sb = at;
        R.end = at + sz;
    }
    R.sb = sb;
    R.need = 0;
    const uint32_t cap = (uint32_t)min(R.end - sb, 0x7fffffffull);
    uint64_t* const scr = p.arena + sb;
    fill_dtab(dtab_cols() + tid, (int)blockDim.x, s);
    const uint32_t lutb = lut_sa() + s.lut_base;
    const uint64_t b4 = (uint64_t)s.tau0 << 2;
    uint32_t xn = 0, xr0 = 0;
    Cursor cur[4];
    uint32_t ini[4];
    locate_all(p, s.src, s.k, s.tau0, cur, ini);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int ci = i * kThreads + tid;
        uint32_t h = kRelInf;
        if ((uint32_t)i >= s.k) {
            sts32(cs.rem(ci), 0u);                                   // absent pin: exhausted
        } else {
            const Cursor& cc = cur[i];
            const uint32_t rem = (uint32_t)(cc.end - cc.ptr);
            sts64(cs.ptr(ci), (uint64_t)cc.ptr);
            sts32(cs.rem(ci), rem);
            sts32(cs.ck(ci), cc.ck);
            ring_fill(cs, ci, cc.ptr, rem);
            h = rem ? to_rel(*cc.ptr, b4) : kRelInf;
            xn |= 2u << (2 * i);                                     // inputs start at X
            xr0 |= ini[i] << (2 * i);                                // raw values in effect at tau0
        }
        S.h[i][tid] = h;
    }
    cp_commit();
    cp_wait<0>();                                                    // the rings are filled
    uint32_t t0q, lim;
    int more;
    thresholds(b4, s.T0, s.T1, t0q, lim, more);
    // the halo start (t = tau0, relative 0): the inputs take their values in effect there;
    // a first event (E != X) is pushed onto the empty stack (its delay: the min over the
    // pins that left X, readings R1-R3; nothing when every such pin is unrelated, R9)
    uint32_t n = 0, top = 0, Eprev = 2;
    const uint32_t nn = xr0 ^ ((xr0 >> 1) & xr0 & 0x55u);           // Z -> X
    if (nn != xn) {
        const uint32_t E = lds8(lutb + nn);
        if (E != 2u) {
            const uint32_t dt_sa = (uint32_t)__cvta_generic_to_shared(dtab_cols() + tid);
            const uint32_t d = nn ^ xn;
            uint32_t cm = (d | (d >> 1)) & 0x55u, del = 0xffffffffu;
            do {
                const int b = __ffs(cm) - 1;
                const uint32_t rise = (0x206u >> ((((xn >> b) & 3u) << 2) | ((nn >> b) & 3u))) & 1u;
                const uint32_t dw = lds32(dt_sa + (uint32_t)((b >> 1) * 2 + (int)rise) * (kThreads * 4));
                del = min(del, __funnelshift_r(dw, 0u, 16u * E) & 0xFFFFu);
                cm &= cm - 1;
            } while (cm);
            if (del != kDelayInf16) {
                top = (del << 2) | E;
                stg64(scr, (uint64_t)top + b4);
                n = 1;
            }
            Eprev = E;
        }
        xn = nn;
    }
    S.b4[tid] = b4;
    S.scr[tid] = (unsigned long long)scr;
    S.nr[tid] = xr0;
    S.xn[tid] = xn;
    S.eprev[tid] = Eprev;
    S.lutb[tid] = lutb;
    S.t0q[tid] = t0q;
    S.lim[tid] = lim;
    S.n[tid] = n;
    S.cap[tid] = cap;
    S.nfl[tid] = 2u << 16;                                           // nothing final yet; value before: X
    S.top[tid] = top;
    return S_RUN;
}

// The chunk is swept: its outputs are the stack entries (increasing in time) in
// [T0, min(T1, duration + 1)); the entry below them gives the value before T0 (X if
// none).  n == ~0: the stack outgrew the page — restart on a page twice the size.
__device__ __noinline__ uint32_t finish(const SimParams& p, uint32_t n, uint32_t cap) {
    LaneRec& R = lane_recs(p)[threadIdx.x & 31];
    if (n == 0xffffffffu) {
        R.need = (uint32_t)min(2ull * cap + 64ull, 0x7fffffffull);
        R.top = R.end;                                               // (the page is abandoned)
        return S_CLAIMED;
    }
    const uint64_t* scr = p.arena + R.sb;
    const long long T0 = R.T0, T1e = min(R.T1, p.duration + 1);
    uint32_t lo = 0, hi = n, vb = 2u;
    while (lo < hi && ((long long)ldg64(scr + lo) >> 2) < T0) ++lo;
    while (hi > lo && ((long long)ldg64(scr + hi - 1) >> 2) >= T1e) --hi;
    if (lo > 0) vb = (uint32_t)(ldg64(scr + lo - 1) & 3u);
    R.lo = lo;
    R.hi = hi;
    R.vb = vb;
    R.top = R.sb + hi;
    return S_DONE;
}

// One round of the lane's sweep (up to AROUND fan-in entries): state from the shared
// columns into registers, Algorithm 2, state back.  Returns the iterations run; st
// becomes S_DONE / S_CLAIMED (restart) when the chunk ends in this round.
__device__ __forceinline__ int sweep_round(const SimParams& p, uint32_t& st, uint32_t& l_cnt) {
    StateCols& S = state();
    const PinCols cs = pins();
    const int tid = threadIdx.x;
    const uint32_t dt_sa = (uint32_t)__cvta_generic_to_shared(dtab_cols() + tid);
    uint64_t b4 = S.b4[tid];
    uint64_t* const scr = (uint64_t*)S.scr[tid];
    uint32_t h0 = S.h[0][tid], h1 = S.h[1][tid], h2 = S.h[2][tid], h3 = S.h[3][tid];
    uint32_t m = min(min(h0, h1), min(h2, h3));
    uint32_t nr = S.nr[tid], xn = S.xn[tid], Eprev = S.eprev[tid];
    const uint32_t lutb = S.lutb[tid], cap = S.cap[tid];
    uint32_t t0q = S.t0q[tid], lim = S.lim[tid], n = S.n[tid], nfl = S.nfl[tid], top = S.top[tid];
    uint32_t cnt = 0;                      // gate-evals (bits 0-15) and events (16-31) of the round
    int it = 0;
    for (; it < AROUND; ++it) {
        if (m >= lim) {
            if (lim == kRebaseQ) {
                // rebase (the sweep reached B + 2^29 before T1): the stack entries before the
                // true next head tmin are final (any later event appears at >= tmin), B := tmin
                uint64_t raw = kInfEntry;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int ci = i * kThreads + tid;
                    if (lds32(cs.rem(ci))) raw = min(raw, ldg_entry((const uint64_t*)lds64(cs.ptr(ci))));
                }
                const LaneRec& R = lane_recs(p)[tid & 31];
                const long long T1 = R.T1;
                const long long tmin = raw == kInfEntry ? LLONG_MAX : etime(raw);
                if (tmin < T1) {
                    uint32_t f = n;
                    const uint32_t fl = nfl & 0xffffu;
                    while (f > fl && ((long long)ldg64(scr + f - 1) >> 2) >= tmin) --f;
                    if (f > fl) nfl = f | ((uint32_t)(ldg64(scr + f - 1) & 3u) << 16);
                    b4 = (uint64_t)tmin << 2;                        // every live entry is >= tmin
                    int more;
                    thresholds(b4, R.T0, T1, t0q, lim, more);
                    top = n > (nfl & 0xffffu) ? to_rel(ldg64(scr + n - 1), b4) : 0u;
                    uint32_t hh[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int ci = i * kThreads + tid;
                        hh[i] = lds32(cs.rem(ci)) ? to_rel(ldg_entry((const uint64_t*)lds64(cs.ptr(ci))), b4) : kRelInf;
                    }
                    h0 = hh[0];
                    h1 = hh[1];
                    h2 = hh[2];
                    h3 = hh[3];
                    m = min(min(h0, h1), min(h2, h3));
                    continue;
                }
            }
            // ---- chunk swept
            cp_wait<0>();                                            // no copy may land in the next chunk's cursors
            st = n == 0xffffffffu ? S_CLAIMED : S_DONE;              // (the caller runs finish())
            break;
        }
        // ---- one fan-in entry: the pin with the smallest head
        const int b = h0 == m ? 0 : h1 == m ? 1 : h2 == m ? 2 : 3;
        nr = (nr & ~(3u << (2 * b))) | ((m & 3u) << (2 * b));
        const int ci = b * kThreads + tid;
        const uint64_t* ptr = (const uint64_t*)lds64(cs.ptr(ci)) + 1;
        uint32_t rem = lds32(cs.rem(ci)) - 1u;
        uint64_t hn;
        if (rem != 0) {
            // the new head's ring slot was requested when the entry RING - 1 positions
            // before it became the head, >= RING - 1 iterations (groups) ago
            cp_wait<RING - 2>();
            hn = lds64(cs.slot(ci, ptr));
            // its own slot now takes the entry RING positions ahead (one group per iteration)
            cp_req8_if(rem >= (uint32_t)RING, cs.slot(ci, ptr + (RING - 1)), ptr + (RING - 1));
        } else {                                                     // segment end: next non-empty segment
            const uint32_t g = __ldcg(&p.ck_gate[lane_recs(p)[tid & 31].id]);
            const uint32_t src = __ldg(&p.pin_src[__ldg(&p.gate[g].pin_off) + (uint32_t)b]);
            const Seg sg = next_segment(p, lds32(cs.ck(ci)), src);
            hn = kInfEntry;
            if (sg.rem) {
                ptr = sg.ptr;
                rem = sg.rem;
                sts32(cs.ck(ci), sg.ck);
                ring_fill(cs, ci, ptr, rem);
                hn = ldg_entry(ptr);
                cp_commit();
                cp_wait<0>();                                        // (rare: a synchronous refill)
            }
        }
        cp_commit();
        const uint32_t nh = rem ? to_rel(hn, b4) : kRelInf;
#if GLS_PF > 0
        // entering a new 128-byte line: bring the line GLS_PF lines ahead into L2
        if ((((uint32_t)(uintptr_t)ptr) & 127u) == 0u && rem > 16u * GLS_PF)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr + 16 * GLS_PF));
#endif
        sts64(cs.ptr(ci), (uint64_t)ptr);
        sts32(cs.rem(ci), rem);
        h0 = b == 0 ? nh : h0;
        h1 = b == 1 ? nh : h1;
        h2 = b == 2 ? nh : h2;
        h3 = b == 3 ? nh : h3;
        const uint32_t tq = m | 3u;
        m = min(min(h0, h1), min(h2, h3));
        if ((m | 3u) == tq) continue;                                // more entries at this timestamp
        cnt += tq >= t0q ? 1u : 0u;
        // ---- one distinct timestamp tq (entry form | 3) with raw input vector nr (Alg. 2 body)
        const uint32_t nn = nr ^ ((nr >> 1) & nr & 0x55u);           // Z -> X
        if (nn != xn) {
            const uint32_t E = lds8(lutb + nn);                      // calculateSignals
            if (E != Eprev) {                                        // "o_k.v is changed" (R4a)
                const uint32_t d = nn ^ xn;
                uint32_t cm = (d | (d >> 1)) & 0x55u;                // changed pins (R3)
                uint32_t del = 0xffffffffu;
                do {
                    const int bb = __ffs(cm) - 1;
                    // rise iff rank(new) > rank(old), rank 0 < X < 1 (R2)
                    const uint32_t rise = (0x206u >> ((((xn >> bb) & 3u) << 2) | ((nn >> bb) & 3u))) & 1u;
                    const uint32_t dw = lds32(dt_sa + (uint32_t)((bb >> 1) * 2 + (int)rise) * (kThreads * 4));
                    // (E = 0, 1: the half; X: the smaller half, R1) — min rule
                    del = min(del, E == 2u ? min(dw & 0xFFFFu, dw >> 16) : __funnelshift_r(dw, 0u, 16u * E) & 0xFFFFu);
                    cm &= cm - 1;
                } while (cm);
                const uint32_t rq = ((tq >> 2) + del) << 2;          // appearance time, entry form
                // addSignalChange with Eq. 1: deny every pending schedule at >= rq
                // (del = 0xFFFF: every changed pin is unrelated, nothing scheduled, R9)
                const uint32_t fl = nfl & 0xffffu;
                while (del != kDelayInf16 && n > fl && top >= rq) {
                    --n;
                    top = n > fl ? to_rel(ldg64(scr + n - 1), b4) : 0u;
                }
                const uint32_t tv = n > fl ? (top & 3u) : (nfl >> 16);
                if (tv != E && del != kDelayInf16) {                 // push unless it repeats the tail
                    if (n < cap) {
                        top = rq | E;
                        stg64(scr + n, (uint64_t)top + b4);
                        ++n;
                    } else {
                        lim = 0;                                     // the page is full: restart larger
                        m = kRelInf;
                        n = 0xffffffffu;
                    }
                }
                cnt += tq >= t0q ? 0x10000u : 0u;
                Eprev = E;
            }
            xn = nn;
        }
    }
    S.b4[tid] = b4;
    S.h[0][tid] = h0;
    S.h[1][tid] = h1;
    S.h[2][tid] = h2;
    S.h[3][tid] = h3;
    S.nr[tid] = nr;
    S.xn[tid] = xn;
    S.eprev[tid] = Eprev;
    S.t0q[tid] = t0q;
    S.lim[tid] = lim;
    S.n[tid] = n;
    S.nfl[tid] = nfl;
    S.top[tid] = top;
    l_cnt = cnt;
    return it;
}

// Service point (whole warp, converged): publish finished chunks, claim ids for idle
// lanes, mark lanes whose id is published ready.  Returns false when the run is over
// (every gate complete, or an error).
__device__ __noinline__ bool service(const SimParams& p, unsigned& backoff, unsigned long long& seen,
                                     unsigned long long& t_seen) {
    LaneRec* const LR = lane_recs(p);
    WarpAcc& A = wacc();
    const int lane = threadIdx.x & 31;
    const long long c0 = clock64();
    // ---- publish finished chunks (one after the other, whole warp)
    unsigned done = __ballot_sync(FULL, LR[lane].st == S_DONE);
    const bool any_done = done != 0;
    while (done) {
        const int l = __ffs(done) - 1;
        done &= done - 1;
        const LaneRec& R = LR[l];
        const unsigned long long id = R.id;
        ChunkResult C;
        C.gi = __ldcg(&p.ck_gate[id]);
        C.nch = __ldcg(&p.net_nck[p.P + C.gi]);
        C.s.T0 = R.T0;
        C.total = R.hi - R.lo;
        C.off = R.sb + R.lo;
        C.fits = true;
        C.vb = R.vb;
        C.evals = R.ev;
        C.events = R.evt;
        __syncwarp();
        chunk_done<true>(p, id, C, A.acc);
        if (lane == l) LR[lane].st = S_IDLE;
        __syncwarp();
    }
    const long long c1 = clock64();
    // ---- claim: idle lanes take the next ids of the queue (one atomicAdd for the warp;
    // an id may be published a little later: its lane waits at the next service points)
    const unsigned idle = __ballot_sync(FULL, LR[lane].st == S_IDLE);
    if (idle) {
        unsigned long long h = 0, k = 0;
        if (lane == 0) {
            const unsigned long long head = ld_relaxed_u64(&p.ctl->work_head);
            const unsigned long long top = ld_relaxed_u64(&p.ctl->chunk_top);
            k = top > head ? min((unsigned long long)__popc(idle), top - head) : 0ull;
            if (ld_relaxed_u32(&p.ctl->error) != 0u) k = 0;          // the run is aborting: take nothing
            if (k) h = atomicAdd(&p.ctl->work_head, k);
        }
        h = __shfl_sync(FULL, h, 0);
        k = __shfl_sync(FULL, k, 0);
        const unsigned r = __popc(idle & ((1u << lane) - 1u));
        if ((idle >> lane) & 1u && r < k) {
            LR[lane].id = h + r;
            LR[lane].st = S_CLAIMED;
        }
    }
    __syncwarp();
    // ---- lanes whose id is published are ready to set up
    bool ready = false;
    if (LR[lane].st == S_CLAIMED) {
        const unsigned long long id = LR[lane].id;
        if (id < p.ck_cap && ld_relaxed_u32(&p.ck_gate[id]) != 0xffffffffu) {
#if GLS_ACQ_CLAIM
            (void)ld_acquire_u32(&p.ck_gate[id]);                    // pairs with plan_gate's release
#endif
            ready = true;
            LR[lane].st = S_READY;
        }
    }
    const unsigned nready = __ballot_sync(FULL, ready);
    // (the per-lane engine for long delays runs in the set-up, synchronously: the warp's
    // deep-ring region is free again)
    if (nready && lane == 0) p.deep_wtop[warp_global_id()] = 0;
    const unsigned run = __ballot_sync(FULL, LR[lane].st == S_RUN) | nready;
    const long long c2 = clock64();
    if (lane == 0) {
        A.acc[A_CYC + 3] += (unsigned long long)(c1 - c0);
        A.acc[A_CYC + 0] += (unsigned long long)(c2 - c1);
    }
    if (run == 0) {
        // nothing to sweep: is the run over?  Else back off until work is published.
        if (__shfl_sync(FULL, lane == 0 ? (int)(ld_relaxed_u32(&p.ctl->error) != 0u) : 0, 0)) return false;
        unsigned long long dg = 0;
        if (lane == 0) dg = ld_relaxed_u64(&p.ctl->done_gates);
        dg = __shfl_sync(FULL, dg, 0);
        if (dg >= (unsigned long long)p.G) return false;
        if (lane == 0) {
            const unsigned long long now = gtimer();                 // watchdog: 10 s without a completion
            if (dg != seen) {
                seen = dg;
                t_seen = now;
            } else if (now - t_seen > 10000000000ull) {
                atomicOr(&p.ctl->error, kErrWatchdog);
            }
        }
        if (!any_done) {
            __nanosleep(backoff);
            if (backoff < GLS_MAXSLEEP) backoff <<= 1;
        }
        if (lane == 0) A.acc[A_CYC + 4] += (unsigned long long)(clock64() - c2);
    } else {
        backoff = GLS_MINSLEEP;
    }
    __syncwarp();
    return true;
}

// The whole run of one warp: service points, set-ups and sweep rounds.
__device__ __noinline__ void run(const SimParams& p) {
    LaneRec& R = lane_recs(p)[threadIdx.x & 31];
    WarpAcc& A = wacc();
    const int lane = threadIdx.x & 31;
    R.st = S_IDLE;
    R.top = R.end = 0;
    R.need = 0;
    if (lane == 0)
        for (int k = 0; k < A_N; ++k) A.acc[k] = 0;
    __syncwarp();
    unsigned backoff = GLS_MINSLEEP;
    unsigned long long seen = ~0ull, t_seen = 0;
    for (;;) {
        if (!service(p, backoff, seen, t_seen)) break;
        uint32_t st = R.st;
        unsigned long long dcb = 0;                                  // this lane's set-up clocks
        if (st == S_READY) {
            const long long cb = clock64();
            st = begin(p);
            R.st = st;
            dcb = (unsigned long long)(clock64() - cb);
        }
        {
            const unsigned long long sdc = warp_max64(dcb);
            if (lane == 0) A.acc[A_CYC + 1] += sdc;
        }
        // ---- sweep round
        const long long cs0 = clock64();
        int it = 0;
        if (st == S_RUN) {
            uint32_t cnt = 0;
            it = sweep_round(p, st, cnt);
            R.ev += cnt & 0xffffu;
            R.evt += cnt >> 16;
            if (st != S_RUN) {
                st = finish(p, state().n[threadIdx.x], state().cap[threadIdx.x]);
                R.st = st;
            }
        }
        // ---- lane-utilisation counters: lane iterations vs 32 x the longest lane's
        const unsigned itmax = __reduce_max_sync(FULL, (unsigned)it), itsum = __reduce_add_sync(FULL, (unsigned)it);
        if (lane == 0) {
            A.acc[A_WARP_IT] += 32ull * itmax;
            A.acc[A_LANE_IT] += itsum;
            if (itmax) A.acc[A_CYC + 2] += (unsigned long long)(clock64() - cs0);
        }
        __syncwarp();
    }
    __syncwarp();
    if (lane == 0) acc_flush(p, A);
    __syncwarp();
}

}  // namespace au

size_t auto_lane_bytes(int blocks) { return (size_t)blocks * kThreads * sizeof(au::LaneRec); }

}  // namespace gls
