// gls_lanes.cuh — engine 0 (default): one warp per batch of (gate, time-chunk) work
// items, its lanes on time-slice *units* of them, rebalanced inside the warp while
// they run.  Included by gls_kernels.cu.  DESIGN.md §7.
//
// A unit is a time range [T0, T1) of one chunk of gate g.  It is an exact time chunk
// (DESIGN.md §4): the lane starts at tau0 = T0 - (dmax + 1) with the inputs' values
// there and runs Algorithm 2 sequentially over the merged fan-in lists:
//   * one fan-in ENTRY per iteration (the pin holding the smallest head), times
//     relative to a base B in 32 bits (entry form ((t - B) << 2) | v, rebased when
//     the sweep passes B + 2^29), cursors in shared memory, a one-entry lookahead
//     per pin copied global -> shared by cp.async;
//   * a timestamp is evaluated once its last entry is applied (LUT in shared
//     memory on the Z -> X normalised vector), an event is a change
//     of that evaluation (reading R4a), its delay the min over the pins that
//     changed (readings R1-R3);
//   * Eq. 1 is the paper's own addSignalChange list, kept as a STACK
//     in the lane's output scratch: every schedule at >= the new one is denied
//     (popped), the new one is pushed unless it repeats the value below it
//     (P:508 recursion, reading R5 for ties).  The stack is increasing in time, so
//     at the unit's end the change points in [T0, min(T1, duration + 1)) are one
//     contiguous run of it (the entries before T0 give the value before the
//     unit, the ones after T1 are the next unit's).  No pending ring, no drain,
//     no backtrace limit (reading R13).
// A batch's units are cut statically at quantiles of each chunk's longest fan-in,
// pulled from a warp queue, and every ROUND iterations the warp re-balances: an
// idle lane takes the upper half (in time) of the busiest lane's remaining range
// — again an exact unit, by the same halo argument — so lanes stay busy whatever
// the activity skew (the straggler problem of P:543, inside a warp).
// A unit's outputs are the run of its stack; a chunk's outputs are its units'
// runs in time order: one prefix, one atomicAdd for its exact segment (P:499,
// no page waste), a per-lane copy.  A unit whose stack overflows the lane
// scratch, or whose gate has a delay >= 2^16, runs the per-lane ring engine
// (run_chunk, exact with the deep ring) instead.
#pragma once

namespace gls {
namespace ln {

constexpr unsigned FULL = 0xffffffffu;
constexpr uint32_t kRelInf = 0xffffffffu;
constexpr uint32_t kRebaseQ = 0x80000000u;       // entry form of t - B = 2^29
constexpr uint32_t kFastDelay = 0xFFFFu;         // gates with dmax below this use the 32-bit sweep (u16 delays;
                                                 // 0xFFFF there = GLS_DELAY_INF)
#ifndef GLS_LCAP
#define GLS_LCAP 8192
#endif
constexpr int LCAP = GLS_LCAP;                   // per-lane output scratch (stack) entries
constexpr unsigned long long U_MAX = LCAP / 4;   // most expected entries of a static unit
constexpr size_t kScratchPerWarp = 32u * LCAP;
#ifndef GLS_WLANE
#define GLS_WLANE 256
#endif
constexpr int W_LANE = GLS_WLANE;                // a batch is filled up to 32 x W_LANE expected entries
#ifndef GLS_WMIN
#define GLS_WMIN 32
#endif
constexpr int W_MIN = GLS_WMIN;                  // fewest expected entries per static unit
#ifndef GLS_ROUND
#define GLS_ROUND 512
#endif
constexpr int ROUND = GLS_ROUND;                 // sweep iterations between re-balancing points
#ifndef GLS_ROUND_BIG
#define GLS_ROUND_BIG 512
#endif
constexpr int ROUND_BIG = GLS_ROUND_BIG;         // the same for a batch of one big chunk (>= GLS_ALONE)
#ifndef GLS_MQ_MIN
#define GLS_MQ_MIN 0                             // chunks with at least this many expected entries are
#endif                                           // sliced at merged-count quantiles (0: never)
#ifndef GLS_MINSPLIT
#define GLS_MINSPLIT 64
#endif
constexpr float MINSPLIT = (float)GLS_MINSPLIT;  // split only a remainder of >= 2 x this many entries
#ifndef GLS_MAXSPLIT
#define GLS_MAXSPLIT 8
#endif
constexpr int MAXSPLIT = GLS_MAXSPLIT;           // splits per re-balancing point
#ifndef GLS_MINSLEEP
#define GLS_MINSLEEP 64                          // ns: first back-off of a waiting warp
#endif
#ifndef GLS_MAXSLEEP
#define GLS_MAXSLEEP 8192                        // ns: longest back-off of a warp waiting for published work
#endif
#ifndef GLS_BATCH_AA
#define GLS_BATCH_AA 32                          // backlog above which a busy warp claims more ids by
#endif                                           // atomicAdd (0: compare-and-swap on a published head only)
#ifndef GLS_ALONE
#define GLS_ALONE 4096                           // chunks of at least this many expected entries form a batch alone
#endif
#ifndef GLS_ADAPT
#define GLS_ADAPT 0                              // 1: one chunk per batch when the queue is shallow (dataflow)
#endif
#ifndef GLS_ADAPT_FILL
#define GLS_ADAPT_FILL 1                         // expected entries a shallow-queue batch is filled to
#endif
#ifndef GLS_MAXU
#define GLS_MAXU 64
#endif
#ifndef GLS_MAXC
#define GLS_MAXC 16
#endif
constexpr int MAXC = GLS_MAXC;                   // chunks per batch
constexpr int MAXU = GLS_MAXU;                   // units per batch (static + split)
constexpr int MAXU_STATIC = MAXU * 5 / 8;        // static units per batch (the rest is room for splits)
constexpr uint8_t kEnd = 0xff;

__device__ __forceinline__ uint64_t lds64(uint32_t a) {
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
    uint16_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts64(uint32_t a, uint64_t v) { asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v)); }
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v)); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
// wait_group 0 if same (the pin's request is the newest group) else wait_group 1, without a branch
__device__ __forceinline__ void cp_wait_pin(int b, int lastpin) {
    asm volatile("{\n .reg .pred p;\n setp.eq.s32 p, %0, %1;\n @p cp.async.wait_group 0;\n"
                 " @!p cp.async.wait_group 1;\n}\n" ::"r"(b), "r"(lastpin) : "memory");
}
// request one entry (8 B, global -> shared) and commit it as a group, if `go` (predicated)
__device__ __forceinline__ void cp_async8_if(bool go, uint32_t sa, const void* g) {
    asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %0, 0;\n @p cp.async.ca.shared.global [%1], [%2], 8;\n"
                 " @p cp.async.commit_group;\n}\n" ::"r"((uint32_t)go), "r"(sa), "l"(g) : "memory");
}
// global load of one transition entry (cursor pointers live in shared memory, so the
// compiler cannot infer the state space of their targets)
__device__ __forceinline__ uint64_t ldg_entry(const uint64_t* a) {
    uint64_t v;
    asm("ld.global.u64 %0, [%1];" : "=l"(v) : "l"(a));
    return v;
}
__device__ __forceinline__ uint64_t ldg64(const uint64_t* a) {
    uint64_t v;
    asm volatile("ld.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ void stg64(uint64_t* a, uint64_t v) { asm volatile("st.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory"); }
__device__ __forceinline__ uint32_t to_rel(uint64_t e, uint64_t b4) {
    const uint64_t d = e - b4;
    return (d >> 32) ? kRelInf : (uint32_t)d;
}

// per-thread cursor columns in shared memory, [pin * kThreads + tid]
struct PinSm {
    uint32_t b;
    __device__ __forceinline__ uint32_t ptr(int ci) const { return b + (uint32_t)ci * 8u; }                       // head entry address
    __device__ __forceinline__ uint32_t rem(int ci) const { return b + 4u * kThreads * 8u + (uint32_t)ci * 4u; }  // entries from the head on
    __device__ __forceinline__ uint32_t ck(int ci) const { return b + 4u * kThreads * 12u + (uint32_t)ci * 4u; }  // chunk of the segment
    __device__ __forceinline__ uint32_t hn(int ci) const { return b + 4u * kThreads * 16u + (uint32_t)ci * 8u; }  // lookahead entry
};
constexpr size_t kPinSmBytes = (size_t)4 * kThreads * (8 + 4 + 4 + 8);

// next non-empty segment of a net after chunk ck (by value: the cursor stays in registers)
struct Seg {
    const uint64_t* ptr;
    uint32_t rem, ck;
};
__device__ __forceinline__ Seg next_segment(const SimParams& p, uint32_t ck, uint32_t src) {
    const uint32_t ckend = __ldcg(&p.net_ck[src]) + __ldcg(&p.net_nck[src]);
    Seg r{nullptr, 0u, ck};
    while (r.rem == 0 && r.ck + 1 < ckend) {
        ++r.ck;
        GLS_ASSERT(r.ck < p.ck_cap);
        r.ptr = p.arena + __ldcg(&p.ck_off[r.ck]);
        r.rem = __ldcg(&p.ck_cnt[r.ck]);
        GLS_ASSERT(r.rem == 0 || __ldcg(&p.ck_off[r.ck]) + r.rem <= p.arena_cap);
    }
    return r;
}

// per-warp statistics, accumulated in shared memory and added to Ctl once per warp
enum Acc { A_EVALS, A_EVENTS, A_OUTS, A_CHUNKS, A_LANE_IT, A_WARP_IT, A_BATCHES, A_BLANES, A_BEST,
           A_CYC, A_BAL = A_CYC + 6, A_N = A_BAL + 8 };
// balance counters (gls_stats.balance): [0] static units, [1] split units, [2] re-balancing
// rounds, [3] fallback units, [4] units set up, [5] iterations spent in unit setup
struct Batch {
    unsigned long long acc[A_N];
    unsigned long long id[MAXC];           // chunk ids
    unsigned long long c_off[MAXC];        // arena offset of the chunk's segment (~0: did not fit)
    long long c_T0[MAXC];                  // chunk start time
    uint32_t c_total[MAXC];
    uint8_t c_first[MAXC], c_nsl[MAXC];    // first unit, static slices
    uint8_t c_inf[MAXC];                   // the chunk's gate has a GLS_DELAY_INF pin: one unit, never split
    long long u_T0[MAXU], u_T1[MAXU];      // unit time range
    uint32_t u_est[MAXU];                  // expected merged entries
    uint8_t u_chunk[MAXU], u_slice[MAXU], u_lane[MAXU], u_vb[MAXU], u_st[MAXU], u_next[MAXU];
    int qhead;                             // next static unit to hand out
    int round;                             // re-balancing rounds of the batch so far
    uint16_t u_r0[MAXU];                   // round in which the unit started
    int nun;                               // units (static + split)
    int big;                               // the batch is one big chunk (GLS_ALONE)
    int8_t pend[32];                       // unit handed to a lane by a split (-1: none)
    uint32_t lev[32], levt[32];            // per-lane gate-evals / events of the batch
    uint16_t sv_it[32];                    // (set-up call: the lane's round iteration,
    uint16_t sv_used[32];                  //  scratch fill)
    int8_t u_lnext[MAXU];                  // next unit taken by the same lane (-1: last)
    int8_t lane_first[32], lane_last[32];  // the lane's units in the order it took them
};
constexpr size_t kBatchBytes = (sizeof(Batch) + 15) & ~(size_t)15;
// rarely used per-unit fields in global memory (per warp), so that the shared Batch
// leaves room for L1
struct WarpAux {
    uint32_t u_deep[MAXU];                 // fallback: deep-ring offset in the warp's region (~0: none)
    uint32_t u_sev[MAXU], u_sevt[MAXU];    // the lane's counts when the unit started
    // unit outputs: lane-scratch offset, count, offset inside the chunk's segment (written by
    // one lane, read by others after __syncwarp: accessed with ld/st.cg, L2 only)
    uint32_t u_soff[MAXU], u_cnt[MAXU], u_pre[MAXU];
    unsigned long long c_t[MAXC];          // claim time (gls_config.trace; lane 0 only)
    unsigned long long lcyc[32];           // per-lane clocks spent in unit set-up (own lane only)
    uint32_t lit[32], lsu[32];             // per-lane iterations / unit set-ups of the batch (trace)
};
__device__ __forceinline__ WarpAux& warp_aux(const SimParams& p) {
    return reinterpret_cast<WarpAux*>(p.waux)[warp_global_id()];
}
// the same, recomputed at each use (an opaque base: not hoisted out of the sweep loop, where
// a live 64-bit address would cost registers the entry path needs)
__device__ __forceinline__ WarpAux& warp_aux_cold(const SimParams& p) {
    void* a;
    asm volatile("mov.b64 %0, %1;" : "=l"(a) : "l"(p.waux));
    return reinterpret_cast<WarpAux*>(a)[warp_global_id()];
}

// Shared memory of a CTA (namespace scope, so addresses are constants plus the thread
// index, not registers): the 4-value LUT (a3, staged per CTA), then per-thread delay
// tables (u16 [24][kThreads]), one Batch per warp, the per-thread pin cursor columns.
constexpr int kDtabWords = 16;                   // u16 halves of 8 words [pin][edge] = d(->0) | d(->1) << 16
__shared__ uint8_t g_lut[kLutCap];
extern __shared__ __align__(16) unsigned char g_dyn[];
constexpr size_t kDynBytes = (size_t)kDtabWords * kThreads * 2 + kBatchBytes * (kThreads / 32) + kPinSmBytes;
__device__ __forceinline__ Batch& warp_batch() {
    return reinterpret_cast<Batch*>(g_dyn + (size_t)kDtabWords * kThreads * 2)[threadIdx.x >> 5];
}
__device__ __forceinline__ PinSm pin_cols() {
    return PinSm{(uint32_t)__cvta_generic_to_shared(g_dyn + (size_t)kDtabWords * kThreads * 2 +
                                                    kBatchBytes * (kThreads / 32))};
}
__device__ __forceinline__ uint32_t* dtab_cols() { return reinterpret_cast<uint32_t*>(g_dyn); }
__device__ __forceinline__ uint32_t lut_sa() { return (uint32_t)__cvta_generic_to_shared(g_lut); }

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

template <class T>
__device__ __forceinline__ void fill_dtab(T* dtab, int dstride, const ChunkSetup& s) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {                       // R1: output X takes the smaller delay
        const uint4 d = s.d[i];
        // (GLS_DELAY_INF -> 0xFFFF, above every finite delay of a gate on this path; the min
        // for X then takes the related one)
        // (word [pin][edge]: edge 0 = FALL (z, w), 1 = RISE (x, y); the X delay is the min of
        // the halves, taken in the sweep)
        const uint32_t z = min(d.z, 0xFFFFu), w = min(d.w, 0xFFFFu), x = min(d.x, 0xFFFFu), y = min(d.y, 0xFFFFu);
        dtab[(i * 2 + 0) * dstride] = (T)(z | w << 16);
        dtab[(i * 2 + 1) * dstride] = (T)(x | y << 16);
    }
}

// ChunkSetup of unit u (its chunk's gate, pins and delays; the unit's time range)
__device__ __forceinline__ void unit_setup(const SimParams& p, const Batch& B, int u, ChunkSetup& s) {
    uint32_t gi, cidx, nch;
    setup_chunk(p, B.id[B.u_chunk[u]], s, gi, cidx, nch);
    s.T0 = B.u_T0[u];
    s.T1 = B.u_T1[u];
    s.tau0 = s.T0 - (long long)s.dmax - 1;
}

// The per-lane ring engine on one unit (fallback): count pass (deep ring if the
// 32-entry ring overflows; its region is kept for the write pass).
__device__ __noinline__ void fallback_count(const SimParams& p, Batch& B, int u, const uint8_t* lut,
                                            uint32_t& evals, uint32_t& events) {
    ChunkSetup s;
    unit_setup(p, B, u, s);
    ChunkOut r{0, 0, 0, 2, false};
    WarpAux& X = warp_aux(p);
    X.u_deep[u] = 0xffffffffu;
    run_chunk<false, false>(p, s, lut, nullptr, nullptr, 0, r);
    if (r.overflow) {
        const unsigned long long dcap = window_bound(p, s);
        const unsigned long long at = deep_alloc(p, dcap);
        r = ChunkOut{0, 0, 0, 2, false};
        if (at != ~0ull) {
            X.u_deep[u] = (uint32_t)(at - (unsigned long long)warp_global_id() * p.deep_per_warp);
            run_chunk<false, true>(p, s, lut, nullptr, p.deep + at, dcap, r);
        }
    }
    __stcg(&X.u_cnt[u], r.cnt);
    B.u_vb[u] = (uint8_t)r.vb;
    evals += r.evals;
    events += r.events;
}
__device__ __noinline__ void fallback_write(const SimParams& p, const Batch& B, int u, const uint8_t* lut,
                                            uint64_t* dst) {
    ChunkSetup s;
    unit_setup(p, B, u, s);
    ChunkOut r{0, 0, 0, 2, false};
    const uint32_t dofs = warp_aux(p).u_deep[u];
    if (dofs == 0xffffffffu) {
        run_chunk<true, false>(p, s, lut, dst, nullptr, 0, r);
    } else {
        const unsigned long long dcap = window_bound(p, s);
        run_chunk<true, true>(p, s, lut, dst,
                              p.deep + (unsigned long long)warp_global_id() * p.deep_per_warp + dofs, dcap, r);
    }
    if (r.cnt != __ldcg(&warp_aux(p).u_cnt[u]) || r.overflow) atomicOr(&p.ctl->error, kErrBug);
}

// per-base thresholds (entry form, relative to B = b4 >> 2): t >= T0 <=> e >= t0q;
// the sweep stops at a head >= lim (T1, or B + 2^29 when more: rebase first)
__device__ __forceinline__ void thresholds(uint64_t b4, long long T0, long long T1, uint32_t& t0q, uint32_t& lim,
                                           int& more) {
    const long long Bs = (long long)b4 >> 2;
    const long long a0 = T0 - Bs, a2 = T1 - Bs;
    t0q = a0 <= 0 ? 0u : (a0 < (1ll << 30) ? (uint32_t)(a0 << 2) : kRelInf);
    more = a2 >= (1ll << 29);
    lim = more ? kRebaseQ : (a2 <= 0 ? 0u : (uint32_t)(a2 << 2));
}

// Cursors of all k pins at tau0 (as locate(), gls_kernels.cu): the binary searches over
// the chunk start times and then inside the segments advance in lockstep, so the k chains
// of dependent global loads overlap — the set-up latency of a unit is about one search,
// not k.
__device__ __forceinline__ void locate_all(const SimParams& p, const uint32_t* src, uint32_t k, long long tau0,
                                           Cursor* c, uint32_t* init) {
    uint32_t cb[4], lo[4], hi[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        cb[i] = (uint32_t)i < k ? __ldcg(&p.net_ck[src[i]]) : 0u;
        lo[i] = 0;
        hi[i] = (uint32_t)i < k ? __ldcg(&p.net_nck[src[i]]) : 1u;
        c[i].ck_end = cb[i] + hi[i];
    }
    for (;;) {                                      // largest j with ck_T[j] <= tau0 + 1 (default 0)
        bool any = false;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (hi[i] - lo[i] > 1) {
                any = true;
                const uint32_t mid = (lo[i] + hi[i]) >> 1;
                if (__ldcg(&p.ck_T[cb[i] + mid]) <= tau0 + 1) lo[i] = mid; else hi[i] = mid;
            }
        }
        if (!any) break;
    }
    const uint64_t* seg[4];
    uint32_t a[4], b[4], cnt[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t j = cb[i] + lo[i];
        GLS_ASSERT((uint32_t)i >= k || (j < p.ck_cap && j < c[i].ck_end &&
                                        __ldcg(&p.ck_off[j]) + __ldcg(&p.ck_cnt[j]) <= p.arena_cap));
        seg[i] = (uint32_t)i < k ? p.arena + __ldcg(&p.ck_off[j]) : p.arena;
        cnt[i] = (uint32_t)i < k ? __ldcg(&p.ck_cnt[j]) : 0u;
        a[i] = 0;
        b[i] = cnt[i];
        c[i].ck = j;
    }
    for (;;) {                                      // first index with t > tau0
        bool any = false;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (a[i] < b[i]) {
                any = true;
                const uint32_t m = (a[i] + b[i]) >> 1;
                if (etime(seg[i][m]) <= tau0) a[i] = m + 1; else b[i] = m;
            }
        }
        if (!any) break;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if ((uint32_t)i >= k) continue;
        init[i] = a[i] > 0 ? (uint32_t)(seg[i][a[i] - 1] & 3u) : (uint32_t)__ldcg(&p.ck_vb[c[i].ck]);
        c[i].ptr = seg[i] + a[i];
        c[i].end = seg[i] + cnt[i];
        refill(p, c[i]);
    }
}

// Number of entries before time T summed over the k pins' nets (count_before of
// gls_kernels.cu for all pins at once, the binary searches in lockstep).
__device__ unsigned long long count_before_all(const SimParams& p, const uint32_t* src, uint32_t k, long long T) {
    uint32_t cb[4], lo[4], hi[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        cb[i] = (uint32_t)i < k ? __ldcg(&p.net_ck[src[i]]) : 0u;
        lo[i] = 0;
        hi[i] = (uint32_t)i < k ? __ldcg(&p.net_nck[src[i]]) : 1u;
    }
    for (;;) {                                      // largest j with ck_T[j] <= T (default 0)
        bool any = false;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (hi[i] - lo[i] > 1) {
                any = true;
                const uint32_t mid = (lo[i] + hi[i]) >> 1;
                if (__ldcg(&p.ck_T[cb[i] + mid]) <= T) lo[i] = mid; else hi[i] = mid;
            }
        }
        if (!any) break;
    }
    const uint64_t* seg[4];
    uint32_t a[4], b[4];
    unsigned long long base = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t j = cb[i] + lo[i];
        seg[i] = (uint32_t)i < k ? p.arena + __ldcg(&p.ck_off[j]) : p.arena;
        a[i] = 0;
        b[i] = (uint32_t)i < k ? __ldcg(&p.ck_cnt[j]) : 0u;
        base += (uint32_t)i < k ? __ldcg(&p.ck_cum[j]) : 0ull;
    }
    for (;;) {                                      // first index with t >= T
        bool any = false;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (a[i] < b[i]) {
                any = true;
                const uint32_t m = (a[i] + b[i]) >> 1;
                if (etime(seg[i][m]) < T) a[i] = m + 1; else b[i] = m;
            }
        }
        if (!any) break;
    }
    return base + a[0] + a[1] + a[2] + a[3];
}

// Start unit u on this lane (the set-up path, kept out of the sweep's registers):
// its delay table, the cursors of its pins at tau0 = T0 - dmax - 1 (binary search over
// chunk start times, then inside the segment; value in effect from ck_vb), the first
// heads relative to B = tau0.  false: the gate has a delay >= 2^16 (fallback unit).
struct UnitInit {
    uint64_t b4;
    uint32_t h[4];
    uint32_t xn, xr0, lutb, t0q, lim;
    int more;
};
__device__ __noinline__ bool unit_begin(const SimParams& p, int u, UnitInit& o) {
    Batch& B = warp_batch();
    const PinSm cs = pin_cols();
    const int tid = threadIdx.x, lane = tid & 31;
    B.u_lane[u] = (uint8_t)lane;
    B.u_lnext[u] = -1;                                                   // append u to the lane's list
    if (B.lane_last[lane] >= 0) B.u_lnext[B.lane_last[lane]] = (int8_t)u; else B.lane_first[lane] = (int8_t)u;
    B.lane_last[lane] = (int8_t)u;
    ChunkSetup s;
    unit_setup(p, B, u, s);
    if (s.dmax >= kFastDelay) {
        B.u_st[u] = 1;
        return false;
    }
    fill_dtab(dtab_cols() + tid, (int)blockDim.x, s);
    o.lutb = lut_sa() + s.lut_base;
    const uint64_t b4 = (uint64_t)s.tau0 << 2;
    o.b4 = b4;
    uint32_t xn = 0, xr0 = 0;
    Cursor cur[4];
    uint32_t ini[4];
    locate_all(p, s.src, s.k, s.tau0, cur, ini);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int ci = i * kThreads + tid;
        o.h[i] = kRelInf;
        if ((uint32_t)i >= s.k) {
            sts32(cs.rem(ci), 0u);                                       // absent pin: exhausted
        } else {
            const Cursor& cc = cur[i];
            const uint32_t init = ini[i];
            const uint32_t rem = (uint32_t)(cc.end - cc.ptr);
            sts64(cs.ptr(ci), (uint64_t)cc.ptr);
            sts32(cs.rem(ci), rem);
            sts32(cs.ck(ci), cc.ck);
            sts64(cs.hn(ci), rem > 1 ? cc.ptr[1] : kInfEntry);
            o.h[i] = rem ? to_rel(*cc.ptr, b4) : kRelInf;
            xn |= 2u << (2 * i);                                         // inputs start at X
            xr0 |= init << (2 * i);                                      // raw values in effect at tau0
        }
    }
    o.xn = xn;
    o.xr0 = xr0;
    thresholds(b4, s.T0, s.T1, o.t0q, o.lim, o.more);
    return true;
}

// Rebase (the sweep reached B + 2^29 before T1): the stack entries before the true next
// head tmin are final (any later event appears at >= tmin), B moves to tmin.  false:
// no input left before T1 (the unit is done).
struct RebaseIO {
    uint64_t b4;
    uint32_t h[4];
    uint32_t n, nfloor, floorv, top, t0q, lim;
    int more;
};
__device__ __forceinline__ bool unit_rebase(const SimParams& p, const Batch& B, int u, PinSm cs, uint32_t sbase,
                                         RebaseIO& io) {
    const int tid = threadIdx.x;
    const uint64_t* scr = p.wscr + sbase;
    uint64_t raw = kInfEntry;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int ci = i * kThreads + tid;
        if (lds32(cs.rem(ci))) raw = min(raw, ldg_entry((const uint64_t*)lds64(cs.ptr(ci))));
    }
    const long long T1 = B.u_T1[u];
    const long long tmin = raw == kInfEntry ? LLONG_MAX : etime(raw);
    if (tmin >= T1) return false;
    const uint64_t tminq = (uint64_t)tmin << 2;
    uint32_t f = io.n;
    while (f > io.nfloor && ((long long)scr[f - 1] >> 2) >= tmin) --f;
    if (f > io.nfloor) {
        io.floorv = (uint32_t)(scr[f - 1] & 3u);
        io.nfloor = f;
    }
    io.b4 = tminq;                                                       // every live entry is >= tmin
    thresholds(io.b4, B.u_T0[u], T1, io.t0q, io.lim, io.more);
    io.top = io.n > io.nfloor ? to_rel(scr[io.n - 1], io.b4) : 0u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int ci = i * kThreads + tid;
        io.h[i] = lds32(cs.rem(ci)) ? to_rel(ldg_entry((const uint64_t*)lds64(cs.ptr(ci))), io.b4) : kRelInf;
    }
    return true;
}

// Unit u is done: its outputs are the stack entries (increasing in time) in
// [T0, min(T1, duration + 1)) — one contiguous run; the entry below it gives the value
// before T0 (X if none).  n == ~0: the stack overflowed (fallback unit).
__device__ __forceinline__ void unit_end(const SimParams& p, Batch& B, int u, uint32_t sbase, uint32_t n,
                                      uint32_t& used, uint32_t l_cnt) {
    if (n == 0xffffffffu) {
        // the fallback counts the whole unit again: take back what this partial run counted
        const int lane = threadIdx.x & 31;
        B.u_st[u] = 1;
        B.lev[lane] -= B.lev[lane] + (l_cnt & 0xffffu) - warp_aux_cold(p).u_sev[u];
        B.levt[lane] -= B.levt[lane] + (l_cnt >> 16) - warp_aux_cold(p).u_sevt[u];
        return;
    }
    const uint64_t* scr = p.wscr + sbase;
    const long long T0 = B.u_T0[u], T1e = min(B.u_T1[u], p.duration + 1);
    uint32_t lo = used, hi = n, vb = 2u;
    while (lo < hi && ((long long)scr[lo] >> 2) < T0) ++lo;
    while (hi > lo && ((long long)scr[hi - 1] >> 2) >= T1e) --hi;
    if (lo > used) vb = (uint32_t)(scr[lo - 1] & 3u);
    __stcg(&warp_aux_cold(p).u_soff[u], lo);
    __stcg(&warp_aux_cold(p).u_cnt[u], hi - lo);
    B.u_vb[u] = (uint8_t)vb;
    used = hi;
}

// driver net of pin b of unit u's gate (segment crossings only: a few dependent loads)
__device__ __forceinline__ uint32_t unit_src(const SimParams& p, const Batch& B, int u, int b) {
    const uint32_t g = __ldcg(&p.ck_gate[B.id[B.u_chunk[u]]]);
    return __ldg(&p.pin_src[__ldg(&p.gate[g].pin_off) + (uint32_t)b]);
}

// The sweep of one batch (whole warp): rounds of up to ROUND iterations per lane, the
// warp re-balancing in between.  A function of its own so that only the sweep's state
// competes for registers.  Statistics go to B.acc (lane 0).
__device__ __noinline__ void sweep_rounds(const SimParams& p, int nstatic) {
    Batch& B = warp_batch();
    const int rlen = B.big ? ROUND_BIG : ROUND;
    const PinSm cs = pin_cols();
    const int lane = threadIdx.x & 31;
    const int tid = threadIdx.x;
    // this lane's output scratch (the Eq. 1 stack)
    const uint32_t sbase = (warp_global_id() * 32u + (uint32_t)lane) * (uint32_t)LCAP;
    uint64_t* const scr = p.wscr + sbase;
    const uint32_t dt_sa = (uint32_t)__cvta_generic_to_shared(dtab_cols() + tid);   // [q * blockDim.x + tid]
    int u = -1;                            // current unit
    uint32_t used = 0;                     // lane scratch fill
    uint32_t l_cnt = 0;                    // this round's gate-evals (bits 0-15) and events (16-31), <= ROUND each
    // sweep state of the current unit
    uint64_t b4 = 0;                       // base B in entry form
    uint32_t h0 = kRelInf, h1 = kRelInf, h2 = kRelInf, h3 = kRelInf, m = kRelInf;
    uint32_t nr = 0, xn = 0, Eprev = 2, lutb = lut_sa();
    uint32_t t0q = 0, lim = 0;             // lim == kRebaseQ: the unit runs beyond B + 2^29 (rebase)
    uint32_t n = 0;                        // Eq. 1 stack: SCR[start .. n)
    uint32_t nfl = 0;                      // entries below (nfl & 0xffff) are final; nfl >> 16: value of the last of them
    uint32_t top = 0;                      // top of the stack, entry form relative to B (n > floor)
    int lastpin = -1;                      // pin of the newest cp.async request
    B.pend[lane] = -1;
    B.lane_first[lane] = B.lane_last[lane] = -1;
    B.lev[lane] = B.levt[lane] = 0;
    if (p.trace) {
        warp_aux_cold(p).lcyc[lane] = 0;
        warp_aux_cold(p).lit[lane] = warp_aux_cold(p).lsu[lane] = 0;
    }
    __syncwarp();

    for (;;) {
        int it = 0;
        for (; it < rlen; ++it) {
            uint32_t tq;
            if (u < 0) {
                // ---- take a unit: handed over by a split, else the next static one
                int v = B.pend[lane];
                if (v >= 0) {
                    B.pend[lane] = -1;
                } else {
                    v = atomicAdd(&B.qhead, 1);
                    if (v >= nstatic) break;
                }
                u = v;
                // the previous unit's state is dead: constants across the set-up call
                b4 = 0;
                h0 = h1 = h2 = h3 = m = kRelInf;
                nr = xn = 0;
                lutb = lut_sa();
                t0q = lim = n = nfl = top = 0;
                Eprev = 2;
                lastpin = -1;
                // nothing but constants lives across the set-up call: the round's counts, the
                // iteration and the scratch fill go through shared memory (set-up path only)
                B.lev[lane] += l_cnt & 0xffffu;
                if (p.trace) warp_aux_cold(p).lit[lane] += (uint32_t)it;
                B.levt[lane] += l_cnt >> 16;
                l_cnt = 0;
                B.sv_it[lane] = (uint16_t)it;
                B.sv_used[lane] = (uint16_t)used;
                UnitInit ui;                                             // (local memory: set-up path only)
                const long long c_u0 = clock64();
                const bool fast = unit_begin(p, u, ui);
                {
                    const unsigned long long dc = (unsigned long long)(clock64() - c_u0);
                    if (p.trace) warp_aux_cold(p).lcyc[lane] += dc;
                    if (lane == __ffs(__activemask()) - 1) B.acc[A_BAL + 4] += dc;   // warp-level: one pass
                }
                if (p.trace) warp_aux_cold(p).lsu[lane] += 1;
                it = B.sv_it[lane];
                used = B.sv_used[lane];
                if (!fast) {                                             // long delays: per-lane ring engine
                    u = -1;
                    continue;
                }
                b4 = ui.b4;
                h0 = ui.h[0];
                h1 = ui.h[1];
                h2 = ui.h[2];
                h3 = ui.h[3];
                xn = ui.xn;
                nr = ui.xr0;
                lutb = ui.lutb;
                t0q = ui.t0q;
                lim = ui.lim;
                asm volatile("" ::: "memory");                           // (keeps the copies in registers: ui is dead)
                warp_aux_cold(p).u_sev[u] = B.lev[lane];                      // counts so far (a fallback takes them back)
                B.u_r0[u] = (uint16_t)B.round;
                warp_aux_cold(p).u_sevt[u] = B.levt[lane];
                n = used;
                nfl = used | (2u << 16);                                 // nothing final yet; value before: X
                top = 0;
                Eprev = 2;
                lastpin = -1;
                m = min(min(h0, h1), min(h2, h3));
                tq = 3u;                                                 // the unit's halo start (t = tau0)
            } else if (m >= lim) {
                if (lim == kRebaseQ) {
                    RebaseIO io{b4, {h0, h1, h2, h3}, n, nfl & 0xffffu, nfl >> 16, top, t0q, lim, 0};
                    if (unit_rebase(p, B, u, cs, sbase, io)) {
                        b4 = io.b4;
                        h0 = io.h[0];
                        h1 = io.h[1];
                        h2 = io.h[2];
                        h3 = io.h[3];
                        nfl = io.nfloor | (io.floorv << 16);
                        top = io.top;
                        t0q = io.t0q;
                        lim = io.lim;
                        m = min(min(h0, h1), min(h2, h3));
                        continue;
                    }
                }
                // ---- unit done: its outputs are the stack entries in [T0, min(T1, duration + 1))
                cp_wait<0>();                                            // no copy may land in the next unit's cursors
                const long long c_e0 = clock64();
                unit_end(p, B, u, sbase, n, used, l_cnt);
                if (lane == __ffs(__activemask()) - 1) B.acc[A_BAL + 5] += (unsigned long long)(clock64() - c_e0);
                u = -1;
                continue;
            } else {
                // ---- one fan-in entry: the pin with the smallest head
                const int b = h0 == m ? 0 : h1 == m ? 1 : h2 == m ? 2 : 3;
                nr = (nr & ~(3u << (2 * b))) | ((m & 3u) << (2 * b));
                const int ci = b * kThreads + tid;
                const uint64_t* ptr = (const uint64_t*)lds64(cs.ptr(ci)) + 1;
                uint32_t rem = lds32(cs.rem(ci)) - 1u;
                GLS_ASSERT(rem < 0x80000000u && ptr >= p.arena && ptr + rem <= p.arena + p.arena_cap);
                cp_wait_pin(b, lastpin);                                 // the pin's lookahead has landed
                uint64_t hn = lds64(cs.hn(ci));
                if (rem == 0) {                                          // segment end: next non-empty segment
                    const Seg g = next_segment(p, lds32(cs.ck(ci)), unit_src(p, B, u, b));
                    if (g.rem) {
                        ptr = g.ptr;
                        rem = g.rem;
                        sts32(cs.ck(ci), g.ck);
                        hn = ldg_entry(ptr);
                    } else {
                        hn = kInfEntry;
                    }
                }
                const uint32_t nh = rem ? to_rel(hn, b4) : kRelInf;
                cp_async8_if(rem > 1, cs.hn(ci), ptr + 1);               // nothing waits for it until pin b moves again
                lastpin = rem > 1 ? b : lastpin;
                sts64(cs.ptr(ci), (uint64_t)ptr);
                sts32(cs.rem(ci), rem);
                h0 = b == 0 ? nh : h0;
                h1 = b == 1 ? nh : h1;
                h2 = b == 2 ? nh : h2;
                h3 = b == 3 ? nh : h3;
                tq = m | 3u;
                m = min(min(h0, h1), min(h2, h3));
                if ((m | 3u) == tq) continue;                            // more entries at this timestamp
                l_cnt += tq >= t0q ? 1u : 0u;
            }
            // ---- one distinct timestamp tq (entry form | 3) with raw input vector nr (Alg. 2 body)
            const uint32_t nn = nr ^ ((nr >> 1) & nr & 0x55u);           // Z -> X
            if (nn != xn) {
                const uint32_t E = lds8(lutb + nn);                      // calculateSignals
                if (E != Eprev) {                                        // "o_k.v is changed" (R4a)
                    const uint32_t d = nn ^ xn;
                    uint32_t cm = (d | (d >> 1)) & 0x55u;                // changed pins (R3)
                    uint32_t del = 0xffffffffu;
                    do {
                        const int b = __ffs(cm) - 1;
                        // rise iff rank(new) > rank(old), rank 0 < X < 1 on normalised codes (R2):
                        // (old, new) in {(0,1), (0,X), (X,1)} = bits 1, 2, 9 of (old << 2 | new)
                        const uint32_t rise = (0x206u >> ((((xn >> b) & 3u) << 2) | ((nn >> b) & 3u))) & 1u;
                        const uint32_t dw = lds32(dt_sa + (uint32_t)((b >> 1) * 2 + (int)rise) * (kThreads * 4));
                        // (E = 0, 1: the half; X: the smaller half, R1) — min rule
                        del = min(del, E == 2u ? min(dw & 0xFFFFu, dw >> 16) : __funnelshift_r(dw, 0u, 16u * E) & 0xFFFFu);
                        cm &= cm - 1;
                    } while (cm);
                    const uint32_t rq = ((tq >> 2) + del) << 2;         // appearance time, entry form
                    // addSignalChange with Eq. 1: deny every pending schedule at >= rq
                    // (del = 0xFFFF: every changed pin is unrelated, nothing scheduled, R9)
                    const uint32_t fl = nfl & 0xffffu;
                    while (del != kDelayInf16 && n > fl && top >= rq) {
                        GLS_ASSERT(n >= 1u && n <= (uint32_t)LCAP);
                        --n;
                        top = n > fl ? to_rel(ldg64(scr + n - 1), b4) : 0u;
                    }
                    const uint32_t tv = n > fl ? (top & 3u) : (nfl >> 16);
                    if (tv != E && del != kDelayInf16) {                 // push unless it repeats the tail
                        if (n < (uint32_t)LCAP) {
                            top = rq | E;
                            GLS_ASSERT(sbase + n < (uint32_t)(gridDim.x * (blockDim.x >> 5)) * 32u * (uint32_t)LCAP);
                            stg64(scr + n, (uint64_t)top + b4);
                            ++n;
                        } else {
                            lim = 0;                                     // stack overflow: fallback unit
                            n = 0xffffffffu;
                        }
                    }
                    l_cnt += tq >= t0q ? 0x10000u : 0u;
                    Eprev = E;
                }
                xn = nn;
            }
        }
        // ---- re-balancing point
        __syncwarp();
        const long long c_rb = clock64();
        {
            const unsigned itmax = __reduce_max_sync(FULL, (unsigned)it), itsum = __reduce_add_sync(FULL, (unsigned)it);
            B.lev[lane] += l_cnt & 0xffffu;
            if (p.trace) warp_aux_cold(p).lit[lane] += (uint32_t)it;
            B.levt[lane] += l_cnt >> 16;
            l_cnt = 0;
            if (lane == 0) {
                B.acc[A_WARP_IT] += 32ull * itmax;
                B.acc[A_LANE_IT] += itsum;
                B.acc[A_BAL + 2] += 1ull;
                B.round = min(B.round + 1, 65535);
            }
        }
        const bool qempty = *(volatile int*)&B.qhead >= nstatic;
        const unsigned idle = __ballot_sync(FULL, u < 0 && B.pend[lane] < 0);
        if (idle == FULL && qempty) break;
        if (!qempty || idle == 0) {
            __syncwarp();
            continue;
        }
        // idle lanes take the upper half (in time) of the busiest lanes' remaining ranges
        float re = 0.f;
        long long tn = 0, T1u = 0, ts = 0;
        if (u >= 0 && m < lim) {
            const long long T0u = B.u_T0[u];
            T1u = B.u_T1[u];
            tn = ((long long)b4 >> 2) + (long long)(m >> 2);             // next timestamp to process
            if (tn >= T0u && T1u - tn >= 2 && B.u_est[u]) {
                // entries left: the unit's estimate scaled by the time left, or the lane's own
                // pace so far (ROUND iterations per round since the unit started) if larger —
                // an estimate from the chunk average misses bursts inside the unit
                const float left = (float)(T1u - tn);
                const float est = (float)B.u_est[u] * left / (float)max(1ll, T1u - T0u);
                const float done = ((float)(B.round - (int)B.u_r0[u]) + 0.5f) * (float)rlen;
                re = fmaxf(est, done * left / (float)max(1ll, tn - T0u));
                ts = tn + (T1u - tn) / 2;                                 // > every timestamp applied so far
            }
        }
        // (a lane whose scratch is half full takes no split: the units it already holds keep
        // their room, and no unit ends in the slow fallback for want of it)
        unsigned rcv = idle & __ballot_sync(FULL, used < (uint32_t)LCAP / 2);
        int nun = B.nun;
        for (int q = 0; q < MAXSPLIT && rcv && nun < MAXU; ++q) {
            const unsigned mx = __reduce_max_sync(FULL, __float_as_uint(re));   // re >= 0: bits order like values
            if (__uint_as_float(mx) < 2.f * MINSPLIT) break;
            const int dl = __ffs(__ballot_sync(FULL, __float_as_uint(re) == mx)) - 1;
            const int rl = __ffs(rcv) - 1;
            rcv &= rcv - 1;
            if (lane == dl) {
                GLS_ASSERT(nun < MAXU && u >= 0 && u < MAXU);
                B.u_T0[nun] = ts;
                B.u_T1[nun] = T1u;
                B.u_chunk[nun] = B.u_chunk[u];
                B.u_slice[nun] = 0xff;
                B.u_next[nun] = B.u_next[u];
                B.u_next[u] = (uint8_t)nun;
                B.u_est[nun] = (uint32_t)(re * 0.5f);
                B.u_st[nun] = 0;
                B.u_T1[u] = ts;
                int mo;
                thresholds(b4, B.u_T0[u], ts, t0q, lim, mo);
                B.pend[rl] = (int8_t)nun;
                re = 0.f;
            }
            ++nun;
            if (lane == 0) B.acc[A_BAL + 1] += 1ull;
        }
        __syncwarp();
        if (lane == 0) {
            B.nun = nun;
            B.acc[A_BAL + 6] += (unsigned long long)(clock64() - c_rb);
        }
        __syncwarp();
    }
    const unsigned ev = __reduce_add_sync(FULL, B.lev[lane]), evt = __reduce_add_sync(FULL, B.levt[lane]);
    const unsigned long long sc = p.trace ? warp_sum64(warp_aux_cold(p).lcyc[lane]) : 0ull;
    if (lane == 0) {
        B.acc[A_EVALS] += ev;
        B.acc[A_EVENTS] += evt;
        B.acc[A_CYC + 5] += sc / 32;                                     // (lane-average set-up clocks)
    }
    __syncwarp();
}

// Whole warp: evaluate one batch.  Returns false when there is no more work
// (dataflow: every gate done or an error; levels: the level is exhausted).
// `carry` (lane 0) holds a claimed chunk id that did not fit the last batch.
template <bool DATAFLOW>
__device__ bool lane_batch(const SimParams& p, unsigned long long& carry, unsigned long long lvl_begin,
                           unsigned long long lvl_n, unsigned long long* lvl_work) {
    Batch& B = warp_batch();
    const uint8_t* lut = g_lut;
    const int lane = threadIdx.x & 31;
    constexpr unsigned long long NONE = ~0ull;
    int nc = 0, nu = 0;
    bool more_work = true;
    const long long c_start = clock64();
    if (lane == 0) {
        // ---- claim published chunks until the batch holds about 32 x W_LANE expected entries
        unsigned long long est[MAXC];
        unsigned long long total = 0;
        int units_needed = 0;
        // shallow queue (fewer published chunks than warps): one chunk per batch, so its
        // units spread over all 32 lanes and the critical path through the netlist shortens
        unsigned long long fill = 32ull * W_LANE;
        if (DATAFLOW && GLS_ADAPT) {
            const unsigned long long pub = ld_relaxed_u64(&p.ctl->chunk_top), head = ld_relaxed_u64(&p.ctl->work_head);
            if (pub < head + (unsigned long long)gridDim.x * (blockDim.x >> 5)) fill = GLS_ADAPT_FILL;
        }
        while (nc < MAXC && total < fill) {
            unsigned long long id;
            if (carry != NONE) {
                id = carry;
                carry = NONE;
            } else if (DATAFLOW) {
                if (nc == 0) {
                    id = atomicAdd(&p.ctl->work_head, 1ull);    // (an idle warp may wait for its id)
                } else {
                    // a busy warp never holds an unpublished id (its consumers would wait for
                    // this whole batch): take the head only if published, by compare-and-swap —
                    // or, with a backlog of allocated ids ahead of the head (GLS_BATCH_AA), by
                    // atomicAdd (such ids are published moments after their allocation; one
                    // that is not yet is carried to the next batch)
                    const unsigned long long h = ld_relaxed_u64(&p.ctl->work_head);
                    if (GLS_BATCH_AA > 0 &&
                        ld_relaxed_u64(&p.ctl->chunk_top) > h + (unsigned long long)GLS_BATCH_AA) {
                        id = atomicAdd(&p.ctl->work_head, 1ull);
                    } else {
                        if (h >= p.ck_cap || ld_relaxed_u32(&p.ck_gate[h]) == 0xffffffffu) break;
                        if (atomicCAS(&p.ctl->work_head, h, h + 1ull) != h) break;
                        id = h;
                    }
                }
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
                    // wait for the claimed id to be published: poll its own ck_gate word
                    // (every waiting warp a different line); the shared completion count and
                    // error word only every 16th poll
                    unsigned ns = GLS_MINSLEEP, polls = 0;
                    unsigned long long t_start = 0, seen = ~0ull;
                    for (;;) {
                        if (id < p.ck_cap) {
                            g = ld_relaxed_u32(&p.ck_gate[id]);   // (polls stay relaxed: an acquire
                            if (g != 0xffffffffu) break;            //  invalidates the SM's L1 each time)
                        }
                        if ((++polls & 15u) == 0u || id >= p.ck_cap) {
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
                        }
                        __nanosleep(ns);
                        if (ns < GLS_MAXSLEEP) ns <<= 1;
                    }
                    if (g == 0xffffffffu) {
                        more_work = false;
                        break;
                    }
                }
                // acquire once the chunk is seen published: pairs with plan_gate's release, so
                // the gate's plan (chunk times, counts, fan-in lengths) is visible below
                g = ld_acquire_u32(&p.ck_gate[id]);
            } else {
                g = __ldcg(&p.ck_gate[id]);
            }
            const unsigned long long nch = __ldcg(&p.net_nck[p.P + g]);
            const unsigned long long e = __ldcg(&p.gate_nin[g]) / (nch ? nch : 1ull);
            // static units of at most U_MAX expected entries (a unit's outputs must fit the lane
            // scratch); a chunk that would not fit the batch's unit budget waits for the next batch
            const int need = (int)min(32ull, max(1ull, (e + U_MAX - 1) / U_MAX));
            // a big chunk travels alone (GLS_ALONE: at least this many expected entries):
            // small chunks batched with it would complete only when it does, and one of them
            // may be on the critical path
            const bool big = GLS_ALONE > 0 && e >= (unsigned long long)GLS_ALONE;
            if (nc > 0 && (units_needed + need > MAXU_STATIC || big)) {
                carry = id;
                break;
            }
            units_needed += need;
            GLS_ASSERT(nc < MAXC && id < p.ck_cap && g < (uint32_t)p.G);
            B.c_inf[nc] = (p.gate[g].flags & kGateInf) != 0;
            B.id[nc] = id;
            warp_aux(p).c_t[nc] = p.trace ? gtimer() : 0ull;
            est[nc] = e;
            total += e;
            ++nc;
            if (big) break;
        }
        if (nc > 0) {
            B.acc[A_BATCHES] += 1ull;
            B.acc[A_BEST] += total;
        }
        // ---- static units: a chunk with at least w = total/32 expected entries is cut into
        // about est/w time slices, a smaller chunk is one unit
        // (32-bit arithmetic: a batch holds at most ~16 chunks of ~M expected entries)
        const uint32_t w = (uint32_t)max((unsigned long long)W_MIN, min((total + 31) / 32, 0x3fffffffull));
        for (int j = 0; j < nc; ++j) {
            const uint32_t e = (uint32_t)min(est[j], 0x3fffffffull);
            int ns = e >= w && !B.c_inf[j] ? (int)min(32u, max(1u, (e + w / 2) / w)) : 1;
            if (!B.c_inf[j]) ns = max(ns, (int)min(32u, (e + (uint32_t)U_MAX - 1u) / (uint32_t)U_MAX));
            ns = max(1, min(ns, MAXU_STATIC - nu - (nc - 1 - j)));   // room for the later chunks
            B.c_first[j] = (uint8_t)nu;
            B.c_nsl[j] = (uint8_t)ns;
            for (int q = 0; q < ns; ++q, ++nu) {
                GLS_ASSERT(nu < MAXU_STATIC);
                B.u_chunk[nu] = (uint8_t)j;
                B.u_slice[nu] = (uint8_t)q;
                B.u_est[nu] = B.c_inf[j] ? 0u : e / (uint32_t)ns;   // (0: never split)
                B.u_next[nu] = q + 1 < ns ? (uint8_t)(nu + 1) : kEnd;
                B.u_st[nu] = 0;
                B.u_lane[nu] = 0;
            }
        }
        B.qhead = 0;
        B.round = 0;
        B.big = GLS_ALONE > 0 && nc == 1 && est[0] >= (unsigned long long)GLS_ALONE;
        B.acc[A_BAL + 0] += (unsigned long long)nu;
        B.acc[A_BLANES] += (unsigned long long)min(nu, 32);
        p.deep_wtop[warp_global_id()] = 0;          // this warp's deep scratch, reused per batch
    }
    nc = __shfl_sync(FULL, nc, 0);
    more_work = __shfl_sync(FULL, (int)more_work, 0) != 0;
    __syncwarp();
    if (nc == 0) return DATAFLOW ? more_work : false;
    const int nstatic = __shfl_sync(FULL, nu, 0);
    const long long c_asm = clock64();

    // ---- static unit boundaries, warp-parallel: quantiles of the chunk's longest fan-in
    for (int u = lane; u < nstatic; u += 32) {
        const int j = B.u_chunk[u], q = B.u_slice[u], ns = B.c_nsl[j];
        ChunkSetup s;
        uint32_t gi, cidx, nch, ref;
        unsigned long long q0, q1, nin;
        setup_chunk(p, B.id[j], s, gi, cidx, nch, &q0, &q1, &ref, &nin);
        B.u_T0[u] = q == 0 ? s.T0 : time_at(p, ref, q0 + ((q1 - q0) * (unsigned long long)q) / (unsigned long long)ns);
        if (q + 1 == ns) B.u_T1[u] = s.T1;
        if (q == 0) B.c_T0[j] = s.T0;
    }
    __syncwarp();
#if GLS_MQ_MIN > 0
    // big chunks: slices at quantiles of the MERGED input count instead (what a lane's work
    // is), found warp-cooperatively — lane l takes the candidate time t_l at the l/32
    // quantile of the longest fan-in and counts all k fan-ins' entries before it (binary
    // searches in lockstep); boundary s is the latest candidate whose merged count is at
    // most s/ns of the chunk's
    for (int j = 0; j < nc; ++j) {
        const int ns = B.c_nsl[j];
        if (ns <= 1 || B.u_est[B.c_first[j]] * (unsigned)ns < (unsigned)GLS_MQ_MIN) continue;
        ChunkSetup s;
        uint32_t gi, cidx, nch, ref;
        unsigned long long q0, q1, nin;
        setup_chunk(p, B.id[j], s, gi, cidx, nch, &q0, &q1, &ref, &nin);
        const long long t = lane == 0 ? s.T0 : time_at(p, ref, q0 + ((q1 - q0) * (unsigned long long)lane) / 32ull);
        const unsigned long long mc = count_before_all(p, s.src, s.k, t);
        const unsigned long long m1 = lane == 0 ? count_before_all(p, s.src, s.k, s.T1) : 0ull;
        const unsigned long long m0 = __shfl_sync(FULL, mc, 0), me = __shfl_sync(FULL, m1, 0);
        const int f = B.c_first[j];
        for (int q = 1; q < ns; ++q) {
            const unsigned long long target = m0 + (me - m0) * (unsigned long long)q / (unsigned long long)ns;
            const unsigned bal = __ballot_sync(FULL, mc <= target);
            const long long tq = __shfl_sync(FULL, t, 31 - __clz(bal));
            if (lane == 0) B.u_T0[f + q] = tq;
        }
    }
    __syncwarp();
#endif
    for (int u = lane; u < nstatic; u += 32)
        if (B.u_next[u] != kEnd) B.u_T1[u] = B.u_T0[u + 1];
    __syncwarp();
    const long long c_bnd = clock64();

    // ---- the sweep
    if (lane == 0) B.nun = nstatic;
    __syncwarp();
    sweep_rounds(p, nstatic);
    const long long c_run = clock64();
    // ---- fallback units (long delays, stack overflow): exact count with the per-lane ring engine
    uint32_t f_ev = 0, f_evt = 0, nfb = 0;
    for (int v = B.lane_first[lane]; v >= 0; v = B.u_lnext[v])
        if (B.u_st[v] != 0) {
            fallback_count(p, B, v, lut, f_ev, f_evt);
            ++nfb;
        }
    {
        const unsigned long long se = warp_sum64(f_ev), sv = warp_sum64(f_evt), sf = warp_sum64(nfb);
        if (sf) atomicAdd(&p.ctl->deep_chunks, lane == 0 ? sf : 0ull);
        if (lane == 0) {
            B.acc[A_EVALS] += se;
            B.acc[A_EVENTS] += sv;
            B.acc[A_BAL + 3] += sf;
        }
    }
    __syncwarp();
    // ---- per chunk: unit offsets (in time order), total and one exact segment
    for (int j = lane; j < nc; j += 32) {
        uint32_t tot = 0;
        for (int v = B.c_first[j]; v != kEnd; v = B.u_next[v]) {
            __stcg(&warp_aux(p).u_pre[v], tot);
            tot += __ldcg(&warp_aux(p).u_cnt[v]);
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
    // ---- each lane moves its units into place (independent loads, overlapped latency)
    for (int v = B.lane_first[lane]; v >= 0; v = B.u_lnext[v]) {
        const unsigned long long off = B.c_off[B.u_chunk[v]];
        const uint32_t cu = __ldcg(&warp_aux(p).u_cnt[v]);
        if (off == ~0ull || cu == 0) continue;
        uint64_t* dst = p.arena + off + __ldcg(&warp_aux(p).u_pre[v]);
        if (B.u_st[v] != 0) {
            fallback_write(p, B, v, lut, dst);
            continue;
        }
        const uint64_t* src = p.wscr + (warp_global_id() * 32u + (uint32_t)lane) * (uint32_t)LCAP + __ldcg(&warp_aux(p).u_soff[v]);
        GLS_ASSERT(off + __ldcg(&warp_aux(p).u_pre[v]) + cu <= p.arena_cap);
        GLS_ASSERT(__ldcg(&warp_aux(p).u_soff[v]) + cu <= (uint32_t)LCAP);
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
    __syncwarp();
    const long long c_out = clock64();
    unsigned long long t_maxit = 0, t_maxsu = 0;
    if (p.trace) {
        t_maxit = __reduce_max_sync(FULL, warp_aux(p).lit[lane]);
        t_maxsu = __reduce_max_sync(FULL, warp_aux(p).lsu[lane]);
    }
    // ---- complete the chunks (whole warp, one after the other)
    for (int j = 0; j < nc; ++j) {
        const unsigned long long id = B.id[j];
        ChunkResult R;
        R.gi = __ldcg(&p.ck_gate[id]);
        R.nch = __ldcg(&p.net_nck[p.P + R.gi]);
        R.s.T0 = B.c_T0[j];
        R.off = B.c_off[j];
        R.fits = R.off != ~0ull;
        R.total = B.c_total[j];
        R.vb = B.u_vb[B.c_first[j]];
        R.evals = 0;                                   // (counted per lane above)
        R.events = 0;
        if (p.trace && lane == 0) {
            const unsigned long long d = gtimer() - warp_aux(p).c_t[j];
            unsigned long long* tr = p.trace + 8ull * R.gi;
            atomicAdd(&tr[2], d);
            if (atomicMax(&tr[3], d) < d) {                 // the slowest chunk's batch (racy only across chunks)
                tr[4] = (unsigned long long)B.round;
                tr[5] = (unsigned long long)B.nun;
                tr[6] = t_maxit;
                tr[7] = t_maxsu;
            }
        }
        chunk_done<DATAFLOW>(p, id, R, B.acc);
    }
    const long long c_end = clock64();
    if (lane == 0) {
        B.acc[A_CYC + 0] += (unsigned long long)(c_asm - c_start);
        B.acc[A_CYC + 1] += (unsigned long long)(c_bnd - c_asm);
        B.acc[A_CYC + 2] += (unsigned long long)(c_run - c_bnd);
        B.acc[A_CYC + 3] += (unsigned long long)(c_out - c_run);
        B.acc[A_CYC + 4] += (unsigned long long)(c_end - c_out);
    }
    return true;
}

}  // namespace ln
}  // namespace gls
