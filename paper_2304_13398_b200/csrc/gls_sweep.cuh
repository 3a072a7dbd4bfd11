// gls_sweep.cuh — the lean per-lane sweep of engine 0 (run_slice32), included by
// gls_slice.cuh.  Same arithmetic as run_slice (Algorithm 2, with the
// Eq. 1 filter P:240-248 and streaming finality), restructured for
// issue efficiency:
//   * times relative to a per-slice base B in 32 bits: an entry (t << 2) | v
//     with B <= t < B + 2^30 is held as ((t - B) << 2) | v, later entries as
//     kRelInf; when the sweep reaches B + 2^29 before the slice end, the
//     pending schedules that are final are emitted and B moves forward
//     ("rebase"), so any duration works;
//   * one fan-in ENTRY per iteration (the pin holding the smallest head), its
//     cursor in shared memory indexed by the pin (no 4-way predicated advance);
//     a timestamp is evaluated once its last entry is applied;
//   * a one-entry lookahead per pin, in registers: the load of a pin's next entry
//     is issued (predicated, straight into that pin's register) when its current
//     one becomes the head, so it has a whole pin period to land.
// Used when every delay of the gate is < 2^16 (u16 delay table in shared memory;
// rr = t + delay stays below 2^32 in entry form); otherwise run_slice (64-bit) runs.
#pragma once

namespace gls {
namespace sl {

constexpr uint32_t kRelInf = 0xffffffffu;
constexpr uint32_t kRebaseQ = 0x80000000u;       // entry form of t - B = 2^29
constexpr uint32_t kFastDelay = 1u << 16;        // gates with dmax below this use the 32-bit sweep (u16 delay table)


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

// per-thread cursor columns in shared memory, [pin * kThreads + tid], at fixed
// offsets from one 32-bit shared address
struct PinSm {
    uint32_t b;
    __device__ __forceinline__ uint32_t ptr(int ci) const { return b + (uint32_t)ci * 8u; }          // head entry (u64 address)
    __device__ __forceinline__ uint32_t rem(int ci) const { return b + 4u * kThreads * 8u + (uint32_t)ci * 4u; }   // entries from the head on
    __device__ __forceinline__ uint32_t ck(int ci) const { return b + 4u * kThreads * 12u + (uint32_t)ci * 4u; }   // chunk of the segment
    __device__ __forceinline__ uint32_t hn(int ci) const { return b + 4u * kThreads * 16u + (uint32_t)ci * 8u; }   // lookahead entry
};
constexpr size_t kPinSmBytes = (size_t)4 * kThreads * (8 + 4 + 4 + 8);

// global load of one transition entry (the cursor pointers live in shared memory, so the
// compiler cannot infer the state space of their targets)
__device__ __forceinline__ uint64_t ldg_entry(const uint64_t* a) {
    uint64_t v;
    asm("ld.global.u64 %0, [%1];" : "=l"(v) : "l"(a));
    return v;
}

__device__ __forceinline__ uint32_t to_rel(uint64_t e, uint64_t b4) {
    const uint64_t d = e - b4;
    return (d >> 32) ? kRelInf : (uint32_t)d;
}

// Returns 0, or 1 on ring overflow, 2 on scratch overflow (as run_slice).
template <bool DIRECT>
__device__ __noinline__ int run_slice32(const SimParams& p, const ChunkSetup& s, uint32_t lut,
                                        uint32_t dtab, PinSm cs, uint64_t* out,
                                        uint32_t cap, uint32_t* res /* cnt, vb, evals, events, iters */,
                                        long long* c_loc) {
    const long long c_l0 = clock64();
    const int tid = threadIdx.x;
    uint64_t b4 = (uint64_t)s.tau0 << 2;                // the base B in entry form (B = (int64)b4 >> 2)
    uint32_t xr0 = 0, xn = 0;                           // raw values at tau0; normalised "previous" (all X)
    uint32_t h0 = kRelInf, h1 = kRelInf, h2 = kRelInf, h3 = kRelInf;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if ((uint32_t)i < s.k) {
            Cursor cc;
            uint32_t init;
            locate(p, s.src[i], s.tau0, cc, init);
            const uint32_t rem = (uint32_t)(cc.end - cc.ptr);
            const int ci = i * kThreads + tid;
            sts64(cs.ptr(ci), (uint64_t)cc.ptr);
            sts32(cs.rem(ci), rem);
            sts32(cs.ck(ci), cc.ck);
            const uint64_t hn = rem > 1 ? cc.ptr[1] : kInfEntry;
            const uint32_t h = rem ? to_rel(*cc.ptr, b4) : kRelInf;
            sts64(cs.hn(ci), hn);
            if (i == 0) h0 = h;
            if (i == 1) h1 = h;
            if (i == 2) h2 = h;
            if (i == 3) h3 = h;
            xn |= 2u << (2 * i);                        // inputs start at X
            xr0 |= init << (2 * i);                     // raw values in effect at tau0
        }
    }
    *c_loc += clock64() - c_l0;

    const uint32_t lb = s.lut_base;
    const uint32_t dminq = s.dmin << 2;
    const long long T1e = min(s.T1, p.duration + 1);    // outputs in [T0, T1) and <= duration (R7)
    // per-base thresholds (entry form, relative to B)
    uint32_t t0q, t1q, lim;
    bool more;
    auto thresholds = [&]() {
        const long long B = (long long)b4 >> 2;
        const long long a0 = s.T0 - B, a1 = T1e - B, a2 = s.T1 - B;
        t0q = a0 <= 0 ? 0u : (uint32_t)(a0 << 2);                       // r >= T0  <=>  e >= t0q
        t1q = a1 < (1ll << 30) ? (uint32_t)(a1 << 2) : kRelInf;         // r < T1e  <=>  e < t1q
        more = a2 > (1ll << 29);
        lim = more ? kRebaseQ : (uint32_t)(a2 << 2);                    // head >= lim: stop
    };
    thresholds();

    uint32_t rg0 = 0, rg1 = 0, rg2 = 0, rg3 = 0;        // pending ring: rg0 newest
    int rn = 0;
    uint32_t ftq = kRelInf;                             // oldest pending entry (none: inf)
    uint32_t Eprev = 2, lastv = 2, vb = 2;
    uint32_t n_out = 0, n_ev = 0, n_evals = 0;
    int status = 0;

    auto emit = [&](uint32_t e) {                       // a final schedule (predicated)
        const bool before = e < t0q;
        vb = before ? (e & 3u) : vb;
        const bool w = !before && e < t1q;
        if (w && (DIRECT || n_out < cap)) out[n_out] = (uint64_t)e + b4;
        n_out += w ? 1u : 0u;
        lastv = e & 3u;
    };
    auto front = [&]() -> uint32_t { return rn == 1 ? rg0 : rn == 2 ? rg1 : rn == 3 ? rg2 : rg3; };
    auto drain = [&](uint32_t limq) {                   // emit pending entries <= limq, oldest first
        while (ftq <= limq) {
            emit(ftq);
            --rn;
            ftq = rn > 0 ? front() : kRelInf;
        }
    };
    // one distinct timestamp (tq = (t << 2) | 3) with raw input vector nr
    auto step = [&](uint32_t tq, uint32_t nr) {
        const uint32_t nn = nr ^ ((nr >> 1) & nr & 0x55u);   // Z -> X
        if (nn != xn) {
            const uint32_t E = lds8(lut + lb + nn);          // calculateSignals
            if (E != Eprev) {                                // "o_k.v is changed" (R4a)
                const uint32_t d = nn ^ xn;
                uint32_t cm = (d | (d >> 1)) & 0x55u;        // changed pins (R3)
                uint32_t del = 0xffffffffu;
                do {
                    const int b = __ffs(cm) - 1;
                    // rise iff rank(new) > rank(old), rank 0 < X < 1 on normalised codes (R2):
                    // (old, new) in {(0,1), (0,X), (X,1)} = bits 1, 2, 9 of (old << 2 | new)
                    const uint32_t rise = (0x206u >> ((((xn >> b) & 3u) << 2) | ((nn >> b) & 3u))) & 1u;
                    del = min(del, lds16(dtab + (uint32_t)((b >> 1) * 6 + (int)rise * 3 + (int)E) * (kThreads * 2)));   // min rule
                    cm &= cm - 1;
                } while (cm);
                const uint32_t rq = ((tq >> 2) + del) << 2;  // appearance time, entry form
                // addSignalChange with Eq. 1: deny pending schedules at >= rr
                while (rn > 0 && rg0 >= rq) {
                    rg0 = rg1; rg1 = rg2; rg2 = rg3;
                    --rn;
                }
                if (rn == 0) ftq = kRelInf;
                const uint32_t tv = rn > 0 ? (rg0 & 3u) : lastv;
                if (tv != E) {
                    if (rn == RD) {
                        status = 1;
                        lim = 0;                             // stop at the next iteration
                        more = false;
                    } else {
                        rg3 = rg2; rg2 = rg1; rg1 = rg0;
                        rg0 = rq | E;
                        if (rn == 0) ftq = rg0;
                        ++rn;
                    }
                }
                n_ev += tq >= t0q;
                Eprev = E;
                // streaming finality, applied at events only: an entry with
                // r <= t + dmin is final at t, and no event between two events can deny or
                // reorder anything, so draining at the next event (or at the end) emits the
                // same list in the same order
                drain(tq + dminq);
            }
            xn = nn;
        }
    };

    int lastpin = -1;                                        // pin of the newest cp.async request
    step(3u, xr0);                                           // the slice's halo start (t = tau0)
    uint32_t nr = xr0;
    uint32_t m = min(min(h0, h1), min(h2, h3));
    for (;;) {
        if (m >= lim) {
            if (!more) break;
            // rebase: the true next head (heads beyond the window are saturated)
            uint64_t raw = kInfEntry;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int ci = i * kThreads + tid;
                if ((uint32_t)i < s.k && lds32(cs.rem(ci))) raw = min(raw, ldg_entry((const uint64_t*)lds64(cs.ptr(ci))));
            }
            const long long tmin = raw == kInfEntry ? LLONG_MAX : etime(raw);
            if (tmin >= s.T1) break;
            const long long dB = tmin - ((long long)b4 >> 2);   // >= 2^29; pending entries < tmin are final
            if (dB >= (1ll << 30)) {
                drain(kRelInf - 1u);                         // every pending entry is < B + 2^30 <= tmin
            } else {
                drain(((uint32_t)dB << 2) - 1u);
                const uint32_t sh = (uint32_t)dB << 2;       // every live entry is >= tmin
                rg0 -= sh; rg1 -= sh; rg2 -= sh; rg3 -= sh;
                if (rn > 0) ftq -= sh;
            }
            b4 = (uint64_t)tmin << 2;
            thresholds();
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int ci = i * kThreads + tid;
                const uint32_t h = (uint32_t)i < s.k && lds32(cs.rem(ci)) ? to_rel(ldg_entry((const uint64_t*)lds64(cs.ptr(ci))), b4) : kRelInf;
                if (i == 0) h0 = h;
                if (i == 1) h1 = h;
                if (i == 2) h2 = h;
                if (i == 3) h3 = h;
            }
            m = min(min(h0, h1), min(h2, h3));
            continue;
        }
        const int b = h0 == m ? 0 : h1 == m ? 1 : h2 == m ? 2 : 3;
        nr = (nr & ~(3u << (2 * b))) | ((m & 3u) << (2 * b));
        // advance pin b
        const int ci = b * kThreads + tid;
        const uint64_t* ptr = (const uint64_t*)lds64(cs.ptr(ci)) + 1;
        uint32_t rem = lds32(cs.rem(ci)) - 1u;
        // the pin's lookahead entry (requested when the current head became the head)
        cp_wait_pin(b, lastpin);                             // 0 if requested in the previous iteration, else 1
        uint64_t hn = lds64(cs.hn(ci));
        uint32_t nh;
        if (rem == 0) {                                      // segment end: next non-empty segment
            const uint32_t src = s.src[b];
            const Seg g = next_segment(p, lds32(cs.ck(ci)), __ldcg(&p.net_ck[src]) + __ldcg(&p.net_nck[src]));
            if (g.rem) {
                ptr = g.ptr;
                rem = g.rem;
                sts32(cs.ck(ci), g.ck);
                hn = ldg_entry(ptr);
            } else {
                hn = kInfEntry;
            }
        }
        nh = rem ? to_rel(hn, b4) : kRelInf;
        // request the pin's next entry; nothing waits for it until this pin is advanced again
        cp_async8_if(rem > 1, cs.hn(ci), ptr + 1);
        lastpin = rem > 1 ? b : lastpin;
        sts64(cs.ptr(ci), (uint64_t)ptr);
        sts32(cs.rem(ci), rem);
        h0 = b == 0 ? nh : h0;
        h1 = b == 1 ? nh : h1;
        h2 = b == 2 ? nh : h2;
        h3 = b == 3 ? nh : h3;
        const uint32_t tq = m | 3u;
        m = min(min(h0, h1), min(h2, h3));
        if ((m | 3u) == tq) continue;                        // more entries at this timestamp
        n_evals += tq >= t0q;
        step(tq, nr);
    }
    {                                                        // final for this slice below T1
        const long long a2 = s.T1 - ((long long)b4 >> 2);
        drain(a2 < (1ll << 30) ? (uint32_t)(a2 << 2) - 1u : kRelInf - 1u);
    }
    cp_wait<0>();                                            // no copy may land in the next slice's cursors
    res[0] = n_out;
    res[1] = vb;
    res[2] = n_evals;
    res[3] = n_ev;
    res[4] = n_evals;
    if (!DIRECT && status == 0 && n_out > cap) status = 2;
    return status;
}

}  // namespace sl
}  // namespace gls
