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

constexpr int RD = 4;                  // register pending ring depth
constexpr int LCAP = 256;              // per-lane output scratch entries
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
                                         uint32_t& vb, uint32_t& evals, uint32_t& events) {
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
    const uint32_t lb = s.lut_base;
    const long long T0 = s.T0, T1 = s.T1, dur = p.duration, dmin = (long long)s.dmin;
    const uint64_t lim1 = (uint64_t)T1 << 2;           // entry time >= T1  <=>  entry >= lim1
    uint64_t rg0 = 0, rg1 = 0, rg2 = 0, rg3 = 0;       // pending ring: rg0 newest, rg[rn-1] oldest
    int rn = 0;
    uint32_t Eprev = 2, lastv = 2;
    uint32_t n_out = 0, n_ev = 0, n_evals = 0;
    vb = 2;
    int status = 0;

    auto emit = [&](uint64_t e) {
        const long long r = etime(e);
        if (r < T0) {
            vb = (uint32_t)(e & 3u);
        } else if (r < T1 && r <= dur) {
            if (DIRECT || n_out < (uint32_t)LCAP) out[n_out] = e;
            ++n_out;
        }
        lastv = (uint32_t)(e & 3u);
    };
    auto front = [&]() -> uint64_t { return rn == 1 ? rg0 : rn == 2 ? rg1 : rn == 3 ? rg2 : rg3; };
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
                const uint32_t tv = rn > 0 ? (uint32_t)(rg0 & 3u) : lastv;
                if (tv != E) {
                    if (rn == RD) {
                        status = 1;
                    } else {
                        rg3 = rg2; rg2 = rg1; rg1 = rg0;
                        rg0 = ((uint64_t)rr << 2) | E;
                        ++rn;
                    }
                }
                if (t >= T0) ++n_ev;
                Eprev = E;
            }
            xn = nx;
        }
        const long long lim = t + dmin;                // streaming finality
        while (rn > 0) {
            const uint64_t f = front();
            if (etime(f) > lim) break;
            emit(f);
            --rn;
        }
    };

    step(s.tau0, x0);                                   // the slice's halo start
    for (;;) {
        const uint64_t m = min(min(h[0], h[1]), min(h[2], h[3]));
        if (m >= lim1 || status) break;
        const long long t = etime(m);
        uint32_t nx = xn;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if ((h[i] ^ m) < 4ull) {                   // pin i changes at t
                nx = (nx & ~(3u << (2 * i))) | (norm_code((uint32_t)(h[i] & 3u)) << (2 * i));
                ++c[i].ptr;
                if (--c[i].rem == 0) {
                    const Seg g = next_segment(p, c[i].ck, c[i].ckend);
                    if (g.rem) { c[i].ptr = g.ptr; c[i].rem = g.rem; c[i].ck = g.ck; }
                }
                h[i] = c[i].rem ? *c[i].ptr : kInfEntry;
                if ((((uintptr_t)c[i].ptr) & 127u) == 0 && c[i].rem > 32)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(c[i].ptr + 32));
            }
        }
        n_evals += (t >= T0);
        step(t, nx);
    }
    while (rn > 0) {                                    // final for this slice below T1
        const uint64_t f = front();
        if (etime(f) >= T1) break;
        emit(f);
        --rn;
    }
    cnt = n_out;
    evals = n_evals;
    events = n_ev;
    if (!DIRECT && status == 0 && n_out > (uint32_t)LCAP) status = 2;
    return status;
}

// One chunk with the slice engine (whole warp).
__device__ void process_chunk_slice(const SimParams& p, unsigned long long id, const uint8_t* lut, uint32_t* s_dtab,
                                    ChunkResult& R) {
    const int lane = threadIdx.x & 31;
    uint64_t* scr = p.wscr + (size_t)warp_global_id() * kScratchPerWarp;
    uint32_t* dtab = s_dtab + threadIdx.x;              // [q * blockDim.x + tid]
    const int dstride = (int)blockDim.x;
    ChunkSetup& s = R.s;
    unsigned long long q0 = 0, q1 = 0, n_in = 0;
    uint32_t ref = 0, cidx = 0;
    setup_chunk(p, id, s, R.gi, cidx, R.nch, &q0, &q1, &ref, &n_in);
    // lanes and slice boundaries (quantiles of the longest fan-in inside the chunk)
    const unsigned long long span = q1 - q0;
    const unsigned long long lenref = __ldcg(&p.net_len[ref]);
    const double est = lenref ? (double)span * (double)n_in / (double)lenref : 0.0;
    int nl = (int)fmin(32.0, fmax(1.0, est / (double)E_MIN));
    if ((unsigned long long)nl > span) nl = (int)max(1ull, span);
    long long Tl = s.T0;
    if (lane > 0 && lane < nl) {
        const unsigned long long qi = q0 + (span * (unsigned long long)lane) / (unsigned long long)nl;
        Tl = time_at(p, ref, qi);
    }
    const long long Tn0 = __shfl_down_sync(FULL, Tl, 1);
    const long long Tn = lane + 1 < nl ? Tn0 : s.T1;
    uint32_t cnt = 0, vb = 2, ev = 0, evt = 0;
    int st = 0;
    ChunkSetup ls = s;
    ls.T0 = Tl;
    ls.T1 = Tn;
    ls.tau0 = Tl - (long long)s.dmax - 1;
    if (lane < nl) {
        // this lane's delay table (R1: output X takes the smaller delay)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint4 d = s.d[i];
            dtab[(i * 6 + 0) * dstride] = d.z;
            dtab[(i * 6 + 1) * dstride] = d.w;
            dtab[(i * 6 + 2) * dstride] = min(d.z, d.w);
            dtab[(i * 6 + 3) * dstride] = d.x;
            dtab[(i * 6 + 4) * dstride] = d.y;
            dtab[(i * 6 + 5) * dstride] = min(d.x, d.y);
        }
        st = run_slice<false>(p, ls, lut, dtab, dstride, scr + (size_t)lane * LCAP, cnt, vb, ev, evt);
        if (st == 1) {
            // pending ring overflow: exact count of the slice by the per-lane engine (deep ring if needed)
            ChunkOut r{0, 0, 0, 2, false};
            run_chunk<false, false>(p, ls, lut, nullptr, nullptr, 0, r);
            if (r.overflow) {
                const unsigned long long dcap = window_bound(p, ls);
                const unsigned long long at = deep_alloc(p, dcap);
                if (at != ~0ull) {
                    r = ChunkOut{0, 0, 0, 2, false};
                    run_chunk<false, true>(p, ls, lut, nullptr, p.deep + at, dcap, r);
                }
            }
            cnt = r.cnt;
            vb = r.vb;
            ev = r.evals;
            evt = r.events;
        }
    }
    if (lane < nl && st != 0) atomicAdd(&p.ctl->deep_chunks, 1ull);
    uint32_t pre = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t a = __shfl_up_sync(FULL, pre, o);
        if (lane >= o) pre += a;
    }
    const uint32_t total = __shfl_sync(FULL, pre, 31);
    pre -= cnt;
    const unsigned long long off = arena_alloc(p, total);
    R.fits = off != ~0ull;
    if (R.fits) {
        const unsigned clean = __ballot_sync(FULL, st == 0);
        for (int j = 0; j < nl; ++j) {                    // coalesced copy-out, lane by lane
            if (!((clean >> j) & 1u)) continue;
            const uint32_t cj = __shfl_sync(FULL, cnt, j);
            const uint32_t pj = __shfl_sync(FULL, pre, j);
            const uint64_t* src = scr + (size_t)j * LCAP;
            for (uint32_t q = lane; q < cj; q += 32) p.arena[off + pj + q] = src[q];
        }
        if (lane < nl && st == 2) {                       // scratch overflow: re-run straight into place
            uint32_t c2, v2, e2, t2;
            run_slice<true>(p, ls, lut, dtab, dstride, p.arena + off + pre, c2, v2, e2, t2);
            if (c2 != cnt) atomicOr(&p.ctl->error, kErrBug);
        } else if (lane < nl && st == 1) {                 // ring overflow: per-lane engine writes in place
            ChunkOut r2{0, 0, 0, 2, false};
            run_chunk<true, false>(p, ls, lut, p.arena + off + pre, nullptr, 0, r2);
            if (r2.overflow) {
                const unsigned long long dcap = window_bound(p, ls);
                const unsigned long long at = deep_alloc(p, dcap);
                if (at != ~0ull) {
                    r2 = ChunkOut{0, 0, 0, 2, false};
                    run_chunk<true, true>(p, ls, lut, p.arena + off + pre, p.deep + at, dcap, r2);
                }
            }
            if (r2.cnt != cnt) atomicOr(&p.ctl->error, kErrBug);
        }
    }
    R.off = off;
    R.total = total;
    R.vb = __shfl_sync(FULL, vb, 0);
    R.evals = warp_sum64(ev);
    R.events = warp_sum64(evt);
}

}  // namespace sl
}  // namespace gls
