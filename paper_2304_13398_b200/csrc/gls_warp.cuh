// gls_warp.cuh — warp-cooperative evaluation of one (gate, time-chunk) work item.
// Included by gls_kernels.cu (after the per-lane engine, which stays as the
// fallback for pathological chunks).
//
// One warp owns one chunk.  Per tile:
//   1. coalesced refills of one shared-memory ring per fan-in pin (the k rings
//      share 512 entries), Alg. 2 reading its input waveforms;
//   2. the tile = every ring entry with t <= T_lim (T_lim = the earliest
//      last-loaded time among pins with more data, so no later entry can
//      interleave), found by binary search per ring;
//   3. k-way merge by merge path straight from the rings (pairwise for k = 3,
//      4); lane l receives merged entries [l*E, (l+1)*E) as 32-bit keys
//      (t - base) << 4 | pin << 2 | v in a conflict-free [j][lane] layout and,
//      in the same loop, composes its input updates and marks distinct
//      timestamps;
//   4. a warp scan of the composed updates gives each lane its input vector;
//      each lane evaluates the LUT at its distinct timestamps and finds events
//      and their delays (only the changed pins are visited);
//   5. Eq. 1 survivors = events whose appearance time is below every later
//      event's (per-lane reverse minimum + warp suffix minimum); dedupe against
//      the previous survivor; survivors with r <= T_lim + dmin are final
//       and go to the warp's output scratch, later ones stay
//      pending across tiles.
// At the end the chunk's exact count is known: one atomic allocates its segment
// and the scratch is copied out with coalesced stores.  Results are
// bit-identical to the per-lane engine and the oracle (tests/test_gpu_parity.py).
#pragma once

namespace gls {
namespace wv {

constexpr int RING = 512;                  // ring entries shared by the k pins
constexpr int TMAX = 512;                  // entries per tile at most
constexpr int EPL = TMAX / 32;             // entries per lane at most (16)
constexpr int PMAX = 64;                   // pending schedules carried between tiles
constexpr int NSPILL = 32;                 // spilled scratch blocks per chunk
constexpr unsigned FULL = 0xffffffffu;
constexpr long long SPAN = (1ll << 28) - 1; // key time span of one tile
constexpr uint32_t RINF = 0xffffffffu;

struct WS {
    uint64_t ring[RING];                   // 4 KB  raw entries; pin i at [i*cap, (i+1)*cap)
    union {
        struct {                           // level-1 merge outputs (k = 3, 4)
            uint32_t tmpA[TMAX / 2];
            uint32_t tmpB[TMAX / 2];
        } m;
        uint32_t evr[EPL][32];             // event appearance time (relative), RINF if none
    } u;                                   // 2 KB
    uint32_t merged[EPL][32];              // 2 KB  merged keys
    uint8_t gev[EPL][32];                  // 512 B bits 0..1 evaluation
    uint64_t pend[PMAX];                   // 512 B
    unsigned long long spill_off[NSPILL];
    uint32_t spill_cnt[NSPILL];
    uint32_t dtab[4 * 6];                  // per pin: [fall, rise][out 0, 1, X] (R1)
    unsigned long long c_off[4];           // cursors (warp-uniform, written by lane 0)
    uint32_t c_rem[4], c_ck[4], c_ckend[4], whead[4], wcnt[4], more[4];
};
constexpr int kWarpsPerBlock = kThreads / 32;
constexpr size_t kSmemBytes = sizeof(WS) * kWarpsPerBlock;
constexpr int OBG = 4096;                  // per-warp output scratch entries (global memory)

__device__ __forceinline__ uint32_t expand4(uint32_t m) {  // pin bit i -> value field bits 2i, 2i+1
    return ((m & 1u) * 3u) | ((m & 2u) * 6u) | ((m & 4u) * 12u) | ((m & 8u) * 24u);
}
__device__ __forceinline__ uint32_t apply_upd(uint32_t vec, uint32_t x) {  // x = mask << 8 | vals
    return (vec & ~expand4(x >> 8)) | (x & 0xffu);
}
__device__ __forceinline__ uint32_t set_pin(uint32_t v, uint32_t key) {
    const uint32_t pin = (key >> 2) & 3u;
    return (v & ~(3u << (2 * pin))) | (norm_code(key & 3u) << (2 * pin));
}
__device__ __forceinline__ uint32_t mkkey(uint64_t e, long long tbase, uint32_t pin) {
    return ((uint32_t)(etime(e) - tbase) << 4) | (pin << 2) | (uint32_t)(e & 3u);
}

// per-lane accumulation while the final merge emits the lane's entries
struct LaneAcc {
    uint32_t upd;      // composed update of the lane's entries (mask << 8 | vals)
    uint32_t upd_ge;   // composed update up to the lane's last distinct-timestamp end
    uint32_t gemask;   // bit j: entry j ends a distinct timestamp
    uint32_t last_t;
};
__device__ __forceinline__ void acc_emit(WS& ws, LaneAcc& a, uint32_t key, int j, int lane) {
    const uint32_t t = key >> 4;
    if (j > 0 && t != a.last_t) {
        a.gemask |= 1u << (j - 1);
        a.upd_ge = a.upd;
    }
    const uint32_t pin = (key >> 2) & 3u;
    a.upd = ((a.upd | (0x100u << pin)) & ~(3u << (2 * pin))) | (norm_code(key & 3u) << (2 * pin));
    a.last_t = t;
    ws.merged[j][lane] = key;
}

// Merge path over two pins' ring prefixes (raw entries; on equal times the
// lower pin, A, comes first).  FINAL: outputs go to merged[j][lane] with the
// lane accumulation; else keys go to C[d].
template <bool FINAL>
__device__ __forceinline__ void merge_rings(WS& ws, const uint64_t* Ab, uint32_t Ah, uint32_t Am, uint32_t Ap, int na,
                                            const uint64_t* Bb, uint32_t Bh, uint32_t Bm, uint32_t Bp, int nb,
                                            long long tbase, uint32_t* C, int per, int lane, LaneAcc& acc) {
    const int n = na + nb;
    const int d0 = min(lane * per, n), d1 = min(d0 + per, n);
    int lo = max(0, d0 - nb), hi = min(d0, na);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (etime(Ab[(Ah + mid) & Am]) <= etime(Bb[(Bh + d0 - 1 - mid) & Bm])) lo = mid + 1; else hi = mid;
    }
    int ia = lo, ib = d0 - lo;
    uint64_t ha = ia < na ? Ab[(Ah + ia) & Am] : kInfEntry;
    uint64_t hb = ib < nb ? Bb[(Bh + ib) & Bm] : kInfEntry;
    for (int d = d0; d < d1; ++d) {
        const bool takeA = etime(ha) <= etime(hb);
        const uint32_t key = takeA ? mkkey(ha, tbase, Ap) : mkkey(hb, tbase, Bp);
        if (takeA) {
            ++ia;
            ha = ia < na ? Ab[(Ah + ia) & Am] : kInfEntry;
        } else {
            ++ib;
            hb = ib < nb ? Bb[(Bh + ib) & Bm] : kInfEntry;
        }
        if (FINAL) acc_emit(ws, acc, key, d - d0, lane); else C[d] = key;
    }
}
// merge path over two key arrays (keys unique, pins distinct across A and B)
__device__ __forceinline__ void merge_keys(WS& ws, const uint32_t* A, int na, const uint32_t* B, int nb, int per,
                                           int lane, LaneAcc& acc) {
    const int n = na + nb;
    const int d0 = min(lane * per, n), d1 = min(d0 + per, n);
    int lo = max(0, d0 - nb), hi = min(d0, na);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (A[mid] < B[d0 - 1 - mid]) lo = mid + 1; else hi = mid;
    }
    int ia = lo, ib = d0 - lo;
    uint32_t ha = ia < na ? A[ia] : RINF, hb = ib < nb ? B[ib] : RINF;
    for (int d = d0; d < d1; ++d) {
        const bool takeA = ha < hb;
        const uint32_t key = takeA ? ha : hb;
        if (takeA) { ++ia; ha = ia < na ? A[ia] : RINF; } else { ++ib; hb = ib < nb ? B[ib] : RINF; }
        acc_emit(ws, acc, key, d - d0, lane);
    }
}

struct Emit {   // per-chunk output state (warp-uniform)
    int out_n;
    int nspill;
    uint32_t vb;
    uint32_t last_val;
};

// move the warp's output scratch to the deep-scratch pool; false if out of room
__device__ __noinline__ bool spill(const SimParams& p, WS& ws, uint64_t* scr, Emit& em, int lane) {
    if (em.out_n == 0) return true;
    if (em.nspill >= NSPILL) return false;
    unsigned long long at = 0;
    if (lane == 0) at = deep_alloc(p, (unsigned long long)em.out_n);
    at = __shfl_sync(FULL, at, 0);
    if (at == ~0ull) return false;
    for (int q = lane; q < em.out_n; q += 32) p.deep[at + q] = scr[q];
    if (lane == 0) {
        ws.spill_off[em.nspill] = at;
        ws.spill_cnt[em.nspill] = (uint32_t)em.out_n;
    }
    __syncwarp();
    em.nspill++;
    em.out_n = 0;
    return true;
}

// coalesced refill of pin i's ring up to `cap` entries (warp-uniform control)
__device__ __forceinline__ void refill(const SimParams& p, WS& ws, int i, uint32_t cap, long long T1, int lane) {
    uint32_t wc = ws.wcnt[i], more = ws.more[i];
    if (!more || wc >= cap) return;
    unsigned long long off = ws.c_off[i];
    uint32_t rem = ws.c_rem[i], ck = ws.c_ck[i];
    const uint32_t ckend = ws.c_ckend[i], wh = ws.whead[i], m = cap - 1;
    uint64_t* rb = ws.ring + i * cap;
    while (more && wc < cap) {
        if (rem == 0) {
            if (ck + 1 < ckend) {
                ++ck;
                off = __ldcg(&p.ck_off[ck]);      // L2: never a stale L1 line (dataflow)
                rem = __ldcg(&p.ck_cnt[ck]);
                continue;
            }
            more = 0;
            break;
        }
        const uint32_t take = min(cap - wc, rem);
#pragma unroll 4
        for (uint32_t q = lane; q < take; q += 32) rb[(wh + wc + q) & m] = p.arena[off + q];
        off += take;
        rem -= take;
        wc += take;
        __syncwarp();
        if (etime(rb[(wh + wc - 1) & m]) >= T1) more = 0;   // later entries cannot matter
    }
    __syncwarp();
    if (lane == 0) {
        ws.c_off[i] = off;
        ws.c_rem[i] = rem;
        ws.c_ck[i] = ck;
        ws.wcnt[i] = wc;
        ws.more[i] = more;
    }
    __syncwarp();
}

// exclusive "last valid" scan of 9-bit tagged values (bit 8 = valid)
__device__ __forceinline__ uint32_t excl_last_valid(uint32_t y, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t z = __shfl_up_sync(FULL, y, o);
        if (lane >= o && !(y & 0x100u)) y = z;
    }
    const uint32_t e = __shfl_up_sync(FULL, y, 1);
    return lane == 0 ? 0u : e;
}

// Returns false when the chunk must be redone by the per-lane engine
// (pending list or spill list overflow).
__device__ __noinline__ bool warp_chunk(const SimParams& p, WS& ws, uint64_t* scr, const ChunkSetup& s,
                                        const uint8_t* lut, unsigned long long& out_off, uint32_t& out_cnt,
                                        uint32_t& out_vb, unsigned long long& evals, unsigned long long& events,
                                        bool& fits) {
    const int lane = threadIdx.x & 31;
    const int k = (int)s.k;
    const uint32_t cap = k == 1 ? RING : (k == 2 ? RING / 2 : RING / 4);
    const uint32_t lb = s.lut_base;
    const long long T0 = s.T0, T1 = s.T1, dur = p.duration, dmin = (long long)s.dmin;

    // delay tables (reading R1: output X takes the smaller of the two)
    if (lane < 4) {
        const uint4 d = lane == 0 ? s.d[0] : lane == 1 ? s.d[1] : lane == 2 ? s.d[2] : s.d[3];
        uint32_t* t = ws.dtab + lane * 6;
        t[3] = d.x;               // RISE -> 0
        t[4] = d.y;               // RISE -> 1
        t[5] = min(d.x, d.y);
        t[0] = d.z;               // FALL -> 0
        t[1] = d.w;               // FALL -> 1
        t[2] = min(d.z, d.w);
    }
    // cursors: lane i locates pin i at tau0 (first transition > tau0, value at tau0)
    uint32_t l_init = 2;
    if (lane < k) {
        const uint32_t src = lane == 0 ? s.src[0] : lane == 1 ? s.src[1] : lane == 2 ? s.src[2] : s.src[3];
        Cursor c;
        locate(p, src, s.tau0, c, l_init);
        ws.c_off[lane] = (unsigned long long)(c.ptr - p.arena);
        ws.c_rem[lane] = (uint32_t)(c.end - c.ptr);
        ws.c_ck[lane] = c.ck;
        ws.c_ckend[lane] = c.ck_end;
        ws.whead[lane] = 0;
        ws.wcnt[lane] = 0;
        ws.more[lane] = c.end > c.ptr ? 1u : 0u;
    }
    uint32_t x0 = 0;
    for (int i = 0; i < k; ++i) x0 |= norm_code(__shfl_sync(FULL, l_init, i)) << (2 * i);
    __syncwarp();

    Emit em{0, 0, 2u, 2u};
    int np = 0;
    // the halo start: inputs take their values at tau0 at once
    uint32_t vec_carry = x0;
    {
        const uint32_t E0 = lut[lb + x0];
        if (E0 != 2u) {
            uint32_t del = RINF;
            for (int i = 0; i < k; ++i) {
                const uint32_t f = (x0 >> (2 * i)) & 3u;
                if (f != 2u) del = min(del, ws.dtab[i * 6 + (f == 1u ? 3 : 0) + E0]);
            }
            if (lane == 0) ws.pend[0] = ((uint64_t)(s.tau0 + (long long)del) << 2) | E0;
            np = 1;
        }
    }
    __syncwarp();
    unsigned long long n_evals = 0, n_events = 0;

    for (;;) {
        // ---- 1. refill rings (coalesced)
        for (int i = 0; i < k; ++i) refill(p, ws, i, cap, T1, lane);
        // ---- 2. tile bounds
        long long tbase = LLONG_MAX, tsafe = LLONG_MAX;
        for (int i = 0; i < k; ++i) {
            const uint32_t wc = ws.wcnt[i], wh = ws.whead[i];
            const uint64_t* rb = ws.ring + i * cap;
            if (wc > 0) {
                tbase = min(tbase, etime(rb[wh]));
                if (ws.more[i]) tsafe = min(tsafe, etime(rb[(wh + wc - 1) & (cap - 1)]));
            }
        }
        if (tbase >= T1) break;                               // nothing left before T1
        const long long tlim = min(min(tsafe, T1 - 1), tbase + SPAN);
        int mi[4] = {0, 0, 0, 0};
        int nt = 0;
        for (int i = 0; i < k; ++i) {                         // entries with t <= tlim
            const uint64_t* rb = ws.ring + i * cap;
            const uint32_t wh = ws.whead[i];
            int lo = 0, hi = (int)ws.wcnt[i];
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (etime(rb[(wh + mid) & (cap - 1)]) <= tlim) lo = mid + 1; else hi = mid;
            }
            mi[i] = lo;
            nt += lo;
        }
        // ---- 3. merge; lane l gets merged entries [l*Ep, l*Ep + nv)
        const int Ep = (nt + 31) >> 5;
        const int nv = max(0, min(Ep, nt - lane * Ep));
        LaneAcc acc{0u, 0u, 0u, 0u};
        if (k == 1) {
            const uint64_t* rb = ws.ring;
            const uint32_t wh = ws.whead[0];
            for (int j = 0; j < nv; ++j)
                acc_emit(ws, acc, mkkey(rb[(wh + lane * Ep + j) & (cap - 1)], tbase, 0u), j, lane);
        } else if (k == 2) {
            merge_rings<true>(ws, ws.ring, ws.whead[0], cap - 1, 0u, mi[0], ws.ring + cap, ws.whead[1], cap - 1, 1u,
                              mi[1], tbase, nullptr, Ep, lane, acc);
        } else {
            const int n01 = mi[0] + mi[1];
            merge_rings<false>(ws, ws.ring, ws.whead[0], cap - 1, 0u, mi[0], ws.ring + cap, ws.whead[1], cap - 1, 1u,
                               mi[1], tbase, ws.u.m.tmpA, (n01 + 31) >> 5, lane, acc);
            int n23;
            if (k == 3) {
                n23 = mi[2];
                const uint64_t* rb = ws.ring + 2 * cap;
                const uint32_t wh = ws.whead[2];
                for (int q = lane; q < n23; q += 32) ws.u.m.tmpB[q] = mkkey(rb[(wh + q) & (cap - 1)], tbase, 2u);
            } else {
                n23 = mi[2] + mi[3];
                merge_rings<false>(ws, ws.ring + 2 * cap, ws.whead[2], cap - 1, 2u, mi[2], ws.ring + 3 * cap,
                                   ws.whead[3], cap - 1, 3u, mi[3], tbase, ws.u.m.tmpB, (n23 + 31) >> 5, lane, acc);
            }
            __syncwarp();
            merge_keys(ws, ws.u.m.tmpA, n01, ws.u.m.tmpB, n23, Ep, lane, acc);
        }
        __syncwarp();
        // close the lane's last timestamp group against the next lane's first entry
        {
            const uint32_t tn = (lane < 31 && (lane + 1) * Ep < nt) ? (ws.merged[0][lane + 1] >> 4) : RINF;
            if (nv > 0 && tn != acc.last_t) {
                acc.gemask |= 1u << (nv - 1);
                acc.upd_ge = acc.upd;
            }
        }
        // ---- 4. input vectors: warp scan of the composed updates
        uint32_t x = acc.upd;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x = ((y | x) & 0xf00u) | ((y & ~expand4(x >> 8)) & 0xffu) | (x & 0xffu);
        }
        const uint32_t xe0 = __shfl_up_sync(FULL, x, 1);
        const uint32_t xe = lane == 0 ? 0u : xe0;
        const uint32_t xtot = __shfl_sync(FULL, x, 31);
        const uint32_t vstart = apply_upd(vec_carry, xe);
        // vector at the previous distinct timestamp before my first group end
        uint32_t vprev;
        {
            const uint32_t tagged = acc.gemask ? (0x100u | apply_upd(vstart, acc.upd_ge)) : 0u;
            const unsigned lanes_with = __ballot_sync(FULL, nv > 0);
            const unsigned lanes_ge = __ballot_sync(FULL, acc.gemask != 0u);
            const unsigned need = lanes_with & ~(1u << (31 - __clz(lanes_with | 1u)));
            uint32_t t;
            if ((need & ~lanes_ge) == 0u) {
                const uint32_t u = __shfl_up_sync(FULL, tagged, 1);
                t = lane == 0 ? 0u : u;
            } else {
                t = excl_last_valid(tagged, lane);
            }
            vprev = (t & 0x100u) ? (t & 0xffu) : vec_carry;
        }
        // ---- 5. evaluations and events (Alg. 2; delays P:210)
        const uint32_t thr = T0 <= tbase ? 0u : (uint32_t)min(T0 - tbase, (long long)(1 << 28));
        uint32_t Eprev = lut[lb + vprev];
        uint32_t v = vstart, lmin = RINF, cnt_ge = 0, cnt_ev = 0;
        for (int j = 0; j < nv; ++j) {
            const uint32_t key = ws.merged[j][lane];
            v = set_pin(v, key);
            uint32_t r = RINF, g = 0;
            if ((acc.gemask >> j) & 1u) {
                const uint32_t tj = key >> 4;
                const uint32_t E = lut[lb + v];
                cnt_ge += tj >= thr;
                g = E;
                if (E != Eprev) {
                    uint32_t del = RINF;
                    const uint32_t d = v ^ vprev;
                    for (uint32_t cm = (d | (d >> 1)) & 0x55u; cm; cm &= cm - 1) {
                        const int b = __ffs(cm) - 1;        // 2 * pin
                        const uint32_t fo = (vprev >> b) & 3u, fn = (v >> b) & 3u;
                        del = min(del, ws.dtab[(b >> 1) * 6 + (rank_code(fn) > rank_code(fo) ? 3 : 0) + E]);
                    }
                    r = tj + del;
                    lmin = min(lmin, r);
                    cnt_ev += tj >= thr;
                }
                vprev = v;
                Eprev = E;
            }
            ws.u.evr[j][lane] = r;
            ws.gev[j][lane] = (uint8_t)g;
        }
        n_evals += cnt_ge;
        n_events += cnt_ev;
        // ---- 6. Eq. 1 survivors: r below every later event's r
        uint32_t sm = lmin;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t z = __shfl_down_sync(FULL, sm, o);
            if (lane + o < 32) sm = min(sm, z);
        }
        const uint32_t after0 = __shfl_down_sync(FULL, sm, 1);
        uint32_t run = lane == 31 ? RINF : after0;
        const uint32_t tile_min = __shfl_sync(FULL, sm, 0);
        uint32_t survmask = 0, lsv = 0;
        for (int j = nv - 1; j >= 0; --j) {
            const uint32_t r = ws.u.evr[j][lane];
            if (r < run) {                                   // RINF never passes
                if (!survmask) lsv = ws.gev[j][lane] & 3u;
                survmask |= 1u << j;
                run = r;
            }
        }
        const long long lim_abs = tlim + dmin;
        const long long tmin_abs = tile_min == RINF ? LLONG_MAX : tbase + (long long)tile_min;
        // pending schedules from earlier tiles (increasing r): a prefix survives
        const uint64_t pa = lane < np ? ws.pend[lane] : 0ull;
        const uint64_t pb = lane + 32 < np ? ws.pend[lane + 32] : 0ull;
        const bool sa = lane < np && etime(pa) < tmin_abs;
        const bool sb = lane + 32 < np && etime(pb) < tmin_abs;
        const bool fa = sa && etime(pa) <= lim_abs;
        const bool fb = sb && etime(pb) <= lim_abs;
        const int n_surv = __popc(__ballot_sync(FULL, sa)) + __popc(__ballot_sync(FULL, sb));
        const int n_fin = __popc(__ballot_sync(FULL, fa)) + __popc(__ballot_sync(FULL, fb));
        const bool oa = fa && etime(pa) >= T0 && etime(pa) < T1 && etime(pa) <= dur;
        const bool ob = fb && etime(pb) >= T0 && etime(pb) < T1 && etime(pb) <= dur;
        const uint32_t boa = __ballot_sync(FULL, oa), bob = __ballot_sync(FULL, ob);
        const int n_oout = __popc(boa) + __popc(bob);
        const uint32_t bva = __ballot_sync(FULL, fa && etime(pa) < T0);
        const uint32_t bvb = __ballot_sync(FULL, fb && etime(pb) < T0);
        uint32_t pred_init = em.last_val;
        if (n_surv > 0) pred_init = (uint32_t)(ws.pend[n_surv - 1] & 3u);
        if (bva | bvb) em.vb = (uint32_t)(ws.pend[bvb ? 32 + 31 - __clz(bvb) : 31 - __clz(bva)] & 3u);
        if (n_fin > 0) em.last_val = (uint32_t)(ws.pend[n_fin - 1] & 3u);
        // ---- 7. dedupe, final / pending, outputs
        uint32_t prevv;
        {
            const uint32_t t = excl_last_valid(survmask ? (0x100u | lsv) : 0u, lane);
            prevv = (t & 0x100u) ? (t & 3u) : pred_init;
        }
        const uint64_t lim_rel64 = (uint64_t)(tlim - tbase) + (uint64_t)dmin;
        const uint32_t lim_rel = lim_rel64 >= RINF ? RINF - 1 : (uint32_t)lim_rel64;
        uint32_t pendmask = 0, outmask = 0;
        int last_fin_j = -1, last_vb_j = -1;
        for (uint32_t m = survmask; m; m &= m - 1) {
            const int j = __ffs(m) - 1;
            const uint32_t E = ws.gev[j][lane] & 3u;
            if (E != prevv) {
                const uint32_t r = ws.u.evr[j][lane];
                if (r <= lim_rel) {
                    last_fin_j = j;
                    const long long ra = tbase + (long long)r;
                    if (ra < T0) last_vb_j = j;
                    else if (ra < T1 && ra <= dur) outmask |= 1u << j;
                } else {
                    pendmask |= 1u << j;
                }
            }
            prevv = E;
        }
        const int my_out = __popc(outmask), my_pend = __popc(pendmask);
        uint32_t pre = ((uint32_t)my_pend << 16) | (uint32_t)my_out;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t a = __shfl_up_sync(FULL, pre, o);
            if (lane >= o) pre += a;
        }
        const uint32_t pre_tot = __shfl_sync(FULL, pre, 31);
        pre -= ((uint32_t)my_pend << 16) | (uint32_t)my_out;
        const int tot_out = (int)(pre_tot & 0xffffu), tot_pend = (int)(pre_tot >> 16);
        const int keep_old = n_surv - n_fin;
        if (keep_old + tot_pend > PMAX) return false;           // pending overflow -> per-lane engine
        if (em.out_n + n_oout + tot_out > OBG) {
            if (!spill(p, ws, scr, em, lane)) return false;
        }
        // outputs: old finals, then tile finals, in order
        if (oa) scr[em.out_n + __popc(boa & ((1u << lane) - 1u))] = pa;
        if (ob) scr[em.out_n + __popc(boa) + __popc(bob & ((1u << lane) - 1u))] = pb;
        {
            int q = em.out_n + n_oout + (int)(pre & 0xffffu);
            for (uint32_t m = outmask; m; m &= m - 1) {
                const int j = __ffs(m) - 1;
                const long long ra = tbase + (long long)ws.u.evr[j][lane];
                scr[q++] = ((uint64_t)ra << 2) | (ws.gev[j][lane] & 3u);
            }
        }
        {   // value before T0 and last final value from the tile
            const unsigned bl = __ballot_sync(FULL, last_vb_j >= 0);
            const uint32_t vvb = last_vb_j >= 0 ? ws.gev[last_vb_j][lane] & 3u : 0u;
            const uint32_t wvb = __shfl_sync(FULL, vvb, bl ? 31 - __clz(bl) : 0);
            if (bl) em.vb = wvb;
            const unsigned bf = __ballot_sync(FULL, last_fin_j >= 0);
            const uint32_t vlf = last_fin_j >= 0 ? ws.gev[last_fin_j][lane] & 3u : 0u;
            const uint32_t wlf = __shfl_sync(FULL, vlf, bf ? 31 - __clz(bf) : 0);
            if (bf) em.last_val = wlf;
        }
        __syncwarp();
        // new pending list: surviving non-final old entries, then tile pendings
        if (sa && !fa) ws.pend[lane - n_fin] = pa;
        if (sb && !fb) ws.pend[lane + 32 - n_fin] = pb;
        {
            int q = keep_old + (int)(pre >> 16);
            for (uint32_t m = pendmask; m; m &= m - 1) {
                const int j = __ffs(m) - 1;
                ws.pend[q++] = ((uint64_t)(tbase + (long long)ws.u.evr[j][lane]) << 2) | (ws.gev[j][lane] & 3u);
            }
        }
        np = keep_old + tot_pend;
        em.out_n += n_oout + tot_out;
        // consume the tile
        if (lane < k) {
            const int m = lane == 0 ? mi[0] : lane == 1 ? mi[1] : lane == 2 ? mi[2] : mi[3];
            ws.whead[lane] = (ws.whead[lane] + (uint32_t)m) & (cap - 1);
            ws.wcnt[lane] -= (uint32_t)m;
        }
        __syncwarp();
        vec_carry = apply_upd(vec_carry, xtot);
        if (tlim >= T1 - 1) break;
    }
    // everything still pending that appears before T1 is final for this chunk
    {
        const uint64_t pa = lane < np ? ws.pend[lane] : 0ull;
        const uint64_t pb = lane + 32 < np ? ws.pend[lane + 32] : 0ull;
        const bool oa = lane < np && etime(pa) >= T0 && etime(pa) < T1 && etime(pa) <= dur;
        const bool ob = lane + 32 < np && etime(pb) >= T0 && etime(pb) < T1 && etime(pb) <= dur;
        const uint32_t boa = __ballot_sync(FULL, oa), bob = __ballot_sync(FULL, ob);
        const int n = __popc(boa) + __popc(bob);
        if (em.out_n + n > OBG) {
            if (!spill(p, ws, scr, em, lane)) return false;
        }
        if (oa) scr[em.out_n + __popc(boa & ((1u << lane) - 1u))] = pa;
        if (ob) scr[em.out_n + __popc(boa) + __popc(bob & ((1u << lane) - 1u))] = pb;
        const uint32_t bva = __ballot_sync(FULL, lane < np && etime(pa) < T0);
        const uint32_t bvb = __ballot_sync(FULL, lane + 32 < np && etime(pb) < T0);
        if (bva | bvb) em.vb = (uint32_t)(ws.pend[bvb ? 32 + 31 - __clz(bvb) : 31 - __clz(bva)] & 3u);
        em.out_n += n;
        __syncwarp();
    }
    // exact allocation of the chunk's segment and coalesced copy-out
    uint32_t total = (uint32_t)em.out_n;
    for (int q = 0; q < em.nspill; ++q) total += ws.spill_cnt[q];
    const unsigned long long at = arena_alloc(p, total);
    fits = at != ~0ull;
    if (fits) {
        unsigned long long o = at;
        for (int q = 0; q < em.nspill; ++q) {
            const unsigned long long so = ws.spill_off[q];
            const uint32_t sc = ws.spill_cnt[q];
            for (uint32_t e = lane; e < sc; e += 32) p.arena[o + e] = p.deep[so + e];
            o += sc;
        }
        for (int e = lane; e < em.out_n; e += 32) p.arena[o + e] = scr[e];
    }
    __syncwarp();
    out_off = at;
    out_cnt = total;
    out_vb = em.vb;
    evals = n_evals;
    events = n_events;
    return true;
}

}  // namespace wv
}  // namespace gls
