// gls_warp.cuh — warp-cooperative evaluation of one (gate, time-chunk) work item.
// Included by gls_kernels.cu (after the per-lane engine, which stays as the
// fallback for pathological chunks).
//
// One warp owns one chunk.  Per tile:
//   1. coalesced refills of a 128-entry shared-memory window per fan-in pin
//      (Alg. 2 reads each input waveform);
//   2. the tile = every window entry with t <= T_lim (T_lim = the earliest
//      last-loaded time of a pin that has more data, so no later entry can
//      interleave); entries become 32-bit keys (t - base) << 4 | pin << 2 | v;
//   3. k-way merge by merge path (pairwise for k = 3, 4); lane l receives the
//      merged entries [l*E, (l+1)*E) in a conflict-free [j][lane] layout;
//   4. each lane sweeps its entries: input vector (warp scan of composed
//      updates), distinct timestamps, LUT evaluation, events and delays;
//   5. Eq. 1 survivors = events whose appearance time is below every later
//      event's (per-lane reverse minimum + warp suffix minimum); dedupe against
//      the previous survivor; survivors with r <= T_lim + dmin are final
//       and go to the per-warp output buffer, later ones stay
//      pending across tiles.
// At the end the chunk's exact count is known: one atomic allocates its segment
// and the buffer is copied out with coalesced stores.  Results are bit-identical
// to the per-lane engine and the oracle (tests/test_gpu_parity.py).
#pragma once

namespace gls {
namespace wv {

constexpr int WIN = 128;                   // window entries per pin (ring, power of 2)
constexpr int TMAX = 4 * WIN;              // entries per tile at most
constexpr int EPL = TMAX / 32;             // entries per lane at most (16)
constexpr int PMAX = 64;                   // pending schedules carried between tiles
constexpr int OB = 1024;                   // output buffer entries per warp (>= PMAX + TMAX)
constexpr int NSPILL = 32;                 // spilled output blocks per chunk
constexpr unsigned FULL = 0xffffffffu;
constexpr long long SPAN = (1ll << 28) - 1; // key time span of one tile
constexpr uint32_t RINF = 0xffffffffu;

struct WS {
    uint64_t win[4][WIN];                  // 4 KB  raw entries, ring per pin
    union {
        struct {                           // live during key build + merge
            uint32_t key[4][WIN];
            uint32_t tmpA[2 * WIN];
            uint32_t tmpB[2 * WIN];
        } m;
        struct {                           // live during the sweeps ([j][lane] layout)
            uint32_t evr[EPL][32];         // event appearance time (relative), RINF if none
            uint8_t gev[EPL][32];          // bit0..1 E value, bit2 group end
        } s;
    } u;                                   // 4 KB
    uint32_t merged[EPL][32];              // 2 KB  merged keys, [j][lane]
    uint64_t pend[PMAX];                   // 512 B
    uint64_t out[OB];                      // 8 KB
    unsigned long long spill_off[NSPILL];
    uint32_t spill_cnt[NSPILL];
    uint32_t dtab[4][2][3];                // per pin: [fall, rise][out 0, 1, X] (R1)
    // cursors (warp-uniform, written by lane 0)
    unsigned long long c_off[4];
    uint32_t c_rem[4], c_ck[4], c_ckend[4], whead[4], wcnt[4], more[4];
};
constexpr int kWarpsPerBlock = kThreads / 32;
constexpr size_t kSmemBytes = sizeof(WS) * kWarpsPerBlock;

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

// merge two strictly increasing key lists (keys are unique) with merge path.
// Output d goes to C[d] (linear) or, if T, to CT[d - d0][lane] (lane's slice).
template <bool T>
__device__ __forceinline__ void merge2(const uint32_t* A, int na, const uint32_t* B, int nb, uint32_t* C,
                                       uint32_t (*CT)[32], int per, int lane) {
    const int n = na + nb;
    const int d0 = min(lane * per, n), d1 = min(d0 + per, n);
    int lo = max(0, d0 - nb), hi = min(d0, na);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (A[mid] < B[d0 - 1 - mid]) lo = mid + 1; else hi = mid;
    }
    int ia = lo, ib = d0 - lo;
    for (int d = d0; d < d1; ++d) {
        const bool takeA = ib >= nb || (ia < na && A[ia] < B[ib]);
        const uint32_t v = takeA ? A[ia] : B[ib];
        ia += takeA;
        ib += !takeA;
        if (T) CT[d - d0][lane] = v; else C[d] = v;
    }
}

struct Emit {   // per-chunk output state (warp-uniform)
    int out_n;
    int nspill;
    uint32_t vb;
    uint32_t last_val;
};

// spill the output buffer to the deep-scratch pool; false if out of room
__device__ __noinline__ bool spill(const SimParams& p, WS& ws, Emit& em, int lane) {
    if (em.out_n == 0) return true;
    if (em.nspill >= NSPILL) return false;
    unsigned long long at = 0;
    if (lane == 0) at = atomicAdd(&p.ctl->deep_top, (unsigned long long)em.out_n);
    at = __shfl_sync(FULL, at, 0);
    if (at + (unsigned long long)em.out_n > p.deep_cap) {
        if (lane == 0) {
            atomicOr(&p.ctl->error, kErrDeep);
            atomicMax(&p.ctl->need_deep, at + (unsigned long long)em.out_n);
        }
        return false;
    }
    for (int q = lane; q < em.out_n; q += 32) p.deep[at + q] = ws.out[q];
    if (lane == 0) {
        ws.spill_off[em.nspill] = at;
        ws.spill_cnt[em.nspill] = (uint32_t)em.out_n;
    }
    __syncwarp();
    em.nspill++;
    em.out_n = 0;
    return true;
}

// coalesced refill of pin i's window up to WIN entries (warp-uniform control)
__device__ __forceinline__ void refill(const SimParams& p, WS& ws, int i, long long T1, int lane) {
    uint32_t wc = ws.wcnt[i], more = ws.more[i];
    if (!more || wc >= (uint32_t)WIN) return;
    unsigned long long off = ws.c_off[i];
    uint32_t rem = ws.c_rem[i], ck = ws.c_ck[i];
    const uint32_t ckend = ws.c_ckend[i], wh = ws.whead[i];
    while (more && wc < (uint32_t)WIN) {
        if (rem == 0) {
            if (ck + 1 < ckend) {
                ++ck;
                off = p.ck_off[ck];
                rem = p.ck_cnt[ck];
                continue;
            }
            more = 0;
            break;
        }
        const uint32_t take = min(min((uint32_t)WIN - wc, rem), 32u);
        uint64_t e = 0;
        if ((uint32_t)lane < take) {
            e = p.arena[off + lane];
            ws.win[i][(wh + wc + lane) & (WIN - 1)] = e;
        }
        const uint64_t last = __shfl_sync(FULL, e, take - 1);
        off += take;
        rem -= take;
        wc += take;
        if (etime(last) >= T1) more = 0;   // later entries cannot matter
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
__device__ __noinline__ bool warp_chunk(const SimParams& p, WS& ws, const ChunkSetup& s, const uint8_t* lut,
                                        unsigned long long& out_off, uint32_t& out_cnt, uint32_t& out_vb,
                                        unsigned long long& evals, unsigned long long& events, bool& fits) {
    const int lane = threadIdx.x & 31;
    const int k = (int)s.k;
    const uint32_t lb = s.lut_base;
    const long long T0 = s.T0, T1 = s.T1, dur = p.duration, dmin = (long long)s.dmin;

    // delay tables (reading R1: output X takes the smaller of the two)
    if (lane < 4) {
        const uint4 d = lane == 0 ? s.d[0] : lane == 1 ? s.d[1] : lane == 2 ? s.d[2] : s.d[3];
        ws.dtab[lane][1][0] = d.x;                 // RISE -> 0
        ws.dtab[lane][1][1] = d.y;                 // RISE -> 1
        ws.dtab[lane][1][2] = min(d.x, d.y);
        ws.dtab[lane][0][0] = d.z;                 // FALL -> 0
        ws.dtab[lane][0][1] = d.w;                 // FALL -> 1
        ws.dtab[lane][0][2] = min(d.z, d.w);
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
                if (f != 2u) del = min(del, ws.dtab[i][f == 1u ? 1 : 0][E0]);
            }
            if (lane == 0) ws.pend[0] = ((uint64_t)(s.tau0 + (long long)del) << 2) | E0;
            np = 1;
        }
    }
    __syncwarp();
    unsigned long long n_evals = 0, n_events = 0;

    for (;;) {
        // ---- 1. refill windows (coalesced)
        for (int i = 0; i < k; ++i) refill(p, ws, i, T1, lane);
        // ---- 2. tile bounds
        long long tbase = LLONG_MAX, tsafe = LLONG_MAX;
        for (int i = 0; i < k; ++i) {
            const uint32_t wc = ws.wcnt[i], wh = ws.whead[i];
            if (wc > 0) {
                tbase = min(tbase, etime(ws.win[i][wh]));
                if (ws.more[i]) tsafe = min(tsafe, etime(ws.win[i][(wh + wc - 1) & (WIN - 1)]));
            }
        }
        if (tbase >= T1) break;                               // nothing left before T1
        const long long tlim = min(min(tsafe, T1 - 1), tbase + SPAN);
        int mi[4] = {0, 0, 0, 0};
        int nt = 0;
        for (int i = 0; i < k; ++i) {
            const uint32_t wc = ws.wcnt[i], wh = ws.whead[i];
            int m = 0;
#pragma unroll
            for (int q = 0; q < WIN / 32; ++q) {
                const uint32_t j = lane + 32 * q;
                const uint64_t e = j < wc ? ws.win[i][(wh + j) & (WIN - 1)] : kInfEntry;
                const bool pr = j < wc && etime(e) <= tlim;
                m += __popc(__ballot_sync(FULL, pr));
                if (pr) ws.u.m.key[i][j] = ((uint32_t)(etime(e) - tbase) << 4) | ((uint32_t)i << 2) | (uint32_t)(e & 3u);
            }
            mi[i] = m;
            nt += m;
        }
        __syncwarp();
        // ---- 3. k-way merge; lane l gets merged entries [l*Ep, l*Ep + nv) in merged[j][l]
        const int Ep = (nt + 31) >> 5;
        const int nv = max(0, min(Ep, nt - lane * Ep));
        if (k == 1) {
            for (int j = 0; j < nv; ++j) ws.merged[j][lane] = ws.u.m.key[0][lane * Ep + j];
        } else if (k == 2) {
            merge2<true>(ws.u.m.key[0], mi[0], ws.u.m.key[1], mi[1], nullptr, ws.merged, Ep, lane);
        } else if (k == 3) {
            const int n01 = mi[0] + mi[1];
            merge2<false>(ws.u.m.key[0], mi[0], ws.u.m.key[1], mi[1], ws.u.m.tmpA, nullptr, (n01 + 31) >> 5, lane);
            __syncwarp();
            merge2<true>(ws.u.m.tmpA, n01, ws.u.m.key[2], mi[2], nullptr, ws.merged, Ep, lane);
        } else {
            const int n01 = mi[0] + mi[1], n23 = mi[2] + mi[3];
            merge2<false>(ws.u.m.key[0], mi[0], ws.u.m.key[1], mi[1], ws.u.m.tmpA, nullptr, (n01 + 31) >> 5, lane);
            merge2<false>(ws.u.m.key[2], mi[2], ws.u.m.key[3], mi[3], ws.u.m.tmpB, nullptr, (n23 + 31) >> 5, lane);
            __syncwarp();
            merge2<true>(ws.u.m.tmpA, n01, ws.u.m.tmpB, n23, nullptr, ws.merged, Ep, lane);
        }
        __syncwarp();
        // the entry after my last one (next lane's first), for timestamp grouping
        const uint32_t nxt = (lane < 31 && (lane + 1) * Ep < nt) ? ws.merged[0][lane + 1] : RINF;
        const uint32_t tnxt = nxt == RINF ? RINF : (nxt >> 4);

        // ---- 4a. compose input updates (whole lane and up to the last group end)
        uint32_t upd = 0, upd_ge = 0;
        bool has_ge = false;
        for (int j = 0; j < nv; ++j) {
            const uint32_t key = ws.merged[j][lane];
            const uint32_t pin = (key >> 2) & 3u;
            upd = (upd | (0x100u << pin));
            upd = (upd & ~(3u << (2 * pin))) | (norm_code(key & 3u) << (2 * pin));
            const uint32_t tn = j + 1 < nv ? (ws.merged[j + 1][lane] >> 4) : tnxt;
            if (tn != (key >> 4)) {
                upd_ge = upd;
                has_ge = true;
            }
        }
        uint32_t x = upd;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x = ((y | x) & 0xf00u) | ((y & ~expand4(x >> 8)) & 0xffu) | (x & 0xffu);
        }
        const uint32_t xe0 = __shfl_up_sync(FULL, x, 1);
        const uint32_t xe = lane == 0 ? 0u : xe0;
        const uint32_t xtot = __shfl_sync(FULL, x, 31);
        const uint32_t vstart = apply_upd(vec_carry, xe);
        // vector at the previous timestamp before my first group end
        const uint32_t tagged = has_ge ? (0x100u | apply_upd(vstart, upd_ge)) : 0u;
        uint32_t vprev;
        {
            const unsigned lanes_with = __ballot_sync(FULL, nv > 0);
            const unsigned lanes_ge = __ballot_sync(FULL, has_ge);
            // every lane before the last populated one holds a group end -> one shuffle
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
        // ---- 4b. evaluations and events (Alg. 2; delays P:210)
        const uint32_t thr = T0 <= tbase ? 0u : (uint32_t)min(T0 - tbase, (long long)(1 << 28));
        uint32_t Eprev = lut[lb + vprev];
        uint32_t v = vstart;
        uint32_t lmin = RINF;
        uint32_t cnt_ge = 0, cnt_ev = 0;
        for (int j = 0; j < nv; ++j) {
            const uint32_t key = ws.merged[j][lane];
            v = set_pin(v, key);
            const uint32_t tj = key >> 4;
            const uint32_t tn = j + 1 < nv ? (ws.merged[j + 1][lane] >> 4) : tnxt;
            uint32_t r = RINF, g = 0;
            if (tn != tj) {
                const uint32_t E = lut[lb + v];
                cnt_ge += tj >= thr;
                g = 4u | E;
                if (E != Eprev) {
                    uint32_t del = RINF;
                    const uint32_t diff = v ^ vprev;
                    for (int i = 0; i < k; ++i) {
                        if ((diff >> (2 * i)) & 3u) {
                            const uint32_t fo = (vprev >> (2 * i)) & 3u, fn = (v >> (2 * i)) & 3u;
                            del = min(del, ws.dtab[i][rank_code(fn) > rank_code(fo) ? 1 : 0][E]);
                        }
                    }
                    r = tj + del;
                    lmin = min(lmin, r);
                    cnt_ev += tj >= thr;
                }
                vprev = v;
                Eprev = E;
            }
            ws.u.s.evr[j][lane] = r;
            ws.u.s.gev[j][lane] = (uint8_t)g;
        }
        n_evals += cnt_ge;
        n_events += cnt_ev;
        // ---- 5. Eq. 1 survivors: r below every later event's r
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
            const uint32_t r = ws.u.s.evr[j][lane];
            if (r < run) {                                   // r == RINF never passes
                if (!survmask) lsv = ws.u.s.gev[j][lane] & 3u;
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
        // dedupe predecessor of my first survivor
        uint32_t prevv;
        {
            const uint32_t t = excl_last_valid(survmask ? (0x100u | lsv) : 0u, lane);
            prevv = (t & 0x100u) ? (t & 3u) : pred_init;
        }
        const uint64_t lim_rel64 = (uint64_t)(tlim - tbase) + (uint64_t)dmin;
        const uint32_t lim_rel = lim_rel64 >= RINF ? RINF - 1 : (uint32_t)lim_rel64;
        uint32_t finmask = 0, pendmask = 0, outmask = 0;
        int last_fin_j = -1, last_vb_j = -1;
        for (uint32_t m = survmask; m; m &= m - 1) {
            const int j = __ffs(m) - 1;
            const uint32_t E = ws.u.s.gev[j][lane] & 3u;
            if (E != prevv) {
                const uint32_t r = ws.u.s.evr[j][lane];
                if (r <= lim_rel) {
                    finmask |= 1u << j;
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
        if (em.out_n + n_oout + tot_out > OB) {
            if (!spill(p, ws, em, lane)) return false;
        }
        // outputs: old finals, then tile finals, in order
        if (oa) ws.out[em.out_n + __popc(boa & ((1u << lane) - 1u))] = pa;
        if (ob) ws.out[em.out_n + __popc(boa) + __popc(bob & ((1u << lane) - 1u))] = pb;
        {
            int q = em.out_n + n_oout + (int)(pre & 0xffffu);
            for (uint32_t m = outmask; m; m &= m - 1) {
                const int j = __ffs(m) - 1;
                const long long ra = tbase + (long long)ws.u.s.evr[j][lane];
                ws.out[q++] = ((uint64_t)ra << 2) | (ws.u.s.gev[j][lane] & 3u);
            }
        }
        {   // value before T0 and last final value from the tile
            const unsigned bl = __ballot_sync(FULL, last_vb_j >= 0);
            const uint32_t vvb = last_vb_j >= 0 ? ws.u.s.gev[last_vb_j][lane] & 3u : 0u;
            const uint32_t wvb = __shfl_sync(FULL, vvb, bl ? 31 - __clz(bl) : 0);
            if (bl) em.vb = wvb;
            const unsigned bf = __ballot_sync(FULL, last_fin_j >= 0);
            const uint32_t vlf = last_fin_j >= 0 ? ws.u.s.gev[last_fin_j][lane] & 3u : 0u;
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
                ws.pend[q++] = ((uint64_t)(tbase + (long long)ws.u.s.evr[j][lane]) << 2) | (ws.u.s.gev[j][lane] & 3u);
            }
        }
        np = keep_old + tot_pend;
        em.out_n += n_oout + tot_out;
        // consume the tile
        if (lane < k) {
            const int m = lane == 0 ? mi[0] : lane == 1 ? mi[1] : lane == 2 ? mi[2] : mi[3];
            ws.whead[lane] = (ws.whead[lane] + (uint32_t)m) & (WIN - 1);
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
        if (em.out_n + n > OB) {
            if (!spill(p, ws, em, lane)) return false;
        }
        if (oa) ws.out[em.out_n + __popc(boa & ((1u << lane) - 1u))] = pa;
        if (ob) ws.out[em.out_n + __popc(boa) + __popc(bob & ((1u << lane) - 1u))] = pb;
        const uint32_t bva = __ballot_sync(FULL, lane < np && etime(pa) < T0);
        const uint32_t bvb = __ballot_sync(FULL, lane + 32 < np && etime(pb) < T0);
        if (bva | bvb) em.vb = (uint32_t)(ws.pend[bvb ? 32 + 31 - __clz(bvb) : 31 - __clz(bva)] & 3u);
        em.out_n += n;
        __syncwarp();
    }
    // exact allocation of the chunk's segment and coalesced copy-out
    uint32_t total = (uint32_t)em.out_n;
    for (int q = 0; q < em.nspill; ++q) total += ws.spill_cnt[q];
    unsigned long long at = 0;
    if (lane == 0 && total) at = atomicAdd(&p.ctl->arena_top, (unsigned long long)total);
    at = __shfl_sync(FULL, at, 0);
    fits = at + total <= p.arena_cap;
    if (!fits) {
        if (lane == 0) {
            atomicOr(&p.ctl->error, kErrArena);
            atomicMax(&p.ctl->need_arena, at + total);
        }
    } else {
        unsigned long long o = at;
        for (int q = 0; q < em.nspill; ++q) {
            const unsigned long long so = ws.spill_off[q];
            const uint32_t sc = ws.spill_cnt[q];
            for (uint32_t e = lane; e < sc; e += 32) p.arena[o + e] = p.deep[so + e];
            o += sc;
        }
        for (int e = lane; e < em.out_n; e += 32) p.arena[o + e] = ws.out[e];
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
