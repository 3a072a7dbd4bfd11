// gls_csrp.cuh — engine 2: the paper's own design, literally, on B200 (NEXT-3, an A/B
// baseline for engines 0 and 1).  Included by gls_kernels.cu.
//
//   * CSRP store (§3.1, Fig. 6b/7): waveforms live in fixed pages of `pagelen`
//     slots; each page holds pagelen - 1 entries and, in its last slot, the index of the
//     next page of the same waveform; a terminate marker follows the last entry (it may sit
//     in the last slot).  Pages are handed out by one atomic page iterator, so a
//     waveform's pages are generally not consecutive.  Given and computed waveforms share
//     the store.  Memory waste <= pagelen * k * M_t for k waveforms (Eq. 4, P:316-319;
//     checked by the tests from gls_stats).
//   * Alg. 1: one thread per cell, cells dealt statically to the threads in
//     topological order (thread t takes gates t, t + T, t + 2T, ...); a thread waits until
//     every input waveform of its cell is known (a flag per net, release / acquire), then
//     runs Alg. 2 over the whole waveform, reading its inputs page by page.
//   * The output of a cell is built in the thread's private memory (the paper's individual
//     memory; here the Eq. 1 stack in the lane scratch, exact for any backtrace —
//     reading R13) and copied into CSRP pages as entries become final (r <= t + dmin: no
//     later event can deny them) and at the end.
// Encoding: an entry is (t << 2) | v (t < 2^61, so bit 63 is clear); a next-page slot holds
// kPageLink | page; the terminate marker is ~0.
#pragma once

namespace gls {
namespace cp {

constexpr uint64_t kTerm = ~0ull;
constexpr uint64_t kPageLink = 1ull << 63;

struct Reader {
    const uint64_t* pages;
    uint32_t L;            // pagelen
    unsigned long long page;
    uint32_t slot;
    uint64_t head;         // current entry (kTerm at the end)
    __device__ __forceinline__ void load() {
        for (;;) {
            const uint64_t e = __ldcg(&pages[page * L + slot]);
            if (slot == L - 1 && e != kTerm) {            // next-page pointer
                page = e & ~kPageLink;
                slot = 0;
                continue;
            }
            head = e;
            return;
        }
    }
    __device__ __forceinline__ void next() {
        ++slot;
        load();
    }
};

struct Writer {
    uint64_t* pages;
    uint32_t L;
    unsigned long long page, first;
    uint32_t slot;
    unsigned long long* top;
    unsigned long long cap;    // pages
    bool overflow;
    __device__ void begin() {
        page = first = atomicAdd(top, 1ull);
        slot = 0;
        overflow = page >= cap;
    }
    __device__ void put(uint64_t e) {
        if (overflow) return;
        if (slot == L - 1) {                              // page full: link a new one
            const unsigned long long np = atomicAdd(top, 1ull);
            if (np >= cap) {
                overflow = true;
                return;
            }
            pages[page * L + slot] = kPageLink | np;
            page = np;
            slot = 0;
        }
        pages[page * L + slot++] = e;
    }
    __device__ void end() {
        if (!overflow) pages[page * L + slot] = kTerm;   // may be the last slot
    }
};

struct CsrpParams {
    uint64_t* pages;
    unsigned long long* page_top;
    unsigned long long page_cap;
    uint32_t pagelen;
    unsigned long long* first_page;   // [P + G]
    uint32_t* known;                  // [G] Alg. 1's flag of each gate output
    unsigned long long* out_cnt;      // [P + G] entries stored per net
};

// given waveforms into pages: one thread per given net
__global__ void csrp_given_kernel(SimParams p, CsrpParams c, const long long* in_off) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.P; i += gridDim.x * blockDim.x) {
        Writer w{c.pages, c.pagelen, 0, 0, 0, c.page_top, c.page_cap, false};
        w.begin();
        for (long long j = in_off[i]; j < in_off[i + 1]; ++j) w.put(p.arena[j]);
        w.end();
        if (w.overflow) atomicOr(&p.ctl->error, kErrArena);
        c.first_page[i] = w.first;
        c.out_cnt[i] = (unsigned long long)(in_off[i + 1] - in_off[i]);
    }
}

// Alg. 1 + Alg. 2 with the CSRP store: one thread per cell, statically dealt
__global__ void __launch_bounds__(128) csrp_kernel(SimParams p, CsrpParams c) {
    __shared__ uint8_t lut[kLutCap];
    for (int i = threadIdx.x; i < kLutCap; i += blockDim.x) lut[i] = p.lut[i];
    __syncthreads();
    const unsigned long long T = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t* const stk = p.wscr + tid * (unsigned long long)kCsrpStack;   // the thread's individual memory
    unsigned long long evals = 0, events = 0, outs = 0;
    for (unsigned long long gi = tid; gi < (unsigned long long)p.G; gi += T) {
        const GateInfo g = p.gate[gi];
        const uint32_t k = g.k;
        uint32_t src[4] = {0, 0, 0, 0};
        uint4 d[4];
        uint32_t dmin = 0xffffffffu;
        for (uint32_t i = 0; i < k; ++i) {
            src[i] = p.pin_src[g.pin_off + i];
            d[i] = p.pin_delay[g.pin_off + i];
            const uint32_t f[4] = {d[i].x, d[i].y, d[i].z, d[i].w};
            for (int q = 0; q < 4; ++q)
                if (f[q] != kDelayInf) dmin = min(dmin, f[q]);
        }
        if (dmin == 0xffffffffu) dmin = 0;
        // wait until every input waveform is known (Alg. 1)
        for (uint32_t i = 0; i < k; ++i) {
            if (src[i] < (uint32_t)p.P) continue;
            unsigned ns = 32;
            while (ld_acquire_u32(&c.known[src[i] - p.P]) == 0u) {
                if (ld_relaxed_u32(&p.ctl->error) != 0u) return;
                __nanosleep(ns);
                if (ns < 4096) ns <<= 1;
            }
        }
        Reader rd[4];
        uint32_t xn = 0;
        for (uint32_t i = 0; i < k; ++i) {
            rd[i] = Reader{c.pages, c.pagelen, c.first_page[src[i]], 0, kTerm};
            rd[i].load();
            xn |= 2u << (2 * i);                          // inputs start at X
        }
        for (uint32_t i = k; i < 4; ++i) rd[i].head = kTerm;
        Writer w{c.pages, c.pagelen, 0, 0, 0, c.page_top, c.page_cap, false};
        w.begin();
        uint32_t Eprev = 2;                               // zero-delay evaluation (R4a)
        uint32_t n = 0, flushed = 0;                      // stack [flushed, n) in stk; below: in pages
        uint32_t floorv = 2;                              // value of the last flushed entry (X: none)
        unsigned long long nout = 0;
        bool ovf = false;
        for (;;) {
            const uint64_t m = min(min(rd[0].head, rd[1].head), min(rd[2].head, rd[3].head));
            if (m == kTerm) break;
            const long long t = (long long)(m >> 2);
            uint32_t nx = xn;
            for (uint32_t i = 0; i < k; ++i) {
                if (rd[i].head != kTerm && (long long)(rd[i].head >> 2) == t) {
                    const uint32_t v = (uint32_t)(rd[i].head & 3u);
                    nx = (nx & ~(3u << (2 * i))) | ((v == 3u ? 2u : v) << (2 * i));   // Z -> X
                    rd[i].next();
                }
            }
            ++evals;
            if (nx != xn) {
                const uint32_t E = lut[g.lut_base + nx];  // calculateSignals
                if (E != Eprev) {
                    ++events;
                    uint32_t del = 0xffffffffu;
                    for (uint32_t i = 0; i < k; ++i) {
                        const uint32_t fo = (xn >> (2 * i)) & 3u, fn = (nx >> (2 * i)) & 3u;
                        if (fo == fn) continue;            // changed inputs only (R3)
                        const bool rise = ((fn & 1u) << 1 | fn >> 1) > ((fo & 1u) << 1 | fo >> 1);   // 0 < X < 1 (R2)
                        const uint32_t a = rise ? d[i].x : d[i].z, b = rise ? d[i].y : d[i].w;
                        const uint32_t dd = E == 0u ? a : E == 1u ? b : min(a, b);   // R1
                        del = min(del, dd);                // min rule
                    }
                    if (del != kDelayInf) {                // R9
                        const uint64_t r = (uint64_t)(t + (long long)del);
                        // addSignalChange with Eq. 1 on the stack
                        while (n > flushed && (stk[n - 1] >> 2) >= r) --n;
                        const uint32_t tv = n > flushed ? (uint32_t)(stk[n - 1] & 3u) : floorv;
                        if (tv != E) {
                            if (n == (uint32_t)kCsrpStack) {
                                ovf = true;                // (bounded by the final-entry flushes below)
                            } else {
                                stk[n++] = (r << 2) | E;
                            }
                        }
                    }
                    Eprev = E;
                }
                xn = nx;
            }
            // entries final at t (r <= t + dmin) move from the individual memory into pages
            if (n - flushed >= (uint32_t)kCsrpStack / 2 || n == (uint32_t)kCsrpStack) {
                uint32_t f = flushed;
                while (f < n && (long long)(stk[f] >> 2) <= t + (long long)dmin) {
                    if ((long long)(stk[f] >> 2) <= p.duration) {
                        w.put(stk[f]);
                        ++nout;
                    }
                    floorv = (uint32_t)(stk[f] & 3u);
                    ++f;
                }
                for (uint32_t q = f; q < n; ++q) stk[q - f] = stk[q];
                n -= f;
                flushed = 0;
            }
        }
        for (uint32_t q = flushed; q < n; ++q) {          // the rest, clipped at the duration (R7)
            if ((long long)(stk[q] >> 2) > p.duration) break;
            w.put(stk[q]);
            ++nout;
        }
        w.end();
        if (w.overflow) atomicOr(&p.ctl->error, kErrArena);
        if (ovf) atomicOr(&p.ctl->error, kErrDeep);
        c.first_page[p.P + gi] = w.first;
        c.out_cnt[p.P + gi] = nout;
        outs += nout;
        fence_release();
        st_release_u32(&c.known[gi], 1u);                 // Alg. 1: the output is known
    }
    atomicAdd(&p.ctl->gate_evals, evals);
    atomicAdd(&p.ctl->events, events);
    atomicAdd(&p.ctl->out_trans, outs);
}

// the canonical store of the result: each gate output's pages copied, in order, into one
// exact arena segment (one chunk per net) — "this CSRP structure will be transferred to the
// CPU as the output" — so every reader of the library works unchanged
__global__ void csrp_collect_kernel(SimParams p, CsrpParams c, const unsigned long long* seg_off) {
    for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < p.G;
         gi += (long long)gridDim.x * blockDim.x) {
        const uint32_t net = (uint32_t)p.P + (uint32_t)gi;
        const unsigned long long off = seg_off[gi], cnt = c.out_cnt[net];
        Reader rd{c.pages, c.pagelen, c.first_page[net], 0, kTerm};
        rd.load();
        for (unsigned long long q = 0; q < cnt; ++q) {
            p.arena[off + q] = rd.head;
            rd.next();
        }
        p.net_ck[net] = net;
        p.net_nck[net] = 1;
        p.net_len[net] = cnt;
        p.ck_T[net] = 0;
        p.ck_off[net] = off;
        p.ck_cnt[net] = (uint32_t)cnt;
        p.ck_cum[net] = 0;
        p.ck_vb[net] = 2;
        p.ck_gate[net] = (uint32_t)gi;
    }
}

}  // namespace cp
}  // namespace gls
