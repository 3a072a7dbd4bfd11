// gls_api.cu — host side of the C ABI declared in include/gls.h.
//
// a1 netlist validation + levelisation (Kahn order, counting sort by level,
// fan-in CSR in level order), a2 given-waveform validation + packing into the
// device store, the 4-value LUT build (a3), memory sizing, the single
// persistent-kernel launch (a4-a9) and result readback (a10).  DESIGN.md §5.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/gls.h"
#include "gls_internal.cuh"

using namespace gls;

namespace {

// ---------------------------------------------------------------- 4-value LUT
// Built from a dual-rail reading of X = "0 or 1": a value is the pair
// (can_be_0, can_be_1); Z is read as X.  AND/OR/XOR on the pairs reproduce
// Table 1; N-gates negate; MUX2 is composed as in reading R11.
struct Dual { bool c0, c1; };
Dual dual(int v) { return v == 0 ? Dual{true, false} : v == 1 ? Dual{false, true} : Dual{true, true}; }
int undual(Dual d) { return d.c0 && d.c1 ? 2 : (d.c1 ? 1 : 0); }
Dual d_not(Dual a) { return Dual{a.c1, a.c0}; }
Dual d_and(Dual a, Dual b) { return Dual{a.c0 || b.c0, a.c1 && b.c1}; }
Dual d_or(Dual a, Dual b) { return Dual{a.c0 && b.c0, a.c1 || b.c1}; }
Dual d_xor(Dual a, Dual b) {
    return Dual{(a.c0 && b.c0) || (a.c1 && b.c1), (a.c0 && b.c1) || (a.c1 && b.c0)};
}

int lut_eval(int type, int k, const int* v) {
    if (k < 1 || k > 4) return -1;
    Dual x[4] = {};
    for (int i = 0; i < k && i < 4; ++i) x[i] = dual(v[i]);
    Dual r;
    switch (type) {
        case GLS_BUF: r = x[0]; break;
        case GLS_NOT: r = d_not(x[0]); break;
        case GLS_AND: case GLS_NAND:
            r = x[0];
            for (int i = 1; i < k; ++i) r = d_and(r, x[i]);
            if (type == GLS_NAND) r = d_not(r);
            break;
        case GLS_OR: case GLS_NOR:
            r = x[0];
            for (int i = 1; i < k; ++i) r = d_or(r, x[i]);
            if (type == GLS_NOR) r = d_not(r);
            break;
        case GLS_XOR: case GLS_XNOR:
            r = x[0];
            for (int i = 1; i < k; ++i) r = d_xor(r, x[i]);
            if (type == GLS_XNOR) r = d_not(r);
            break;
        case GLS_MUX2: r = d_or(d_and(x[0], d_not(x[2])), d_and(x[1], x[2])); break;
        default: return -1;
    }
    return undual(r);
}

bool arity_ok(int type, int64_t k) {
    if (type == GLS_BUF || type == GLS_NOT) return k == 1;
    if (type == GLS_MUX2) return k == 3;
    if (type >= GLS_AND && type <= GLS_XNOR) return k >= 2 && k <= 4;
    return false;
}

const std::vector<uint8_t>& lut_table() {
    static std::vector<uint8_t> t;
    if (t.empty()) {
        t.assign(kLutCap, 2);                     // (the rest: cell output functions, gls_load_cells)
        for (int type = 0; type < kNumTypes; ++type)
            for (int k = 1; k <= 4; ++k) {
                int base = lut_offset(type, k);
                for (int idx = 0; idx < (1 << (2 * k)); ++idx) {
                    int v[4];
                    bool valid = true;
                    for (int i = 0; i < k; ++i) {
                        v[i] = (idx >> (2 * i)) & 3;
                        if (v[i] == 3) valid = false;  // the kernel indexes normalised codes
                    }
                    if (!valid || !arity_ok(type, k)) continue;
                    t[base + idx] = (uint8_t)lut_eval(type, k, v);
                }
            }
    }
    return t;
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaError_t alloc(size_t count) {
        release();
        if (count == 0) count = 1;
        cudaError_t e = cudaMalloc(&p, count * sizeof(T));
        if (e != cudaSuccess) { p = nullptr; n = 0; return e; }
        n = count;
        return cudaSuccess;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    cudaError_t ensure(size_t count) { return n >= count && p ? cudaSuccess : alloc(count); }
    ~DevBuf() { release(); }
};

}  // namespace

struct gls_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    gls_config cfg{};
    std::string err;

    // netlist
    bool has_netlist = false;
    int32_t P = 0, G = 0, L = 0;
    int64_t E = 0;
    int64_t halo = 1;
    bool has_inf = false;                   // some pin delay is GLS_DELAY_INF
    std::vector<uint32_t> perm;        // internal gate -> user gate
    std::vector<uint32_t> inv;         // user gate -> internal gate
    std::vector<int64_t> net_fanout;   // internal net -> pins it drives
    DevBuf<uint32_t> d_fo_off, d_fo_gate, d_pend0, d_pend;
    DevBuf<uint32_t> d_fanout;              // internal net -> pins it drives (algorithmic-bytes count)
    DevBuf<unsigned long long> d_deep_wtop;
    DevBuf<int32_t> d_level_off;
    DevBuf<GateInfo> d_gate;
    DevBuf<uint32_t> d_pin_src;
    DevBuf<uint4> d_pin_delay;
    DevBuf<uint8_t> d_lut;
    DevBuf<uint32_t> d_perm;
    DevBuf<uint32_t> d_inv;                 // user gate -> internal gate (canonical readback)
    DevBuf<uint32_t> d_net_ck, d_net_nck, d_gate_done;
    DevBuf<unsigned long long> d_gate_nin;
    DevBuf<unsigned long long> d_net_len;
    DevBuf<unsigned long long> d_work;

    // given waveforms (in the arena prefix)
    bool has_inputs = false;
    int64_t in_total = 0;
    int64_t max_in_time = -1;
    DevBuf<long long> d_in_off;
    // time window (gls_simulate_window): the window's slice of the given waveforms sits
    // after them in the arena, with its own offsets; the full inputs stay in place
    bool window_active = false;
    int64_t prefix_total = 0;          // arena entries to keep (given waveforms [+ window slice])
    int64_t win_max_time = -1;
    DevBuf<long long> d_win_off;
    DevBuf<uint64_t> d_arena;
    bool arena_auto = true;

    // chunk tables
    DevBuf<long long> d_ck_T;
    DevBuf<unsigned long long> d_ck_off, d_ck_cum;
    DevBuf<uint32_t> d_ck_cnt, d_ck_gate;
    DevBuf<uint8_t> d_ck_vb;
    DevBuf<uint64_t> d_deep;
    DevBuf<uint64_t> d_wscr;
    DevBuf<unsigned long long> d_trace;     // gls_config.trace
    DevBuf<uint64_t> d_pages;               // engine 2: CSRP pages
    DevBuf<unsigned long long> d_first_page, d_out_cnt, d_seg_off;
    DevBuf<uint32_t> d_known;
    bool traced = false;
    DevBuf<unsigned char> d_waux;
    DevBuf<uint64_t> d_hash;                // result checksums (kept: no malloc/free per readback)
    DevBuf<Ctl> d_ctl;
    DevBuf<unsigned> d_flag;
    DevBuf<unsigned long long> d_flag64;

    // results
    bool has_result = false;
    int64_t duration = 0;
    int64_t deep_per_warp = 0;
    Ctl last{};
    unsigned long long last_chunk_top = 0;   // chunk ids used by earlier runs (cleared before the next)
    gls_stats stats{};
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
};

namespace {

int fail(gls_ctx* c, int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    return code;
}

#define CK(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) {                                                                   \
            cudaGetLastError();                                                                    \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? GLS_ENOMEM : GLS_ECUDA,             \
                        "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__);      \
        }                                                                                          \
    } while (0)

int64_t free_bytes(gls_ctx* ctx) {
    size_t fr = 0, tot = 0;
    cudaSetDevice(ctx->device);
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return 0;
    return (int64_t)fr;
}

int default_M(int engine) { return engine == 0 ? 32768 : 256; }

SimParams params(gls_ctx* ctx) {
    SimParams p{};
    p.P = ctx->P;
    p.G = ctx->G;
    p.L = ctx->L;
    p.level_off = ctx->d_level_off.p;
    p.gate = ctx->d_gate.p;
    p.pin_src = ctx->d_pin_src.p;
    p.pin_delay = ctx->d_pin_delay.p;
    p.lut = ctx->d_lut.p;
    p.arena = ctx->d_arena.p;
    p.arena_cap = ctx->d_arena.n;
    p.net_ck = ctx->d_net_ck.p;
    p.net_nck = ctx->d_net_nck.p;
    p.net_len = ctx->d_net_len.p;
    p.ck_T = ctx->d_ck_T.p;
    p.ck_off = ctx->d_ck_off.p;
    p.ck_cnt = ctx->d_ck_cnt.p;
    p.ck_cum = ctx->d_ck_cum.p;
    p.ck_vb = ctx->d_ck_vb.p;
    p.ck_gate = ctx->d_ck_gate.p;
    p.ck_cap = ctx->d_ck_T.n;
    p.gate_done = ctx->d_gate_done.p;
    p.gate_nin = ctx->d_gate_nin.p;
    p.work = ctx->d_work.p;
    p.deep = ctx->d_deep.p;
    p.wscr = ctx->d_wscr.p;
    p.waux = ctx->d_waux.p;
    p.trace = ctx->cfg.trace ? ctx->d_trace.p : nullptr;
    p.deep_wtop = ctx->d_deep_wtop.p;
    p.fo_off = ctx->d_fo_off.p;
    p.fo_gate = ctx->d_fo_gate.p;
    p.pend = ctx->d_pend.p;
    p.deep_cap = ctx->d_deep.n;
    p.deep_per_warp = (unsigned long long)ctx->deep_per_warp;
    p.ctl = ctx->d_ctl.p;
    p.duration = ctx->duration;
    p.engine = ctx->cfg.engine;
    p.sched = (p.engine == 1 || ctx->cfg.scheduler == 1) ? 1 : 0;
    p.M = ctx->cfg.chunk_events > 0 ? ctx->cfg.chunk_events : default_M(p.engine);
    int rl = ctx->cfg.ring_limit;
    p.ring_cap = (rl > 0 && rl < kRing) ? rl : kRing;
    return p;
}

// Chunk-table entries per arena entry for auto sizing.
double chunk_ratio(gls_ctx* ctx) {
    int M = ctx->cfg.chunk_events > 0 ? ctx->cfg.chunk_events : default_M(ctx->cfg.engine);
    double fan = (double)ctx->E / std::max<double>(1.0, (double)ctx->P + ctx->G);
    return 1.5 * (fan + 0.5) / (double)M;
}

constexpr int64_t kChunkBytes = 8 + 8 + 8 + 4 + 4 + 1;  // T, off, cum, cnt, gate, vb

// (Re)allocate the arena so that it holds at least `min_entries`; keeps the
// given-waveform prefix.  Auto mode sizes it from an output estimate, capped
// by the free HBM.
int ensure_arena(gls_ctx* ctx, int64_t min_entries, bool grow_max) {
    int64_t want;
    if (ctx->cfg.arena_bytes > 0) {
        want = ctx->cfg.arena_bytes / 8;
        ctx->arena_auto = false;
    } else {
        ctx->arena_auto = true;
        int64_t per_pi = ctx->P ? std::max<int64_t>(16, ctx->in_total / ctx->P) : 16;
        double est = (double)ctx->in_total + 3.0 * (double)ctx->G * (double)per_pi + 4096.0;
        want = (int64_t)std::min(est, 4e18);
        want = std::max<int64_t>(want, (256ll << 20) / 8);
        int64_t have = (int64_t)ctx->d_arena.n;
        int64_t avail = free_bytes(ctx) + have * 8;
        double per_entry = 8.0 + kChunkBytes * chunk_ratio(ctx);
        int64_t reserve = ((int64_t)ctx->G + ctx->P) * 24 + (256ll << 20);
        int64_t cap = (int64_t)(std::max<int64_t>(0, (int64_t)(avail * 0.90) - reserve) / per_entry);
        if (grow_max || want > cap) want = cap;
    }
    if (want < min_entries) want = min_entries;
    if ((int64_t)ctx->d_arena.n >= want && !grow_max) return GLS_OK;
    if ((int64_t)ctx->d_arena.n == want) return GLS_OK;
    bool keep = ctx->d_arena.p && ctx->has_inputs && ctx->prefix_total > 0;
    if (!keep) ctx->d_arena.release();                 // nothing to copy: free before allocating
    uint64_t* np = nullptr;
    cudaError_t e = cudaMalloc(&np, (size_t)std::max<int64_t>(want, 1) * 8);
    if (e != cudaSuccess && keep) {
        // the old arena (given waveforms in its prefix) leaves too little room: move the
        // prefix through host memory, free the old arena, allocate, copy back
        cudaGetLastError();
        std::vector<uint64_t> host((size_t)ctx->prefix_total);
        e = cudaMemcpy(host.data(), ctx->d_arena.p, (size_t)ctx->prefix_total * 8, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) {
            ctx->d_arena.release();
            keep = false;
            e = cudaMalloc(&np, (size_t)std::max<int64_t>(want, 1) * 8);
            if (e == cudaSuccess) e = cudaMemcpy(np, host.data(), (size_t)ctx->prefix_total * 8, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) {
                cudaGetLastError();
                if (np) cudaFree(np);
                ctx->has_inputs = ctx->has_result = false;   // the given waveforms are gone with the old arena
                return fail(ctx, GLS_ENOMEM, "arena allocation of %lld bytes failed (inputs dropped): %s",
                            (long long)want * 8, cudaGetErrorString(e));
            }
        }
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, GLS_ENOMEM, "arena allocation of %lld bytes failed: %s", (long long)want * 8,
                    cudaGetErrorString(e));
    }
    if (keep) {
        e = cudaMemcpyAsync(np, ctx->d_arena.p, (size_t)ctx->prefix_total * 8, cudaMemcpyDeviceToDevice,
                            ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) {
            cudaFree(np);
            return fail(ctx, GLS_ECUDA, "arena copy: %s", cudaGetErrorString(e));
        }
    }
    ctx->d_arena.release();
    ctx->d_arena.p = np;
    ctx->d_arena.n = (size_t)std::max<int64_t>(want, 1);
    return GLS_OK;
}

int ensure_chunks(gls_ctx* ctx, int64_t min_cap) {
    int64_t want;
    if (ctx->cfg.chunk_capacity > 0) {
        want = ctx->cfg.chunk_capacity;
    } else {
        want = (int64_t)ctx->P + 2ll * ctx->G + (int64_t)(chunk_ratio(ctx) * (double)ctx->d_arena.n) + 1024;
    }
    want = std::max(want, min_cap);
    want = std::max<int64_t>(want, (int64_t)ctx->P + ctx->G + 1);
    if (want >= (1ll << 32)) want = (1ll << 32) - 1;
    if ((int64_t)ctx->d_ck_T.n >= want) return GLS_OK;
    cudaError_t e;
    ctx->last_chunk_top = 0;
    if ((e = ctx->d_ck_T.alloc(want)) != cudaSuccess || (e = ctx->d_ck_off.alloc(want)) != cudaSuccess ||
        (e = ctx->d_ck_cum.alloc(want)) != cudaSuccess || (e = ctx->d_ck_cnt.alloc(want)) != cudaSuccess ||
        (e = ctx->d_ck_gate.alloc(want)) != cudaSuccess || (e = ctx->d_ck_vb.alloc(want)) != cudaSuccess) {
        cudaGetLastError();
        ctx->d_ck_T.release();
        return fail(ctx, GLS_ENOMEM, "chunk table of %lld entries: %s", (long long)want, cudaGetErrorString(e));
    }
    return GLS_OK;
}

}  // namespace

extern "C" {

const char* gls_version(void) { return "gls 0.1 (sm_100a, persistent level-barrier kernel)"; }

const char* gls_last_error(const gls_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int gls_lut_lookup(int type, int arity, const uint8_t* v) {
    if (type < 0 || type >= kNumTypes || !arity_ok(type, arity) || !v) return GLS_EINVAL;
    int idx = 0;
    for (int i = 0; i < arity; ++i) {
        if (v[i] > 3) return GLS_EINVAL;
        int c = v[i] == 3 ? 2 : v[i];  // Z read as X
        idx |= c << (2 * i);
    }
    return lut_table()[lut_offset(type, arity) + idx];
}

int gls_create(gls_ctx** out, int cuda_device, void* cuda_stream) {
    if (!out) return GLS_EINVAL;
    *out = nullptr;
    gls_ctx* ctx = new (std::nothrow) gls_ctx();
    if (!ctx) return GLS_ENOMEM;
    ctx->device = cuda_device;
    ctx->stream = (cudaStream_t)cuda_stream;
    cudaError_t e = cudaSetDevice(cuda_device);
    if (e == cudaSuccess) {
        for (auto& ev : ctx->ev)
            if (e == cudaSuccess) e = cudaEventCreate(&ev);
    }
    if (e == cudaSuccess) e = ctx->d_ctl.alloc(1);
    if (e == cudaSuccess) e = ctx->d_flag.alloc(4);
    if (e == cudaSuccess) e = ctx->d_flag64.alloc(4);
    if (e == cudaSuccess) e = ctx->d_lut.alloc(kLutCap);
    if (e == cudaSuccess)
        e = cudaMemcpy(ctx->d_lut.p, lut_table().data(), kLutCap, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaGetLastError();
        delete ctx;
        return e == cudaErrorMemoryAllocation ? GLS_ENOMEM : GLS_ECUDA;
    }
    *out = ctx;
    return GLS_OK;
}

void gls_destroy(gls_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    for (auto& ev : ctx->ev)
        if (ev) cudaEventDestroy(ev);
    delete ctx;
}

int gls_set_config(gls_ctx* ctx, const gls_config* cfg) {
    if (!ctx || !cfg) return GLS_EINVAL;
    if (cfg->arena_bytes < 0 || cfg->chunk_capacity < 0 || cfg->chunk_events < 0 || cfg->blocks_per_sm < 0 ||
        cfg->ring_limit < 0 || cfg->ring_limit > kRing || cfg->engine < 0 || cfg->engine > 2 ||
        cfg->scheduler < 0 || cfg->scheduler > 1 || cfg->deep_per_warp < 0 || cfg->readback_mib < 0 ||
        cfg->trace < 0 || cfg->trace > 1 || cfg->csrp_pagelen == 1 || cfg->csrp_pagelen < 0)
        return fail(ctx, GLS_EINVAL, "invalid gls_config field");
    ctx->cfg = *cfg;
    ctx->deep_per_warp = 0;                  // re-derived from cfg at the next simulate
    return GLS_OK;
}

}  // extern "C"

// a1 for gates given by arity, LUT base and pin delays (basic gates or expanded cell
// outputs): Kahn order, levels, the fan-in CSR in level order, fan-out lists, halo;
// upload (with the LUT table `lut`, kLutCap bytes).
static int load_gates(gls_ctx* ctx, int32_t P, int32_t G, const uint16_t* lb, const int64_t* off, const int32_t* net,
                      const uint32_t* delay, const std::vector<uint8_t>& lut) {
    const int64_t N = (int64_t)P + G;
    const int64_t E = G > 0 ? off[G] : 0;
    // Kahn topological order; level(g) = 1 + max level of driving gates (PIs at 0)
    std::vector<int32_t> indeg(G, 0), level(G, 0), order;
    std::vector<int64_t> fo_off((size_t)G + 1, 0);
    for (int32_t g = 0; g < G; ++g)
        for (int64_t e = off[g]; e < off[g + 1]; ++e)
            if (net[e] >= P) { ++indeg[g]; ++fo_off[net[e] - P + 1]; }
    for (int32_t g = 0; g < G; ++g) fo_off[g + 1] += fo_off[g];
    std::vector<int32_t> fo((size_t)std::max<int64_t>(fo_off[G], 1));
    {
        std::vector<int64_t> fill(fo_off.begin(), fo_off.end() - 1);
        for (int32_t g = 0; g < G; ++g)
            for (int64_t e = off[g]; e < off[g + 1]; ++e)
                if (net[e] >= P) fo[fill[net[e] - P]++] = g;
    }
    order.reserve(G);
    for (int32_t g = 0; g < G; ++g)
        if (indeg[g] == 0) order.push_back(g);
    for (size_t h = 0; h < order.size(); ++h) {
        int32_t g = order[h];
        for (int64_t q = fo_off[g]; q < fo_off[g + 1]; ++q) {
            int32_t c = fo[q];
            level[c] = std::max(level[c], level[g] + 1);
            if (--indeg[c] == 0) order.push_back(c);
        }
    }
    if ((int64_t)order.size() != G) return fail(ctx, GLS_ECYCLE, "combinational loop: %lld gates on cycles",
                                               (long long)(G - (int64_t)order.size()));
    int32_t L = 0;
    for (int32_t g = 0; g < G; ++g) { level[g] += 1; L = std::max(L, level[g]); }
    // stable counting sort by level -> internal order
    std::vector<int32_t> level_off((size_t)L + 1, 0);
    for (int32_t g = 0; g < G; ++g) ++level_off[level[g]];
    for (int32_t l = 1; l <= L; ++l) level_off[l] += level_off[l - 1];
    std::vector<uint32_t> perm(G), inv(G);
    {
        std::vector<int32_t> fill(level_off.begin(), level_off.end() - 1);
        for (int32_t g = 0; g < G; ++g) {
            int32_t i = fill[level[g] - 1]++;
            perm[i] = (uint32_t)g;
            inv[g] = (uint32_t)i;
        }
    }
    std::vector<GateInfo> ginfo(G);
    std::vector<uint32_t> psrc((size_t)E);
    std::vector<uint4> pdel((size_t)E);
    std::vector<int64_t> fanout((size_t)N, 0);
    std::vector<int64_t> arrive((size_t)N, 0);
    int64_t maxA = 0;
    uint32_t pin = 0;
    for (int32_t i = 0; i < G; ++i) {
        int32_t g = (int32_t)perm[i];
        int k = (int)(off[g + 1] - off[g]);
        ginfo[i].pin_off = pin;
        ginfo[i].k = (uint8_t)k;
        ginfo[i].lut_base = lb[g];
        ginfo[i].flags = 0;
        uint32_t dmax = 0;
        int64_t a = 0;
        for (int q = 0; q < k; ++q) {
            int64_t e = off[g] + q;
            int32_t s = net[e];
            uint32_t si = s < P ? (uint32_t)s : (uint32_t)(P + inv[s - P]);
            psrc[pin] = si;
            pdel[pin] = make_uint4(delay[4 * e], delay[4 * e + 1], delay[4 * e + 2], delay[4 * e + 3]);
            for (int d = 0; d < 4; ++d) {
                if (delay[4 * e + d] != kDelayInf) dmax = std::max(dmax, delay[4 * e + d]);   // halo: finite delays
                else ginfo[i].flags |= kGateInf;
            }
            ++fanout[si];
            a = std::max(a, arrive[si]);
            ++pin;
        }
        arrive[P + i] = a + dmax;
        maxA = std::max(maxA, arrive[P + i]);
    }
    // consumers of every internal net (gates only) and initial ready counters
    std::vector<uint32_t> nfo_off((size_t)N + 1, 0), pend0((size_t)std::max<int32_t>(G, 1), 0);
    for (uint32_t q = 0; q < (uint32_t)E; ++q) ++nfo_off[psrc[q] + 1];
    for (int64_t n = 0; n < N; ++n) nfo_off[n + 1] += nfo_off[n];
    std::vector<uint32_t> nfo_gate((size_t)std::max<int64_t>(E, 1));
    {
        std::vector<uint32_t> fill(nfo_off.begin(), nfo_off.end() - 1);
        for (int32_t i = 0; i < G; ++i)
            for (uint32_t q = ginfo[i].pin_off; q < ginfo[i].pin_off + ginfo[i].k; ++q) {
                nfo_gate[fill[psrc[q]]++] = (uint32_t)i;
                if (psrc[q] >= (uint32_t)P) ++pend0[i];
            }
    }
    // upload
    cudaSetDevice(ctx->device);
    ctx->has_netlist = ctx->has_inputs = ctx->has_result = false;
    CK(ctx->d_level_off.alloc(L + 1));
    CK(ctx->d_gate.alloc(G));
    CK(ctx->d_pin_src.alloc(E));
    CK(ctx->d_pin_delay.alloc(E));
    CK(ctx->d_perm.alloc(G));
    CK(ctx->d_net_ck.alloc(N));
    CK(ctx->d_net_nck.alloc(N));
    CK(ctx->d_net_len.alloc(N));
    CK(ctx->d_gate_done.alloc(G));
    CK(ctx->d_gate_nin.alloc(G));
    CK(ctx->d_work.alloc(L + 1));
    CK(ctx->d_fo_off.alloc(N + 1));
    CK(ctx->d_fo_gate.alloc(std::max<int64_t>(E, 1)));
    CK(ctx->d_pend0.alloc(G));
    CK(ctx->d_pend.alloc(G));
    CK(cudaMemcpy(ctx->d_fo_off.p, nfo_off.data(), sizeof(uint32_t) * (N + 1), cudaMemcpyHostToDevice));
    if (E) CK(cudaMemcpy(ctx->d_fo_gate.p, nfo_gate.data(), sizeof(uint32_t) * E, cudaMemcpyHostToDevice));
    if (G) CK(cudaMemcpy(ctx->d_pend0.p, pend0.data(), sizeof(uint32_t) * G, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_level_off.p, level_off.data(), sizeof(int32_t) * (L + 1), cudaMemcpyHostToDevice));
    if (G) {
        CK(cudaMemcpy(ctx->d_gate.p, ginfo.data(), sizeof(GateInfo) * G, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->d_perm.p, perm.data(), sizeof(uint32_t) * G, cudaMemcpyHostToDevice));
        CK(ctx->d_inv.alloc(G));
        CK(cudaMemcpy(ctx->d_inv.p, inv.data(), sizeof(uint32_t) * G, cudaMemcpyHostToDevice));
    }
    if (E) {
        CK(cudaMemcpy(ctx->d_pin_src.p, psrc.data(), sizeof(uint32_t) * E, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->d_pin_delay.p, pdel.data(), sizeof(uint4) * E, cudaMemcpyHostToDevice));
    }
    {
        std::vector<uint32_t> fo32(fanout.begin(), fanout.end());
        CK(ctx->d_fanout.alloc(fo32.size()));
        if (!fo32.empty())
            CK(cudaMemcpy(ctx->d_fanout.p, fo32.data(), sizeof(uint32_t) * fo32.size(), cudaMemcpyHostToDevice));
    }
    ctx->P = P;
    ctx->G = G;
    ctx->L = L;
    ctx->E = E;
    ctx->halo = maxA + 1;
    ctx->has_inf = false;
    for (int32_t i = 0; i < G; ++i) ctx->has_inf = ctx->has_inf || (ginfo[i].flags & kGateInf);
    ctx->perm.swap(perm);
    ctx->inv.swap(inv);
    ctx->net_fanout.swap(fanout);
    CK(cudaMemcpy(ctx->d_lut.p, lut.data(), kLutCap, cudaMemcpyHostToDevice));
    ctx->has_netlist = true;
    return GLS_OK;
}


extern "C" {

int gls_load_netlist(gls_ctx* ctx, int32_t P, int32_t G, const uint8_t* type, const int64_t* off,
                     const int32_t* net, const uint32_t* delay) {
    if (!ctx) return GLS_EINVAL;
    if (P < 0 || G < 0 || (int64_t)P + G >= (1ll << 31)) return fail(ctx, GLS_EINVAL, "bad net counts");
    if (G > 0 && (!type || !off)) return fail(ctx, GLS_EINVAL, "null netlist array");
    const int64_t N = (int64_t)P + G;
    const int64_t E = G > 0 ? off[G] : 0;
    if (G > 0 && off[0] != 0) return fail(ctx, GLS_EINVAL, "fanin_offsets[0] != 0");
    if (E < 0 || E >= (1ll << 31)) return fail(ctx, GLS_EINVAL, "pin count out of range");
    if (E > 0 && (!net || !delay)) return fail(ctx, GLS_EINVAL, "null pin array");
    for (int32_t g = 0; g < G; ++g) {
        int64_t k = off[g + 1] - off[g];
        if (type[g] >= kNumTypes) return fail(ctx, GLS_EINVAL, "gate %d: unknown type %d", g, (int)type[g]);
        if (!arity_ok(type[g], k)) return fail(ctx, GLS_EINVAL, "gate %d: arity %lld invalid", g, (long long)k);
        for (int64_t e = off[g]; e < off[g + 1]; ++e) {
            if (net[e] < 0 || net[e] >= N) return fail(ctx, GLS_EINVAL, "gate %d: net id %d out of range", g, net[e]);
            for (int q = 0; q < 4; ++q)
                if (delay[4 * e + q] >= (1u << 31) && delay[4 * e + q] != kDelayInf)
                    return fail(ctx, GLS_EINVAL, "pin %lld: delay >= 2^31 (and not GLS_DELAY_INF)", (long long)e);
        }
    }
    std::vector<uint16_t> lb((size_t)std::max<int32_t>(G, 1));
    for (int32_t g = 0; g < G; ++g) lb[g] = (uint16_t)lut_offset(type[g], (int)(off[g + 1] - off[g]));
    return load_gates(ctx, P, G, lb.data(), off, net, delay, lut_table());
}

// Multi-output cells (§3.2 Delay P:329-333, §3.3 Module Function P:335-339): every
// template output is a function of the cell's inputs composed of basic gates (the
// library's own dual-rail evaluation, lut_eval), tabulated once per distinct function
// (a basic gate's table when it is one, else a table in the cell area of the LUT); each
// cell output becomes a gate with the cell's input pins and its own slice of the 5-D
// delay matrix (GLS_DELAY_INF: no relation, reading R9).
int gls_load_cells(gls_ctx* ctx, int32_t P, int32_t T, const gls_cell_template* tpl, int32_t C,
                   const int32_t* cell_tpl, const int32_t* cell_fanin, const uint32_t* cell_delay) {
    if (!ctx) return GLS_EINVAL;
    if (P < 0 || T < 0 || C < 0) return fail(ctx, GLS_EINVAL, "bad counts");
    if ((T > 0 && !tpl) || (C > 0 && (!cell_tpl || !cell_fanin || !cell_delay)))
        return fail(ctx, GLS_EINVAL, "null cell array");
    std::vector<uint8_t> lut = lut_table();
    int used = kLutBytes;
    std::vector<std::vector<uint16_t>> out_lb((size_t)T);
    for (int32_t i = 0; i < T; ++i) {
        const gls_cell_template& t = tpl[i];
        if (t.num_inputs < 1 || t.num_inputs > 4 || t.num_outputs < 1 || t.num_outputs > 8 || t.num_gates < 0 ||
            t.num_gates > 64 || (t.num_gates > 0 && (!t.gate_type || !t.gate_fanin_offsets || !t.gate_fanin)) ||
            !t.output_node)
            return fail(ctx, GLS_EINVAL, "template %d: bad shape", i);
        for (int j = 0; j < t.num_gates; ++j) {
            const int64_t k = t.gate_fanin_offsets[j + 1] - t.gate_fanin_offsets[j];
            if (t.gate_type[j] >= kNumTypes || !arity_ok(t.gate_type[j], k))
                return fail(ctx, GLS_EINVAL, "template %d gate %d: type / arity", i, j);
            for (int64_t q = t.gate_fanin_offsets[j]; q < t.gate_fanin_offsets[j + 1]; ++q)
                if (t.gate_fanin[q] < 0 || t.gate_fanin[q] >= t.num_inputs + j)
                    return fail(ctx, GLS_EINVAL, "template %d gate %d: node %d (not an earlier node)", i, j, t.gate_fanin[q]);
        }
        for (int q = 0; q < t.num_outputs; ++q)
            if (t.output_node[q] < 0 || t.output_node[q] >= t.num_inputs + t.num_gates)
                return fail(ctx, GLS_EINVAL, "template %d output %d: node out of range", i, q);
        const int k = t.num_inputs, n = 1 << (2 * k);
        for (int q = 0; q < t.num_outputs; ++q) {
            std::vector<uint8_t> tab((size_t)n, 2);
            for (int idx = 0; idx < n; ++idx) {
                int node[4 + 64];
                bool valid = true;
                for (int a = 0; a < k; ++a) {
                    node[a] = (idx >> (2 * a)) & 3;
                    if (node[a] == 3) valid = false;   // the kernel indexes normalised codes
                }
                if (!valid) continue;
                for (int j = 0; j < t.num_gates; ++j) {
                    int v[4];
                    const int32_t f0 = t.gate_fanin_offsets[j];
                    const int kk = (int)(t.gate_fanin_offsets[j + 1] - f0);
                    for (int a = 0; a < kk; ++a) v[a] = node[t.gate_fanin[f0 + a]];
                    node[k + j] = lut_eval(t.gate_type[j], kk, v);
                }
                const int o = node[t.output_node[q]];
                tab[(size_t)idx] = (uint8_t)(o == 3 ? 2 : o);
            }
            // a basic gate's table, an earlier cell table, or a new one
            int base = -1;
            for (int ty = 0; ty < kNumTypes && base < 0; ++ty)
                if (arity_ok(ty, k) && std::equal(tab.begin(), tab.end(), lut.begin() + lut_offset(ty, k)))
                    base = lut_offset(ty, k);
            for (int b0 = kLutBytes; base < 0 && b0 + n <= used; ++b0)
                if (std::equal(tab.begin(), tab.end(), lut.begin() + b0)) base = b0;
            if (base < 0) {
                if (used + n > kLutCap)
                    return fail(ctx, GLS_EINVAL, "cell output functions need more than the %d-byte LUT area", kLutCap - kLutBytes);
                std::copy(tab.begin(), tab.end(), lut.begin() + used);
                base = used;
                used += n;
            }
            out_lb[(size_t)i].push_back((uint16_t)base);
        }
    }
    // expand: cell c's output q is gate (first[c] + q), net P + first[c] + q
    int64_t G = 0, pins = 0, dl = 0;
    for (int32_t c = 0; c < C; ++c) {
        if (cell_tpl[c] < 0 || cell_tpl[c] >= T) return fail(ctx, GLS_EINVAL, "cell %d: template id", c);
        G += tpl[cell_tpl[c]].num_outputs;
    }
    if ((int64_t)P + G >= (1ll << 31)) return fail(ctx, GLS_EINVAL, "bad net counts");
    const int64_t N = (int64_t)P + G;
    std::vector<uint16_t> lb((size_t)std::max<int64_t>(G, 1));
    std::vector<int64_t> off((size_t)G + 1, 0);
    std::vector<int32_t> net;
    std::vector<uint32_t> delay;
    int64_t g = 0;
    for (int32_t c = 0; c < C; ++c) {
        const gls_cell_template& t = tpl[cell_tpl[c]];
        for (int a = 0; a < t.num_inputs; ++a)
            if (cell_fanin[pins + a] < 0 || cell_fanin[pins + a] >= N)
                return fail(ctx, GLS_EINVAL, "cell %d: net id %d out of range", c, cell_fanin[pins + a]);
        for (int q = 0; q < t.num_outputs; ++q, ++g) {
            lb[(size_t)g] = out_lb[(size_t)cell_tpl[c]][(size_t)q];
            for (int a = 0; a < t.num_inputs; ++a) {
                net.push_back(cell_fanin[pins + a]);
                for (int e = 0; e < 4; ++e) {           // [in][out][edge][value] -> pin (rise0, rise1, fall0, fall1)
                    const uint32_t d = cell_delay[dl + ((int64_t)a * t.num_outputs + q) * 4 + e];
                    if (d >= (1u << 31) && d != kDelayInf)
                        return fail(ctx, GLS_EINVAL, "cell %d: delay >= 2^31 (and not GLS_DELAY_INF)", c);
                    delay.push_back(d);
                }
            }
            off[(size_t)g + 1] = (int64_t)net.size();
        }
        pins += t.num_inputs;
        dl += (int64_t)t.num_inputs * t.num_outputs * 4;
    }
    if ((int64_t)net.size() >= (1ll << 31)) return fail(ctx, GLS_EINVAL, "pin count out of range");
    return load_gates(ctx, P, (int32_t)G, lb.data(), off.data(), net.data(), delay.data(), lut);
}

static int set_inputs_common(gls_ctx* ctx, int32_t P, int64_t total) {
    if (!ctx->has_netlist) return fail(ctx, GLS_ESTATE, "gls_set_input_waveforms before gls_load_netlist");
    if (P != ctx->P) return fail(ctx, GLS_ESTATE, "num_inputs %d != netlist's %d", P, ctx->P);
    if (total < 0) return fail(ctx, GLS_EINVAL, "negative total");
    return GLS_OK;
}

// The per-transition rules (a2) checked on the device, on a copy that is not yet the
// context's: host inputs are uploaded to a staging buffer (device inputs are checked in
// place), and only a valid stimulus replaces the given waveforms in the arena prefix — a
// rejected one leaves the previous inputs and result untouched (gls.h conventions).  If
// the staging buffer cannot be allocated (HBM taken by the arena), the host inputs go
// straight into the arena prefix and a rejected stimulus leaves no inputs (GLS_ESTATE at
// the next simulate; stated in gls.h).
static int upload_and_validate(gls_ctx* ctx, int32_t P, const int64_t* off, const uint64_t* tr, int64_t total,
                               cudaMemcpyKind kind) {
    DevBuf<long long> st_off;
    DevBuf<uint64_t> st_tr;
    const long long* v_off = (const long long*)off;     // what is validated (device)
    const uint64_t* v_tr = tr;
    bool in_place = false, staged_in_arena = false;
    if (kind == cudaMemcpyHostToDevice) {
        CK(st_off.alloc((size_t)P + 1));
        CK(cudaMemcpyAsync(st_off.p, off, sizeof(int64_t) * (P + 1), kind, ctx->stream));
        v_off = st_off.p;
        // staging room inside the arena, past everything the context still owns (given
        // waveforms and the last result) and past where the new ones will go: no cudaMalloc /
        // cudaFree of a stimulus-sized buffer per call
        const int64_t owned = std::max<int64_t>(ctx->prefix_total, ctx->has_result ? (int64_t)ctx->last.arena_top : 0);
        const int64_t at = (std::max<int64_t>(owned, total) + 15) & ~15ll;
        if (total && ctx->d_arena.p && ctx->cfg.engine != 2 && at + total <= (int64_t)ctx->d_arena.n) {
            CK(cudaMemcpyAsync(ctx->d_arena.p + at, tr, sizeof(uint64_t) * total, kind, ctx->stream));
            v_tr = ctx->d_arena.p + at;
            staged_in_arena = true;
        } else if (total) {
            if (st_tr.alloc((size_t)total) != cudaSuccess) {
                cudaGetLastError();
                in_place = true;                        // no room for a staging copy
            } else {
                CK(cudaMemcpyAsync(st_tr.p, tr, sizeof(uint64_t) * total, kind, ctx->stream));
                v_tr = st_tr.p;
            }
        }
    }
    if (in_place) {
        ctx->has_inputs = ctx->has_result = false;
        ctx->window_active = false;
        ctx->prefix_total = 0;
        int rc = ensure_arena(ctx, total + 1, false);
        if (rc) return rc;
        CK(cudaMemcpyAsync(ctx->d_arena.p, tr, sizeof(uint64_t) * total, kind, ctx->stream));
        v_tr = ctx->d_arena.p;
    }
    CK(cudaMemsetAsync(ctx->d_flag.p, 0, sizeof(unsigned) * 4, ctx->stream));
    CK(cudaMemsetAsync(ctx->d_flag64.p, 0, sizeof(unsigned long long) * 4, ctx->stream));
    CK(launch_validate_inputs(P, v_off, v_tr, total, ctx->d_flag.p, ctx->d_flag64.p, ctx->stream));
    unsigned err = 0;
    unsigned long long mt = 0;
    long long last_off = 0;
    CK(cudaMemcpyAsync(&err, ctx->d_flag.p, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(&mt, ctx->d_flag64.p, sizeof(mt), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(&last_off, v_off + P, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (err || last_off != total)
        return fail(ctx, GLS_EINVAL,
                    "given waveforms invalid (%s%s%s)", (err & 1u) ? "bad offsets " : "",
                    (err & 2u) ? "times not strictly increasing / value repeats the previous one (first X) / time >= 2^61 " : "",
                    last_off != total ? "offsets[P] != total" : "");
    // valid: it becomes the context's stimulus (arena prefix + offsets)
    if (!in_place) {
        ctx->has_inputs = ctx->has_result = false;
        ctx->window_active = false;
        ctx->prefix_total = 0;                          // nothing to keep while the arena is (re)sized
        if (!staged_in_arena) {                         // (staged in the arena: it already holds 2 x total)
            int rc = ensure_arena(ctx, total + 1, false);
            if (rc) return rc;
        }
        if (total) CK(cudaMemcpyAsync(ctx->d_arena.p, v_tr, sizeof(uint64_t) * total, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    CK(ctx->d_in_off.ensure((size_t)P + 1));
    CK(cudaMemcpyAsync(ctx->d_in_off.p, v_off, sizeof(int64_t) * (P + 1), cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->in_total = total;
    ctx->max_in_time = total ? (int64_t)mt : -1;
    ctx->prefix_total = total;
    ctx->has_inputs = true;
    return GLS_OK;
}

int gls_set_input_waveforms(gls_ctx* ctx, int32_t P, const int64_t* offsets, const uint64_t* tr) {
    if (!ctx) return GLS_EINVAL;
    if (!offsets) return fail(ctx, GLS_EINVAL, "null offsets");
    int rc = set_inputs_common(ctx, P, 0);
    if (rc) return rc;
    const int64_t total = offsets[P];
    if (offsets[0] != 0) return fail(ctx, GLS_EINVAL, "offsets[0] != 0");
    for (int32_t i = 0; i < P; ++i)
        if (offsets[i + 1] < offsets[i]) return fail(ctx, GLS_EINVAL, "offsets decrease at net %d", i);
    if (total > 0 && !tr) return fail(ctx, GLS_EINVAL, "null transitions");
    // one H2D of the packed CSR ("one round of data transfer"), then the
    // per-transition rules are checked on the device
    return upload_and_validate(ctx, P, offsets, tr, total, cudaMemcpyHostToDevice);
}

int gls_set_input_waveforms_device(gls_ctx* ctx, int32_t P, const int64_t* d_off, const uint64_t* d_tr,
                                   int64_t total) {
    if (!ctx) return GLS_EINVAL;
    int rc = set_inputs_common(ctx, P, total);
    if (rc) return rc;
    if (!d_off || (total > 0 && !d_tr)) return fail(ctx, GLS_EINVAL, "null device pointer");
    return upload_and_validate(ctx, P, d_off, d_tr, total, cudaMemcpyDeviceToDevice);
}

static int simulate_run(gls_ctx* ctx, int64_t duration);

static int check_run(gls_ctx* ctx, int64_t duration) {
    if (!ctx->has_netlist) return fail(ctx, GLS_ESTATE, "gls_simulate before gls_load_netlist");
    if (!ctx->has_inputs) return fail(ctx, GLS_ESTATE, "gls_simulate before gls_set_input_waveforms");
    if (duration < 0 || duration >= (1ll << 61)) return fail(ctx, GLS_ERANGE, "duration out of range");
    if (ctx->max_in_time > duration)
        return fail(ctx, GLS_ERANGE, "a given transition at %lld ps is later than the duration %lld ps",
                    (long long)ctx->max_in_time, (long long)duration);
    return GLS_OK;
}

int gls_simulate(gls_ctx* ctx, int64_t duration) {
    if (!ctx) return GLS_EINVAL;
    int rc = check_run(ctx, duration);
    if (rc) return rc;
    ctx->window_active = false;                        // the full given waveforms
    ctx->prefix_total = ctx->in_total;
    return simulate_run(ctx, duration);
}

int gls_simulate_window(gls_ctx* ctx, int64_t t_begin, int64_t t_end, int64_t duration) {
    if (!ctx) return GLS_EINVAL;
    int rc = check_run(ctx, duration);
    if (rc) return rc;
    if (t_begin < 0 || t_end < t_begin) return fail(ctx, GLS_EINVAL, "window [%lld, %lld) invalid",
                                                    (long long)t_begin, (long long)t_end);
    if (ctx->has_inf && t_begin > 0)
        return fail(ctx, GLS_EINVAL, "time windows need finite delays: with GLS_DELAY_INF an output keeps a value "
                                     "from before any halo (reading R9)");
    cudaSetDevice(ctx->device);
    ctx->has_result = false;
    ctx->window_active = false;
    ctx->prefix_total = ctx->in_total;
    const int32_t P = ctx->P;
    const long long t_clamp = t_begin - ctx->halo;     // reading R17
    // per-net slice sizes -> offsets (after the full inputs, 128-byte aligned)
    DevBuf<long long> d_cnt;
    CK(d_cnt.alloc((size_t)P + 1));
    CK(launch_window_count(P, ctx->d_in_off.p, ctx->d_arena.p, t_clamp, t_end, d_cnt.p, ctx->stream));
    std::vector<long long> cnt((size_t)P + 1, 0), off((size_t)P + 1, 0);
    if (P) CK(cudaMemcpyAsync(cnt.data(), d_cnt.p, sizeof(long long) * P, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    const long long base = (ctx->in_total + 15) & ~15ll;
    off[0] = base;
    for (int32_t i = 0; i < P; ++i) off[i + 1] = off[i] + cnt[i];
    const int64_t total_w = off[P] - base;
    rc = ensure_arena(ctx, base + total_w + 1, false);  // keeps the full inputs
    if (rc) return rc;
    CK(ctx->d_win_off.ensure((size_t)P + 1));
    CK(cudaMemcpyAsync(ctx->d_win_off.p, off.data(), sizeof(long long) * (P + 1), cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(launch_window_fill(P, ctx->d_in_off.p, ctx->d_arena.p, t_clamp, t_end, ctx->d_win_off.p, ctx->d_arena.p,
                          ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->window_active = true;
    ctx->prefix_total = base + total_w;
    const int64_t sim = std::max<int64_t>(0, std::min<int64_t>(duration, t_end - 1));
    return simulate_run(ctx, sim);
}

static int simulate_csrp(gls_ctx* ctx, int64_t duration);

static int simulate_run(gls_ctx* ctx, int64_t duration) {
    cudaSetDevice(ctx->device);
    ctx->has_result = false;
    ctx->duration = duration;
    if (ctx->cfg.engine == 2) return simulate_csrp(ctx, duration);
    int rc = ensure_chunks(ctx, 0);
    if (rc) return rc;
    int per_sm = 0;
    const int sched = (ctx->cfg.engine == 1 || ctx->cfg.scheduler == 1) ? 1 : 0;
    int maxb = max_coresident_blocks(ctx->device, ctx->cfg.engine, sched, &per_sm);
    int sms = per_sm ? maxb / per_sm : 0;
    int blocks = ctx->cfg.blocks_per_sm > 0 ? std::min(maxb, ctx->cfg.blocks_per_sm * sms) : maxb;
    if (blocks < 1) return fail(ctx, GLS_ECUDA, "simulation kernel cannot be resident (occupancy 0)");
    if (ctx->cfg.engine == 0) {     // engine 0's lane scratch and per-warp unit fields
        if (ctx->d_wscr.n < warp_scratch_entries(blocks)) CK(ctx->d_wscr.alloc(warp_scratch_entries(blocks)));
        if (ctx->d_waux.n < warp_aux_bytes(blocks)) CK(ctx->d_waux.alloc(warp_aux_bytes(blocks)));
    }
    const int64_t nwarps = (int64_t)blocks * (kThreads / 32);
    if (ctx->deep_per_warp == 0) ctx->deep_per_warp = ctx->cfg.deep_per_warp > 0 ? ctx->cfg.deep_per_warp : (1 << 16);
    if ((int64_t)ctx->d_deep.n != nwarps * ctx->deep_per_warp) CK(ctx->d_deep.alloc(nwarps * ctx->deep_per_warp));
    if ((int64_t)ctx->d_deep_wtop.n < nwarps) CK(ctx->d_deep_wtop.alloc(nwarps));

    for (int attempt = 0; attempt < 3; ++attempt) {
        SimParams p = params(ctx);
        Ctl init{};
        init.chunk_top = (unsigned long long)ctx->P;
        init.work_head = (unsigned long long)ctx->P;
        init.arena_top = (unsigned long long)((ctx->prefix_total + 15) & ~15ll);   // 128-byte segments
        CK(cudaEventRecord(ctx->ev[0], ctx->stream));
        if (ctx->cfg.trace) {
            CK(ctx->d_trace.ensure((size_t)8 * std::max<int32_t>(ctx->G, 1)));
            CK(cudaMemsetAsync(ctx->d_trace.p, 0, sizeof(unsigned long long) * 8 * std::max<int32_t>(ctx->G, 1),
                               ctx->stream));
            p.trace = ctx->d_trace.p;
        }
        ctx->traced = ctx->cfg.trace != 0;
        CK(cudaMemcpyAsync(ctx->d_ctl.p, &init, sizeof(Ctl), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemsetAsync(ctx->d_work.p, 0, sizeof(unsigned long long) * (ctx->L + 1), ctx->stream));
        if (ctx->G > 0) {
            CK(cudaMemcpyAsync(ctx->d_pend.p, ctx->d_pend0.p, sizeof(uint32_t) * ctx->G, cudaMemcpyDeviceToDevice,
                               ctx->stream));
            // chunk ids not yet planned read as empty (0xffffffff): clear what the last run used
            const size_t clear = ctx->last_chunk_top > 0
                                     ? std::min<size_t>(ctx->d_ck_gate.n, (size_t)ctx->last_chunk_top)
                                     : ctx->d_ck_gate.n;
            CK(cudaMemsetAsync(ctx->d_ck_gate.p, 0xff, sizeof(uint32_t) * clear, ctx->stream));
        }
        CK(launch_init_given(p, ctx->window_active ? ctx->d_win_off.p : ctx->d_in_off.p, ctx->stream));
        CK(cudaEventRecord(ctx->ev[1], ctx->stream));
        if (ctx->G > 0) CK(launch_simulate(p, blocks, ctx->stream));
        CK(cudaEventRecord(ctx->ev[2], ctx->stream));
        CK(cudaMemcpyAsync(&ctx->last, ctx->d_ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        const Ctl& c = ctx->last;
        ctx->last_chunk_top = std::max<unsigned long long>(c.chunk_top, ctx->last_chunk_top);
        if (c.error & kErrWatchdog)
            return fail(ctx, GLS_ECUDA, "dataflow scheduler watchdog: no gate completed for 10 s (%llu of %d done)",
                        c.done_gates, ctx->G);
        if (c.error & (kErrArena | kErrChunks | kErrDeep)) {
            // grow what overflowed and retry (auto sizing), else report what is needed
            bool retried = false;
            if ((c.error & kErrDeep)) {
                ctx->deep_per_warp = std::max<int64_t>(ctx->deep_per_warp * 2, (int64_t)c.need_deep * 2);
                CK(ctx->d_deep.alloc(nwarps * ctx->deep_per_warp));
                retried = true;
            }
            if ((c.error & kErrChunks)) {
                if (ctx->cfg.chunk_capacity > 0)
                    return fail(ctx, GLS_ENOMEM, "chunk table too small: %llu entries needed at the failing level (capacity %zu)",
                                c.need_chunks, ctx->d_ck_T.n);
                ctx->d_ck_T.release();
                rc = ensure_chunks(ctx, (int64_t)(c.need_chunks * 2));
                if (rc) return rc;
                retried = true;
            }
            if ((c.error & kErrArena)) {
                if (!ctx->arena_auto || attempt > 0)
                    return fail(ctx, GLS_ENOMEM,
                                "arena too small: more than %llu bytes needed (arena %zu bytes); set gls_config.arena_bytes",
                                c.need_arena * 8ull, ctx->d_arena.n * 8);
                rc = ensure_arena(ctx, (int64_t)c.need_arena, true);
                if (rc) return rc;
                ctx->d_ck_T.release();
                rc = ensure_chunks(ctx, 0);
                if (rc) return rc;
                retried = true;
            }
            if (retried) continue;
        }
        if (c.error & kErrBug) return fail(ctx, GLS_ECUDA, "internal consistency check failed (pass counts differ)");
        // success
        float ms_k = 0, ms_s = 0;
        cudaEventElapsedTime(&ms_k, ctx->ev[1], ctx->ev[2]);
        cudaEventElapsedTime(&ms_s, ctx->ev[0], ctx->ev[2]);
        gls_stats& s = ctx->stats;
        s = gls_stats{};
        s.gate_evals = (int64_t)c.gate_evals;
        s.events = (int64_t)c.events;
        s.out_transitions = (int64_t)c.out_trans;
        s.chunks = (int64_t)c.chunks;
        s.deep_chunks = (int64_t)c.deep_chunks;
        s.levels = ctx->L;
        s.arena_used_bytes = (int64_t)c.arena_top * 8;
        s.kernel_ms = ms_k;
        s.lane_utilization = c.warp_iters ? (double)c.lane_iters / (double)c.warp_iters : 0.0;
        s.batches = (int64_t)c.batches;
        s.batch_lanes = c.batches ? (double)c.batch_lanes / (double)c.batches : 0.0;
        s.batch_est = c.batches ? (double)c.batch_est / (double)c.batches : 0.0;
        for (int q = 0; q < 6; ++q) s.phase_cycles[q] = (double)c.cyc[q];
        for (int q = 0; q < 8; ++q) s.balance[q] = (double)c.bal[q];
        s.simulate_ms = ms_s;
        s.alg_bytes = -1;  // computed on demand by gls_get_stats
        ctx->has_result = true;
        return GLS_OK;
    }
    return fail(ctx, GLS_ENOMEM, "simulation did not fit after resizing");
}


// Engine 2 (NEXT-3): the paper's CSRP store and Alg. 1 (gls_csrp.cuh) — given waveforms
// copied into pages, one cooperative launch, then the pages of every gate output collected
// into exact arena segments (one chunk per net) for the library's readers.
static int simulate_csrp(gls_ctx* ctx, int64_t duration) {
    const int32_t P = ctx->P, G = ctx->G;
    const int64_t N = (int64_t)P + G;
    const uint32_t L = ctx->cfg.csrp_pagelen > 0 ? (uint32_t)ctx->cfg.csrp_pagelen : 256u;
    int rc = ensure_chunks(ctx, 0);
    if (rc) return rc;
    const int threads = csrp_coresident_threads(ctx->device);
    if (threads < 1) return fail(ctx, GLS_ECUDA, "CSRP kernel cannot be resident");
    if (ctx->d_wscr.n < csrp_scratch_entries(threads)) CK(ctx->d_wscr.alloc(csrp_scratch_entries(threads)));
    // pages: the arena's room for outputs plus the given waveforms, and one page per waveform
    // of slack (Eq. 4's waste bound)
    const int64_t room = (int64_t)ctx->d_arena.n - ctx->prefix_total;
    int64_t want = (ctx->prefix_total + std::max<int64_t>(room, 0)) / (int64_t)(L - 1) + 2 * N + 16;
    const int64_t fit = (int64_t)(0.45 * (double)free_bytes(ctx)) / (8 * (int64_t)L);
    want = std::max<int64_t>(16, std::min(want, fit));
    if ((int64_t)ctx->d_pages.n < want * (int64_t)L) CK(ctx->d_pages.alloc((size_t)want * L));
    CK(ctx->d_first_page.ensure((size_t)N + 1));
    CK(ctx->d_out_cnt.ensure((size_t)N + 1));
    CK(ctx->d_known.ensure((size_t)std::max<int32_t>(G, 1)));
    CK(ctx->d_seg_off.ensure((size_t)std::max<int32_t>(G, 1)));
    const bool auto_size = ctx->cfg.arena_bytes == 0;
    Ctl init{};
    unsigned long long top = 0, pages_used = 0;
    std::vector<unsigned long long> cnt((size_t)std::max<int32_t>(G, 1)), off((size_t)std::max<int32_t>(G, 1));
    // (auto-sized store: a full page store grows once to the largest that fits, and the arena
    // to what the collected result needs, then the run is repeated)
    for (int attempt = 0;; ++attempt) {
    const unsigned long long page_cap = ctx->d_pages.n / L;
    SimParams p = params(ctx);
    init = Ctl{};
    init.chunk_top = (unsigned long long)N;
    init.arena_top = (unsigned long long)((ctx->prefix_total + 15) & ~15ll);
    CK(cudaEventRecord(ctx->ev[0], ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_ctl.p, &init, sizeof(Ctl), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(ctx->d_known.p, 0, sizeof(uint32_t) * std::max<int32_t>(G, 1), ctx->stream));
    CK(cudaMemsetAsync(ctx->d_flag64.p, 0, sizeof(unsigned long long), ctx->stream));     // page iterator
    const long long* in_off = ctx->window_active ? ctx->d_win_off.p : ctx->d_in_off.p;
    CK(launch_init_given(p, in_off, ctx->stream));
    CK(cudaEventRecord(ctx->ev[1], ctx->stream));
    CK(launch_csrp(p, ctx->d_pages.p, ctx->d_flag64.p, page_cap, L, ctx->d_first_page.p, ctx->d_known.p,
                   ctx->d_out_cnt.p, in_off, threads, ctx->stream));
    CK(cudaEventRecord(ctx->ev[2], ctx->stream));
    CK(cudaMemcpyAsync(&ctx->last, ctx->d_ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(&pages_used, ctx->d_flag64.p, sizeof(pages_used), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    const Ctl& c = ctx->last;
    if (c.error & kErrDeep) return fail(ctx, GLS_ECUDA, "CSRP engine: a thread's individual memory overflowed");
    if (c.error & kErrArena) {
        if (auto_size && attempt == 0) {
            const int64_t most = (int64_t)(0.45 * (double)(free_bytes(ctx) + 8 * ctx->d_pages.n)) / (8 * (int64_t)L);
            if (most > (int64_t)page_cap) {
                ctx->d_pages.release();
                CK(ctx->d_pages.alloc((size_t)most * L));
                continue;
            }
        }
        return fail(ctx, GLS_ENOMEM, "CSRP store full: %llu pages of %u entries (raise the arena)", page_cap, L);
    }
    // exact segments for the gate outputs, in net order after the given waveforms
    if (G) CK(cudaMemcpy(cnt.data(), ctx->d_out_cnt.p + P, sizeof(unsigned long long) * G, cudaMemcpyDeviceToHost));
    top = init.arena_top;
    for (int32_t g = 0; g < G; ++g) {
        off[g] = top;
        top += (cnt[g] + 15) & ~15ull;
    }
    if (top > ctx->d_arena.n) {
        if (auto_size && attempt < 2) {
            const int rc2 = ensure_arena(ctx, (int64_t)top + 1, false);
            if (rc2) return rc2;
            continue;                                  // (pages are intact, but re-run: simplest exact path)
        }
        return fail(ctx, GLS_ENOMEM, "arena too small for the collected result: %llu bytes", top * 8ull);
    }
    break;
    }
    SimParams p = params(ctx);
    const Ctl& c = ctx->last;
    if (G) CK(cudaMemcpyAsync(ctx->d_seg_off.p, off.data(), sizeof(unsigned long long) * G, cudaMemcpyHostToDevice,
                              ctx->stream));
    CK(launch_csrp_collect(p, ctx->d_pages.p, L, ctx->d_first_page.p, ctx->d_out_cnt.p, ctx->d_seg_off.p,
                           ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    float ms_k = 0, ms_s = 0;
    cudaEventElapsedTime(&ms_k, ctx->ev[1], ctx->ev[2]);
    cudaEventElapsedTime(&ms_s, ctx->ev[0], ctx->ev[2]);
    gls_stats& s = ctx->stats;
    s = gls_stats{};
    s.gate_evals = (int64_t)c.gate_evals;
    s.events = (int64_t)c.events;
    s.out_transitions = (int64_t)c.out_trans;
    s.chunks = G;
    s.levels = ctx->L;
    s.arena_used_bytes = (int64_t)top * 8;
    s.kernel_ms = ms_k;
    s.simulate_ms = ms_s;
    s.alg_bytes = -1;
    s.csrp_pages = (int64_t)pages_used;
    const int64_t given = ctx->window_active ? ctx->prefix_total - ((ctx->in_total + 15) & ~15ll) : ctx->in_total;
    s.csrp_waste = (int64_t)pages_used * (int64_t)(L - 1) - (given + (int64_t)c.out_trans);
    ctx->last_chunk_top = std::max<unsigned long long>(ctx->last_chunk_top, (unsigned long long)N);
    ctx->has_result = true;
    return GLS_OK;
}

int gls_get_stats(gls_ctx* ctx, gls_stats* out) {
    if (!ctx || !out) return GLS_EINVAL;
    if (!ctx->has_result) return fail(ctx, GLS_ESTATE, "no simulation result");
    if (ctx->stats.alg_bytes < 0) {
        // algorithmic bytes: every fan-in waveform read once per pin;
        // sum over nets of length x fan-out, reduced on the device (no 8 B/net readback)
        unsigned long long reads = 0;
        const long long N = (long long)ctx->P + ctx->G;
        CK(cudaMemsetAsync(ctx->d_flag64.p, 0, sizeof(unsigned long long), ctx->stream));
        CK(launch_fanin_reads(ctx->d_net_len.p, ctx->d_fanout.p, N, ctx->d_flag64.p, ctx->stream));
        CK(cudaMemcpyAsync(&reads, ctx->d_flag64.p, sizeof(reads), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->stats.alg_bytes = (int64_t)(8.0L * (long double)reads + 8.0L * (long double)ctx->stats.out_transitions +
                                         20.0L * ctx->E + 8.0L * ctx->G);
        ctx->stats.fanin_reads = (int64_t)reads;
    }
    *out = ctx->stats;
    return GLS_OK;
}

int gls_get_trace(gls_ctx* ctx, uint64_t* trace) {
    if (!ctx || !trace) return GLS_EINVAL;
    if (!ctx->has_result || !ctx->traced) return fail(ctx, GLS_ESTATE, "no traced simulation result (gls_config.trace)");
    std::vector<unsigned long long> t((size_t)8 * ctx->G);
    if (ctx->G) CK(cudaMemcpy(t.data(), ctx->d_trace.p, sizeof(unsigned long long) * 8 * ctx->G, cudaMemcpyDeviceToHost));
    for (int32_t g = 0; g < ctx->G; ++g)
        for (int q = 0; q < 8; ++q) trace[8ll * g + q] = t[8ll * ctx->inv[g] + q];
    return GLS_OK;
}

int gls_get_halo(gls_ctx* ctx, int64_t* halo) {
    if (!ctx || !halo) return GLS_EINVAL;
    if (!ctx->has_netlist) return fail(ctx, GLS_ESTATE, "no netlist");
    *halo = ctx->halo;
    return GLS_OK;
}

int gls_get_levels(gls_ctx* ctx, int32_t* levels) {
    if (!ctx || !levels) return GLS_EINVAL;
    if (!ctx->has_netlist) return fail(ctx, GLS_ESTATE, "no netlist");
    *levels = ctx->L;
    return GLS_OK;
}

int gls_get_net_counts(gls_ctx* ctx, int64_t* counts) {
    if (!ctx || !counts) return GLS_EINVAL;
    if (!ctx->has_result) return fail(ctx, GLS_ESTATE, "no simulation result");
    const int64_t N = (int64_t)ctx->P + ctx->G;
    std::vector<unsigned long long> len((size_t)N);
    if (N) CK(cudaMemcpy(len.data(), ctx->d_net_len.p, sizeof(unsigned long long) * N, cudaMemcpyDeviceToHost));
    for (int32_t i = 0; i < ctx->P; ++i) counts[i] = (int64_t)len[i];
    for (int32_t g = 0; g < ctx->G; ++g) counts[ctx->P + g] = (int64_t)len[ctx->P + ctx->inv[g]];
    return GLS_OK;
}

// a10 / GK3: the canonical CSR is built on the device (range_gather_kernel: every net's
// chunk segments in time order, user net order) through a bounded staging buffer, batch
// by batch of nets, each batch one D2H into the caller's array.
int gls_get_waveforms(gls_ctx* ctx, int64_t* offsets, uint64_t* tr, int64_t capacity, int64_t* total_out) {
    if (!ctx) return GLS_EINVAL;
    if (!ctx->has_result) return fail(ctx, GLS_ESTATE, "no simulation result");
    cudaSetDevice(ctx->device);
    const int64_t N = (int64_t)ctx->P + ctx->G;
    std::vector<unsigned long long> len((size_t)N);
    if (N) CK(cudaMemcpy(len.data(), ctx->d_net_len.p, sizeof(unsigned long long) * N, cudaMemcpyDeviceToHost));
    auto internal = [&](int64_t u) -> int64_t { return u < ctx->P ? u : ctx->P + ctx->inv[u - ctx->P]; };
    std::vector<int64_t> off((size_t)N + 1, 0);
    for (int64_t u = 0; u < N; ++u) off[u + 1] = off[u] + (int64_t)len[(size_t)internal(u)];
    const int64_t total = off[N];
    if (offsets) std::memcpy(offsets, off.data(), sizeof(int64_t) * (N + 1));
    if (total_out) *total_out = total;
    if (!tr) return GLS_OK;
    if (capacity < total) return fail(ctx, GLS_ERANGE, "capacity %lld < %lld transitions", (long long)capacity, (long long)total);
    if (total == 0) return GLS_OK;
    int64_t maxlen = 0;
    for (int64_t u = 0; u < N; ++u) maxlen = std::max<int64_t>(maxlen, off[u + 1] - off[u]);
    const int64_t mib = ctx->cfg.readback_mib > 0 ? ctx->cfg.readback_mib : 1024;
    const int64_t stage = std::min<int64_t>(total, std::max<int64_t>(maxlen, mib << 17));   // MiB / 8 B
    DevBuf<uint64_t> d_stage;
    DevBuf<long long> d_off;
    CK(d_stage.alloc((size_t)stage));
    CK(d_off.alloc((size_t)N + 1));
    const SimParams p = params(ctx);
    for (int64_t u0 = 0; u0 < N;) {
        int64_t u1 = u0;                               // nets [u0, u1) fit the staging buffer
        while (u1 < N && off[u1 + 1] - off[u0] <= stage) ++u1;
        std::vector<long long> rel((size_t)(u1 - u0) + 1);
        for (int64_t u = u0; u <= u1; ++u) rel[(size_t)(u - u0)] = off[u] - off[u0];
        CK(cudaMemcpyAsync(d_off.p, rel.data(), sizeof(long long) * rel.size(), cudaMemcpyHostToDevice, ctx->stream));
        CK(launch_range_gather(p, ctx->d_inv.p, u0, u1, LLONG_MIN, LLONG_MAX, d_off.p, d_stage.p, ctx->stream));
        CK(cudaMemcpyAsync(tr + off[u0], d_stage.p, sizeof(uint64_t) * (off[u1] - off[u0]), cudaMemcpyDeviceToHost,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        u0 = u1;
    }
    return GLS_OK;
}

int gls_get_waveforms_range_device(gls_ctx* ctx, int64_t net_lo, int64_t net_hi, int64_t t_lo, int64_t t_hi,
                                   int64_t* d_offsets, uint64_t* d_tr, int64_t capacity, int64_t* total_out) {
    if (!ctx) return GLS_EINVAL;
    if (!ctx->has_result) return fail(ctx, GLS_ESTATE, "no simulation result");
    const int64_t N = (int64_t)ctx->P + ctx->G;
    if (net_lo < 0 || net_hi < net_lo || net_hi > N) return fail(ctx, GLS_EINVAL, "net range [%lld, %lld) invalid",
                                                                 (long long)net_lo, (long long)net_hi);
    if (t_hi < t_lo) return fail(ctx, GLS_EINVAL, "t_hi < t_lo");
    if (!d_offsets) return fail(ctx, GLS_EINVAL, "null offsets");
    cudaSetDevice(ctx->device);
    const int64_t n = net_hi - net_lo;
    const SimParams p = params(ctx);
    long long* o = (long long*)d_offsets;
    CK(cudaMemsetAsync(o, 0, sizeof(long long), ctx->stream));
    long long total = 0;
    if (n > 0) {
        DevBuf<long long> cnt;
        CK(cnt.alloc((size_t)n));
        CK(launch_range_counts(p, ctx->d_inv.p, net_lo, net_hi, t_lo, t_hi, cnt.p, ctx->stream));
        size_t tb = 0;
        CK(launch_inclusive_scan(cnt.p, o + 1, n, nullptr, &tb, ctx->stream));
        DevBuf<unsigned char> tmp;
        CK(tmp.alloc(tb));
        CK(launch_inclusive_scan(cnt.p, o + 1, n, tmp.p, &tb, ctx->stream));
        CK(cudaMemcpyAsync(&total, o + n, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    if (total_out) *total_out = total;
    if (!d_tr) {
        CK(cudaStreamSynchronize(ctx->stream));
        return GLS_OK;
    }
    if (capacity < total) return fail(ctx, GLS_ERANGE, "capacity %lld < %lld transitions", (long long)capacity, total);
    CK(launch_range_gather(p, ctx->d_inv.p, net_lo, net_hi, t_lo, t_hi, o, d_tr, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return GLS_OK;
}

int gls_scatter_segments(gls_ctx* ctx, int64_t nseg, const int64_t* d_src_off, const uint64_t* d_src,
                         const int64_t* d_dst_off, uint64_t* d_dst) {
    if (!ctx) return GLS_EINVAL;
    if (nseg < 0 || (nseg > 0 && (!d_src_off || !d_src || !d_dst_off || !d_dst)))
        return fail(ctx, GLS_EINVAL, "bad segment arrays");
    cudaSetDevice(ctx->device);
    CK(launch_scatter_segments(nseg, (const long long*)d_src_off, d_src, (const long long*)d_dst_off, d_dst, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return GLS_OK;
}

int gls_get_net_hashes_device(gls_ctx* ctx, uint64_t* d_hashes) {
    if (!ctx || !d_hashes) return GLS_EINVAL;
    if (!ctx->has_result) return fail(ctx, GLS_ESTATE, "no simulation result");
    cudaSetDevice(ctx->device);
    CK(launch_hashes(params(ctx), ctx->d_perm.p, d_hashes, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return GLS_OK;
}

int gls_get_net_hashes_window(gls_ctx* ctx, int64_t t_lo, int64_t t_hi, uint64_t* hashes) {
    if (!ctx || !hashes) return GLS_EINVAL;
    if (!ctx->has_result) return fail(ctx, GLS_ESTATE, "no simulation result");
    if (t_hi < t_lo) return fail(ctx, GLS_EINVAL, "t_hi < t_lo");
    const int64_t N = (int64_t)ctx->P + ctx->G;
    cudaSetDevice(ctx->device);
    CK(ctx->d_hash.ensure(N));
    CK(launch_hashes_window(params(ctx), ctx->d_perm.p, t_lo, t_hi, ctx->d_hash.p, ctx->stream));
    if (N) CK(cudaMemcpyAsync(hashes, ctx->d_hash.p, sizeof(uint64_t) * N, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return GLS_OK;
}

int gls_get_net_hash_terms_device(gls_ctx* ctx, int64_t t_lo, int64_t t_hi, const int64_t* d_base,
                                  const int64_t* d_total, int64_t* d_counts, uint64_t* d_terms) {
    if (!ctx || !d_counts) return GLS_EINVAL;
    if (!ctx->has_result) return fail(ctx, GLS_ESTATE, "no simulation result");
    if (t_hi < t_lo) return fail(ctx, GLS_EINVAL, "t_hi < t_lo");
    cudaSetDevice(ctx->device);
    CK(launch_hash_terms(params(ctx), ctx->d_perm.p, t_lo, t_hi, (const long long*)d_base,
                         (const long long*)d_total, (long long*)d_counts, d_terms, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return GLS_OK;
}

int gls_get_net_hashes(gls_ctx* ctx, uint64_t* hashes) {
    if (!ctx || !hashes) return GLS_EINVAL;
    if (!ctx->has_result) return fail(ctx, GLS_ESTATE, "no simulation result");
    const int64_t N = (int64_t)ctx->P + ctx->G;
    cudaSetDevice(ctx->device);
    CK(ctx->d_hash.ensure(N));
    int rc = gls_get_net_hashes_device(ctx, ctx->d_hash.p);
    if (rc) return rc;
    if (N) CK(cudaMemcpyAsync(hashes, ctx->d_hash.p, sizeof(uint64_t) * N, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return GLS_OK;
}

}  // extern "C"
