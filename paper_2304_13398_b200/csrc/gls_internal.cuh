// gls_internal.cuh — device data layout shared by the host API (gls_api.cu) and
// the kernels (gls_kernels.cu).  Product code: shares nothing with oracle/.
//
// Layout:
//   nets      0..P-1 given (PI / pseudo-PI), P+i output of internal gate i;
//             internal gates are sorted by topological level.
//   arena     one u64 store for given and computed waveforms (the paper keeps
//             both in one CSRP store); entries (t << 2) | v.
//   chunks    a net's waveform is a time-ordered list of chunk segments; chunk
//             j holds the net's transitions with t in [ck_T[j], ck_T[j+1]) at
//             arena[ck_off[j] .. + ck_cnt[j]).  Given nets have one chunk.
//             A gate's chunks are its (gate, time-chunk) work items.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// Bounds-checked build (make check -> libgls_check.so, -DGLS_CHECK): every store and load of
// the hot path is checked against the buffer it must stay in; a violation prints the
// condition and traps the kernel.  The stand-in for compute-sanitizer, which is closed on
// the GPU pool (profiles/r02_sanitizer_closed.txt).
#ifdef GLS_CHECK
#define GLS_ASSERT(c)                                                                              \
    do {                                                                                           \
        if (!(c)) {                                                                                \
            printf("GLS_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);                        \
            __trap();                                                                              \
        }                                                                                          \
    } while (0)
#else
#define GLS_ASSERT(c) \
    do {              \
    } while (0)
#endif

namespace gls {

constexpr int kNumTypes = 9;
constexpr int kLutPerType = 4 + 16 + 64 + 256;       // arity 1..4, index = packed 2-bit codes
constexpr int kLutBytes = kLutPerType * kNumTypes;   // 3060 B: the basic gates' tables
constexpr int kLutCap = 4096;                        // smem LUT: basic tables + cell output functions (a3)
constexpr uint32_t kDelayInf = 0xFFFFFFFFu;          // "no relation" (reading R9)
constexpr uint32_t kDelayInf16 = 0xFFFFu;            // the same in the u16 delay table of the 32-bit sweep
constexpr uint64_t kInfEntry = ~0ull;                // head of an exhausted cursor
constexpr int kRing = 32;                            // on-chip pending-schedule ring (power of 2)
#ifndef GLS_THREADS
#define GLS_THREADS 256
#endif
constexpr int kThreads = GLS_THREADS;                       // persistent-kernel CTA size

__host__ __device__ inline int lut_offset(int type, int arity) {
    // offset of (type, arity) table; arity 1 -> 0, 2 -> 4, 3 -> 20, 4 -> 84
    return type * kLutPerType + (arity == 1 ? 0 : arity == 2 ? 4 : arity == 3 ? 20 : 84);
}

struct GateInfo {
    uint32_t pin_off;   // first pin in pin_src / pin_delay
    uint16_t lut_base;  // lut_offset(type, arity)
    uint8_t k;          // arity 1..4
    uint8_t flags;      // kGateInf: a pin delay is GLS_DELAY_INF (never time-chunked, see kernels)
};

constexpr uint8_t kGateInf = 1;
enum : unsigned { kErrArena = 1u, kErrChunks = 2u, kErrDeep = 4u, kErrInput = 8u, kErrBug = 16u, kErrWatchdog = 32u };

// device control block, initialised by the host before each run
// (the counters every warp hits — atomics on the queue and the store, the polled completion
// count — each own a 128-byte line: one hot line would serialise all of them in one L2 slice)
struct Ctl {
    unsigned long long chunk_top;   // next free chunk id (starts at P: one chunk per given net)
    unsigned long long pad0[15];
    unsigned long long arena_top;   // next free arena entry (starts after the given waveforms)
    unsigned long long pad1[15];
    unsigned long long work_head;   // dataflow queue: next chunk id to hand out (starts at P)
    unsigned long long pad2[15];
    unsigned long long done_gates;  // dataflow: completed gates
    unsigned int error;             // kErr* bits
    unsigned int pad3a;
    unsigned long long pad3[14];
    unsigned int bar_count;
    unsigned int bar_gen;
    unsigned int bar_abort;
    unsigned int pad4;
    unsigned long long need_arena;  // entries needed when kErrArena was raised
    unsigned long long need_chunks;
    unsigned long long need_deep;
    unsigned long long gate_evals;
    unsigned long long events;
    unsigned long long out_trans;
    unsigned long long chunks;
    unsigned long long deep_chunks;
    unsigned long long lane_iters;    // slice engine: loop iterations summed over lanes
    unsigned long long warp_iters;    // slice engine: 32 x the longest lane's iterations, summed over chunks
    unsigned long long batches;       // slice engine: warp batches
    unsigned long long batch_lanes;   // slice engine: lanes holding work, summed over batches
    unsigned long long batch_est;     // slice engine: expected transitions, summed over batches
    unsigned long long cyc[6];        // slice engine, lane 0 clocks: wait/assemble, setup, locate, sweep, output, complete
    unsigned long long bal[8];        // slice engine lane balance (gls_stats.balance)
};

struct SimParams {
    int32_t P, G, L;
    const int32_t* level_off;   // [L+1] internal gate index ranges per level
    const GateInfo* gate;       // [G]
    const uint32_t* pin_src;    // [E] internal net id of each pin's driver
    const uint4* pin_delay;     // [E] (rise->0, rise->1, fall->0, fall->1)
    const uint8_t* lut;         // [kLutCap]
    uint64_t* arena;
    unsigned long long arena_cap;     // entries
    uint32_t* net_ck;           // [P+G] first chunk id
    uint32_t* net_nck;          // [P+G] number of chunks
    unsigned long long* net_len;      // [P+G] transitions
    long long* ck_T;            // [ck_cap] chunk start time
    unsigned long long* ck_off; // [ck_cap] arena offset of the chunk segment
    uint32_t* ck_cnt;           // [ck_cap] entries in the segment
    unsigned long long* ck_cum; // [ck_cap] entries of the net before this chunk
    uint8_t* ck_vb;             // [ck_cap] net value just before ck_T (for halo starts)
    uint32_t* ck_gate;          // [ck_cap] internal gate of the chunk
    unsigned long long ck_cap;
    uint32_t* gate_done;        // [G] finished chunks per gate
    unsigned long long* gate_nin;   // [G] Σ fan-in transitions (set when the gate is planned)
    unsigned long long* work;   // [L+1] per-level work counters
    uint64_t* deep;             // deep-backtrace scratch: one region per warp
    uint64_t* wscr;             // per-warp output scratch
    void* waux;                 // per-warp auxiliary unit fields (engine 0)
    unsigned long long deep_cap;
    unsigned long long deep_per_warp;
    unsigned long long* deep_wtop;  // [warps] bump pointer of each warp's region
    const uint32_t* fo_off;     // [P+G+1] consumers (internal gates) of each net
    const uint32_t* fo_gate;    // [E_gate]
    uint32_t* pend;             // [G] fan-in pins whose driver gate is not complete yet
    Ctl* ctl;
    long long duration;
    int32_t M;                  // target merged input events per chunk
    int32_t ring_cap;           // <= kRing
    int32_t engine;             // 0 = lanes on re-balanced units, 1 = per-lane chunks
    int32_t sched;              // 0 = dataflow (ready counters), 1 = level barriers
    uint32_t nblocks;
    unsigned long long* trace;  // [8 G] or null (gls_get_trace)
};

// kernels / launchers (gls_kernels.cu)
cudaError_t launch_init_given(const SimParams& p, const long long* in_off, cudaStream_t s);
cudaError_t launch_simulate(const SimParams& p, int blocks, cudaStream_t s);
size_t warp_scratch_entries(int blocks);
size_t warp_aux_bytes(int blocks);
// engine 2 (CSRP pages + Alg. 1, gls_csrp.cuh)
int csrp_coresident_threads(int device);
size_t csrp_scratch_entries(int threads);
cudaError_t launch_csrp(const SimParams& p, uint64_t* pages, unsigned long long* page_top,
                        unsigned long long page_cap, uint32_t pagelen, unsigned long long* first_page,
                        uint32_t* known, unsigned long long* out_cnt, const long long* in_off, int threads,
                        cudaStream_t s);
cudaError_t launch_csrp_collect(const SimParams& p, uint64_t* pages, uint32_t pagelen, unsigned long long* first_page,
                                unsigned long long* out_cnt, const unsigned long long* seg_off, cudaStream_t s);
int max_coresident_blocks(int device, int engine, int sched, int* per_sm);
// time-window slice of the given waveforms (gls_simulate_window): per net the number of
// kept entries, then the entries (collapse at t_clamp, keep t_clamp < t < t_end)
cudaError_t launch_window_count(int32_t P, const long long* off, const uint64_t* tr, long long t_clamp,
                                long long t_end, long long* cnt, cudaStream_t s);
cudaError_t launch_window_fill(int32_t P, const long long* off, const uint64_t* tr, long long t_clamp,
                               long long t_end, const long long* new_off, uint64_t* out, cudaStream_t s);
cudaError_t launch_validate_inputs(int32_t P, const long long* off, const uint64_t* tr, long long total,
                                   unsigned* d_err, unsigned long long* d_maxt, cudaStream_t s);
cudaError_t launch_hashes(const SimParams& p, const uint32_t* perm, uint64_t* out, cudaStream_t s);
// time-window stitching pieces (gls_get_net_hash_terms_device): per user net, count of the
// entries with t_lo <= t <= t_hi and (terms != NULL) their checksum terms at base + j
cudaError_t launch_hash_terms(const SimParams& p, const uint32_t* perm, long long t_lo, long long t_hi,
                              const long long* base, const long long* total, long long* counts, uint64_t* terms,
                              cudaStream_t s);
// sum over nets of len[n] * fanout[n] (fan-in reads of Alg. 2, for gls_stats.alg_bytes) into *out
cudaError_t launch_fanin_reads(const unsigned long long* len, const uint32_t* fanout, long long n,
                               unsigned long long* out, cudaStream_t s);
// canonical CSR of user nets [u0, u1) restricted to t_lo <= t <= t_hi: per-net counts, then
// the gather into dst at the given (relative) offsets; generic segment scatter (stitching)
cudaError_t launch_range_counts(const SimParams& p, const uint32_t* inv, long long u0, long long u1, long long t_lo,
                                long long t_hi, long long* cnt, cudaStream_t s);
cudaError_t launch_range_gather(const SimParams& p, const uint32_t* inv, long long u0, long long u1, long long t_lo,
                                long long t_hi, const long long* off, uint64_t* dst, cudaStream_t s);
cudaError_t launch_scatter_segments(long long nseg, const long long* src_off, const uint64_t* src,
                                    const long long* dst_off, uint64_t* dst, cudaStream_t s);
cudaError_t launch_inclusive_scan(const long long* in, long long* out, long long n, void* tmp, size_t* tmp_bytes,
                                  cudaStream_t s);
cudaError_t launch_hashes_window(const SimParams& p, const uint32_t* perm, long long t_lo, long long t_hi,
                                 uint64_t* out, cudaStream_t s);

}  // namespace gls
