/*
 * gls.h — C ABI of the B200-native waveform-based, timing-aware, 4-value
 * gate-level re-simulation library (libgls.so).  Method: arxiv 2304.13398,
 * "Acceleration for Timing-Aware Gate-Level Logic Simulation with One-Pass GPU
 * Parallelism".  Citations are PAPER.md line numbers (P:n) with the section /
 * equation / algorithm; readings of points the paper leaves open are numbered
 * R1..R17 in DESIGN.md §3-§4.
 *
 * Problem (§2.1): given a combinational netlist of basic gates, the
 * delays of its pins and the waveforms of the given nets (primary inputs and
 * register outputs cut into pseudo-primary inputs, P:87 footnote), compute the
 * waveform of every gate output over [0, duration].  Values are 4-valued
 * 0/1/X/Z (§2.2); Z at a gate input is read as X; gate
 * outputs are never Z.  Delays are pin-to-pin per input edge and output value,
 * the minimum over inputs changing together (§2.3), with inertial
 * "glitch eaten" filtering (Eq. 1).
 *
 * Conventions for every function:
 *   - returns int status: GLS_OK (0) or a negative GLS_E* code; never aborts or
 *     throws.  gls_last_error() gives a message for the last failing call.
 *   - on error the context is unchanged (no partial update), except that a
 *     failing gls_simulate leaves no valid result (gls_get_* -> GLS_ESTATE).
 *   - every input array is COPIED during the call (host pointers may be freed on
 *     return; device pointers may be reused once the call returns, because the
 *     copy is ordered on the context's stream and the call synchronises it).
 *   - a context is not thread-safe; distinct contexts are independent.
 *   - all device work is issued on the stream given to gls_create.
 */
#ifndef GLS_H
#define GLS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
enum {
    GLS_OK = 0,
    GLS_EINVAL = -1,  /* malformed argument (type, arity, id, delay, time, value) */
    GLS_ECYCLE = -2,  /* combinational loop: the netlist is not a DAG (P:87 fn)   */
    GLS_ENOMEM = -3,  /* device memory / arena / chunk table too small; message
                         names the size needed; the call may be retried after
                         gls_set_config with larger limits                         */
    GLS_ESTATE = -4,  /* call-order violation (e.g. simulate before load)         */
    GLS_ERANGE = -5,  /* time > duration, duration >= 2^61, or an output buffer
                         smaller than the result                                   */
    GLS_ECUDA = -6    /* CUDA runtime error (message has the CUDA error string)   */
};

/* ---- values and packing (§2.1 "value and time"; §2.2) ------- */
enum { GLS_V0 = 0, GLS_V1 = 1, GLS_VX = 2, GLS_VZ = 3 };
/* A transition is one uint64: time in ps in bits 63..2, value code in bits 1..0.
 * Time must be < 2^61.  (The paper stores int64 + int8 = 9 B.) */
#define GLS_PACK(t, v) ((((uint64_t)(t)) << 2) | ((uint64_t)(v) & 3u))
#define GLS_TIME(e) ((int64_t)((uint64_t)(e) >> 2))
#define GLS_VAL(e) ((int)((e) & 3u))

/* ---- basic gates (Table 1; composition §3.3) -------- */
enum {
    GLS_BUF = 0,  /* arity 1                                                   */
    GLS_NOT = 1,  /* arity 1                                                   */
    GLS_AND = 2,  /* arity 2..4, left fold of Table 1(a) (reading R10)         */
    GLS_NAND = 3, /* NOT(AND)                                                  */
    GLS_OR = 4,   /* arity 2..4, Table 1(b)                                    */
    GLS_NOR = 5,  /* NOT(OR)                                                   */
    GLS_XOR = 6,  /* arity 2..4, Table 1(c)                                    */
    GLS_XNOR = 7, /* NOT(XOR)                                                  */
    GLS_MUX2 = 8  /* arity 3, pins (a, b, sel): OR(AND(a,NOT sel),AND(b,sel)),
                     reading R11                                              */
};

typedef struct gls_ctx gls_ctx;

/* ---- tuning knobs (all optional; zero = default) ------------------------ */
typedef struct gls_config {
    int64_t arena_bytes;     /* transition store for given + computed waveforms
                                (one store); 0 = auto (most of the
                                free HBM)                     */
    int64_t chunk_capacity;  /* max (gate, time-chunk) work items per run; 0 = auto */
    int32_t chunk_events;    /* target merged input events per work item (M);
                                0 = 32768 / 256 for engines 0 / 1                  */
    int32_t blocks_per_sm;   /* persistent-kernel CTAs per SM; 0 = max co-resident */
    int32_t ring_limit;      /* TESTING: cap on the on-chip pending-schedule ring
                                (1..32) to force the deep-backtrace path; 0 = 32 */
    int32_t engine;          /* evaluation engine of a (gate, time-chunk) item:
                                0 = a warp's lanes on time-slice units of a batch of
                                    items, re-balanced by splitting while they run (default),
                                1 = one item per lane (reference engine for A/B),
                                2 = the paper's design (A/B): CSRP pages with next-page
                                    pointers and an atomic page iterator (§3.1), one
                                    thread per cell statically dealt (Alg. 1)            */
    int32_t scheduler;       /* 0 = dataflow: a gate is scheduled when its last fan-in
                                gate completes (Alg. 1 unlock rule) (default);
                                1 = topological levels separated by device barriers.
                                Engine 1 always uses levels.                        */
    int64_t deep_per_warp;   /* per-warp scratch (entries) for deep backtraces and
                                output spills; 0 = 65536, grown automatically      */
    int32_t readback_mib;    /* gls_get_waveforms: device staging buffer of the
                                canonical CSR (MiB; batches of nets go through it,
                                one D2H each); 0 = 1024                            */
    int32_t trace;           /* 1: record per-gate times for gls_get_trace (diagnostics) */
    int32_t csrp_pagelen;    /* engine 2: CSRP page length in entries (256); 0 = 256 */
} gls_config;

typedef struct gls_stats {
    int64_t gate_evals;      /* Σ_g distinct fan-in timestamps (one calculateSignals
                                of Alg. 2 each)                              */
    int64_t events;          /* zero-delay output changes (Alg. 2 "o_k.v is changed") */
    int64_t out_transitions; /* Σ_g |W(g)| after filtering and clipping            */
    int64_t chunks;          /* (gate, time-chunk) work items processed            */
    int64_t deep_chunks;     /* work items that needed the deep-backtrace path     */
    int64_t levels;          /* topological levels (device barriers = 2 per level) */
    int64_t arena_used_bytes;
    int64_t alg_bytes;       /* algorithmic bytes of the gate-evaluation kernel
                                (DESIGN.md §7): 8·Σ fan-in reads + 8·outputs +
                                20·pins + 8·gates                                  */
    int64_t fanin_reads;     /* Σ over pins of the driving net's transitions      */
    double lane_utilization; /* engine 0: busy lane-iterations / (32 x the busiest lane's
                                iterations), summed over re-balancing rounds          */
    int64_t batches;         /* engine 0: warp batches                              */
    double batch_lanes;      /* engine 0: mean lanes holding a static unit per batch */
    double batch_est;        /* engine 0: mean expected merged entries per batch    */
    double phase_cycles[6];  /* engine 0, lane 0 clocks summed over warps: waiting +
                                batch assembly, static unit boundaries, sweep (rounds),
                                fallback + allocation + output copy, chunk completion,
                                lane-average clocks in unit set-up (part of the sweep) */
    double balance[8];       /* engine 0 counters: [0] static units, [1] units split off
                                while running, [2] re-balancing rounds, [3] fallback
                                units (per-lane ring engine); warp-level clocks (lane
                                0, summed over warps) in [4] unit set-up passes, [5]
                                unit-end passes, [6] re-balancing points; [7] unused  */
    double kernel_ms;        /* CUDA-event time of the gate-evaluation kernel      */
    int64_t csrp_pages;      /* engine 2: CSRP pages handed out                     */
    int64_t csrp_waste;      /* engine 2: page slots not holding an entry (Eq. 4 bounds
                                it by pagelen x waveforms)               */
    double simulate_ms;      /* CUDA-event time of the whole gls_simulate          */
} gls_stats;

/* ---- lifetime ----------------------------------------------------------- */
/* Create a context on CUDA device `cuda_device`, issuing all work on
 * `cuda_stream` (a cudaStream_t; NULL = the legacy default stream; a
 * torch.cuda.Stream's .cuda_stream is accepted).  *out is NULL on error. */
int gls_create(gls_ctx **out, int cuda_device, void *cuda_stream);
/* Free all device and host memory of the context.  NULL is a no-op. */
void gls_destroy(gls_ctx *ctx);
/* Message of the last failing call on ctx ("" if none).  Owned by ctx. */
const char *gls_last_error(const gls_ctx *ctx);
/* Library version string (static storage). */
const char *gls_version(void);
/* Replace the tuning knobs (copied).  Takes effect at the next gls_simulate. */
int gls_set_config(gls_ctx *ctx, const gls_config *cfg);

/* ---- netlist (a1: validation + levelisation) -------------- */
/* Nets: 0..num_inputs-1 are the given waveforms (primary / pseudo-primary
 * inputs); num_inputs + g is the output of gate g (caller's gate order).
 *   gate_type     [num_gates]        GLS_BUF..GLS_MUX2
 *   fanin_offsets [num_gates+1]      CSR over pins, fanin_offsets[0] = 0; the
 *                                    pin order is the gate function's operand order
 *   fanin_net     [E]                driving net id of each pin, E = fanin_offsets[G]
 *   pin_delay     [E][4]             ps, u32 < 2^31, per pin:
 *                                    [0] in-edge RISE, output -> 0
 *                                    [1] in-edge RISE, output -> 1
 *                                    [2] in-edge FALL, output -> 0
 *                                    [3] in-edge FALL, output -> 1
 *                                    (GLS_DELAY_INF: the pin has no relation to
 *                                    the output, reading R9)
 *                                    (the paper's 5-D matrix Delay[cell][in][out]
 *                                    [edge][value], for single-output
 *                                    gates; output -> X uses min of the two,
 *                                    reading R1; an input edge is RISE iff the
 *                                    value rises in the order 0 < X < 1, R2)
 * Errors: GLS_EINVAL (type, arity, id out of range, delay >= 2^31, E >= 2^31,
 * num_inputs + num_gates >= 2^31), GLS_ECYCLE (loop), GLS_ENOMEM, GLS_ECUDA.
 * Loading replaces any previous netlist and clears the inputs and results. */
int gls_load_netlist(gls_ctx *ctx, int32_t num_inputs, int32_t num_gates,
                     const uint8_t *gate_type, const int64_t *fanin_offsets,
                     const int32_t *fanin_net, const uint32_t *pin_delay);

/* ---- multi-output cells and UDPs (NEXT-2: §3.2 Delay P:329-333, §3.3 Module
 * Function P:335-339) ---------------------------------------------------- */
#define GLS_DELAY_INF 0xFFFFFFFFu  /* "no relation" between an input and an output pin
                                      (P:331-333): the pin never enters the delay minimum;
                                      an output change whose changed inputs are all
                                      unrelated is not scheduled (reading R9)          */
/* A standard cell template / UDP: a DAG of basic gates over the cell's inputs (the
 * paper composes every cell function from the basic gates' functions), its
 * outputs some of the DAG's nodes, evaluated with zero internal delay.  Node ids:
 * 0..num_inputs-1 the cell inputs, num_inputs + j basic gate j (fan-in nodes < j's own). */
typedef struct gls_cell_template {
    int32_t num_inputs;              /* 1..4                                          */
    int32_t num_outputs;             /* 1..8                                          */
    int32_t num_gates;               /* 0..64                                         */
    const uint8_t *gate_type;        /* [num_gates] GLS_BUF..GLS_MUX2                  */
    const int32_t *gate_fanin_offsets; /* [num_gates + 1] into gate_fanin            */
    const int32_t *gate_fanin;       /* node ids                                      */
    const int32_t *output_node;      /* [num_outputs]                                 */
} gls_cell_template;
/* Load a netlist of cells (replaces any netlist; clears inputs and results).  Nets:
 * 0..num_inputs-1 given, then the outputs of every cell in cell order (cell c's output
 * q is net num_inputs + (outputs of the cells before c) + q).
 *   cell_template [num_cells]      template id of each cell
 *   cell_fanin    [Σ num_inputs]   driving net of each input pin, cells concatenated
 *   cell_delay    [Σ num_inputs*num_outputs*4]  per cell Delay[in][out][edge][value],
 *                                  edge RISE = 0 / FALL = 1, value 0 / 1 (the paper's 5-D
 *                                  matrix), ps < 2^31 or GLS_DELAY_INF
 * A gate-eval counts per cell OUTPUT.  Distinct output functions that are not a basic
 * gate's share a (kLutCap - 3060 = 1036)-byte table area in shared memory (e.g. 4
 * four-input or 16 three-input functions); more -> GLS_EINVAL.  Errors: GLS_EINVAL,
 * GLS_ECYCLE, GLS_ENOMEM, GLS_ECUDA. */
int gls_load_cells(gls_ctx *ctx, int32_t num_inputs, int32_t num_templates, const gls_cell_template *templates,
                   int32_t num_cells, const int32_t *cell_template, const int32_t *cell_fanin,
                   const uint32_t *cell_delay);

/* ---- given waveforms (a2) ------------------------------------------------ */
/* CSR of packed transitions on the num_inputs given nets (HOST pointers):
 *   offsets     [num_inputs+1], offsets[0] = 0, non-decreasing
 *   transitions [offsets[num_inputs]] GLS_PACK(t, v)
 * Per net: times strictly increasing, 0 <= t < 2^61; value codes 0..3; no
 * value equal to the previous one, where the value before the first transition
 * is X (so a first transition to X is rejected; Z is a distinct code) — the
 * waveform rules of §2.1 and reading R6.  A net with no transition is
 * constant X.  Errors: GLS_EINVAL, GLS_ESTATE (no netlist / num_inputs
 * mismatch), GLS_ENOMEM, GLS_ECUDA.  May be repeated (re-simulation with a new
 * stimulus set, the netlist stays loaded).  The stimulus is checked on a device
 * copy (a staging buffer; device inputs in place) before it replaces the given
 * waveforms, so a rejected one leaves the previous inputs and result in place —
 * except when the staging buffer cannot be allocated (the arena holds nearly all
 * HBM): then a rejected HOST stimulus leaves the context without inputs. */
int gls_set_input_waveforms(gls_ctx *ctx, int32_t num_inputs, const int64_t *offsets,
                            const uint64_t *transitions);
/* Same, from DEVICE pointers on the context's device (validated on the device). */
int gls_set_input_waveforms_device(gls_ctx *ctx, int32_t num_inputs, const int64_t *d_offsets,
                                   const uint64_t *d_transitions, int64_t total);

/* ---- simulation (a3-a9: one persistent-kernel pass, no host round trip) -- */
/* Simulate every gate over [0, duration]; output transitions that would appear
 * after `duration` are dropped (reading R7).  Errors: GLS_ESTATE (no netlist or
 * inputs), GLS_ERANGE (a given transition later than duration, or duration <
 * 0 or >= 2^61), GLS_ENOMEM (arena / chunk table too small: message gives the
 * bytes needed; retry after gls_set_config), GLS_ECUDA.  Synchronous: returns
 * when the result is on the device. */
int gls_simulate(gls_ctx *ctx, int64_t duration);
/* One time window of the same run (time-window sharding; DESIGN.md §4,
 * reading R17): the outputs are exact on [t_begin, t_end) ∩ [0, duration] — the same
 * transitions gls_simulate(duration) produces there — at the cost of the window plus a
 * halo H = gls_get_halo().  From the given waveforms set last, the library keeps
 * every transition with t_begin - H < t < t_end and collapses the earlier ones into one
 * transition at t_begin - H carrying the value then in effect (none if X); inputs at
 * or after t_end cannot change outputs before t_end.  It then simulates to
 * min(duration, t_end - 1).  The result (gls_get_waveforms, hashes, stats) is that run's:
 * transitions before t_begin may differ from the full run's (halo), the stats include
 * the halo's work.  The full given waveforms stay in the context (a device copy), so
 * windows can be simulated in any order, and a later gls_simulate runs the full
 * inputs again.  Errors: as gls_simulate, and GLS_EINVAL if t_end < t_begin or
 * t_begin < 0. */
int gls_simulate_window(gls_ctx *ctx, int64_t t_begin, int64_t t_end, int64_t duration);

/* ---- results (a10) ------------------------------------------------------ */
/* Canonical CSR of all num_inputs + num_gates nets, in net order (given nets
 * verbatim, Z included).  Two-call protocol: with transitions == NULL only
 * *total_out (and offsets if non-NULL) are written.  capacity = number of
 * uint64 slots in `transitions`; GLS_ERANGE if smaller than the total.
 * HOST pointers.  GLS_ESTATE if no successful simulation. */
int gls_get_waveforms(gls_ctx *ctx, int64_t *offsets, uint64_t *transitions,
                      int64_t capacity, int64_t *total_out);
/* The same canonical CSR built on the DEVICE (a10 / GK3 on the GPU: each net's chunk
 * segments gathered in time order, in net order), restricted to the nets
 * [net_lo, net_hi) and to the transitions with t_lo <= t <= t_hi (the whole run:
 * INT64_MIN, INT64_MAX).  d_offsets: DEVICE int64 [net_hi - net_lo + 1], always written
 * (CSR offsets from 0); d_transitions: DEVICE uint64 [capacity] or NULL (size query:
 * only d_offsets and *total_out).  Used by multi-GPU stitching (each rank's owned time
 * window, gathered over NCCL) and by gls_get_waveforms (which runs it batch by batch
 * of nets through a bounded staging buffer, one D2H per batch).  Errors: GLS_EINVAL
 * (range, t_hi < t_lo, NULL offsets), GLS_ERANGE (capacity), GLS_ESTATE (no result).
 * Synchronous. */
int gls_get_waveforms_range_device(gls_ctx *ctx, int64_t net_lo, int64_t net_hi, int64_t t_lo,
                                   int64_t t_hi, int64_t *d_offsets, uint64_t *d_transitions,
                                   int64_t capacity, int64_t *total_out);
/* Stitching helper (multi-GPU results): for i in [0, nseg) copy the
 * segment d_src[d_src_off[i] .. d_src_off[i+1]) to d_dst + d_dst_off[i], on the
 * context's device and stream (one warp per segment).  All DEVICE arrays, caller-owned;
 * segments must not overlap in d_dst.  Errors: GLS_EINVAL (NULL arrays, nseg < 0). */
int gls_scatter_segments(gls_ctx *ctx, int64_t nseg, const int64_t *d_src_off, const uint64_t *d_src,
                         const int64_t *d_dst_off, uint64_t *d_dst);
/* Per-net 64-bit results checksum, host array [num_inputs + num_gates], net order:
 * h = splitmix64(0x9E3779B97F4A7C15 ^ n) XOR (XOR over j = 0..n-1 of
 * splitmix64(e_j + (j + 1) * 0xD1B54A32D192ED03)), e_j the net's j-th packed entry
 * (order-sensitive, computed warp-parallel on the device). */
int gls_get_net_hashes(gls_ctx *ctx, uint64_t *hashes);
/* Same into a DEVICE array (for NCCL gathers). */
int gls_get_net_hashes_device(gls_ctx *ctx, uint64_t *d_hashes);
/* Same checksum over only the transitions with t_lo <= t <= t_hi, j counted from
 * the first of them (host array, net order).  Used to verify time windows (multi-GPU sharding, sampled parity at
 * full size).  GLS_EINVAL if t_hi < t_lo. */
int gls_get_net_hashes_window(gls_ctx *ctx, int64_t t_lo, int64_t t_hi, uint64_t *hashes);
/* Time-window stitching (multi-GPU sharding): the pieces of the
 * full-run checksum above contributed by this context's transitions with
 * t_lo <= t <= t_hi.  DEVICE arrays of num_inputs + num_gates elements, net order:
 *   d_counts[n] (out, int64)  number of such transitions;
 *   d_terms[n]  (out, uint64, NULL = counts only)  XOR over them of
 *               splitmix64(e_j + (d_base[n] + j + 1) * 0xD1B54A32D192ED03), j their
 *               position inside the window and d_base[n] (in, int64, NULL = 0) the
 *               number of the net's transitions before t_lo in the whole run;
 *               if d_total (in, int64) is non-NULL, splitmix64(0x9E3779B97F4A7C15 ^
 *               d_total[n]) is XORed in as well.
 * With the windows of all ranks partitioning [0, duration], d_base = the exclusive
 * prefix over ranks of d_counts, d_total = their sum passed by exactly one rank, the
 * XOR over ranks of d_terms equals gls_get_net_hashes of the full run.  The arrays are
 * written on the context's stream before return.  GLS_EINVAL if t_hi < t_lo or
 * d_counts is NULL, GLS_ESTATE without a result. */
int gls_get_net_hash_terms_device(gls_ctx *ctx, int64_t t_lo, int64_t t_hi, const int64_t *d_base,
                                  const int64_t *d_total, int64_t *d_counts, uint64_t *d_terms);
/* Per-net transition counts, host int64 [num_inputs + num_gates]. */
int gls_get_net_counts(gls_ctx *ctx, int64_t *counts);
/* Counters and timings of the last gls_simulate. */
int gls_get_stats(gls_ctx *ctx, gls_stats *out);
/* 1 + maximum path delay (Σ of max pin delays along the worst path): the halo
 * that makes a time window exact (reading R17).  Needs a netlist. */
int gls_get_halo(gls_ctx *ctx, int64_t *halo_ps);
/* Scheduling trace of the last gls_simulate run with gls_config.trace = 1 (diagnostics,
 * SURVEY §5 tracing): host uint64 [8 * num_gates], per gate in the caller's order:
 * [0] %globaltimer ns when the gate was planned (its chunks published, Alg. 1's unlock),
 * [1] when its last chunk completed, [2] the sum and [3] the maximum of its chunks'
 * durations (claim to completion, ns); for the batch of the slowest chunk (engine 0):
 * [4] re-balancing rounds, [5] units, [6] the busiest lane's iterations, [7] the most unit
 * set-ups of one lane.  GLS_ESTATE without a traced result. */
int gls_get_trace(gls_ctx *ctx, uint64_t *trace);
/* Number of topological levels of the loaded netlist (0 without gates). */
int gls_get_levels(gls_ctx *ctx, int32_t *levels);

/* ---- test hook ---------------------------------------------------------- */
/* The library's own 4-value LUT entry for gate `type` with `arity` pins at
 * input codes v[0..arity-1] (host-built table staged in shared memory by the
 * kernel).  Returns the output code (0,1,2) or GLS_EINVAL. */
int gls_lut_lookup(int type, int arity, const uint8_t *v);

#ifdef __cplusplus
}
#endif
#endif /* GLS_H */
