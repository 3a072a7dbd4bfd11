/*
 * oracle/gls_oracle.c — CPU oracle for 4-value, timing-aware, waveform-based
 * gate-level re-simulation (arxiv 2304.13398).
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the plain, slow, obviously-correct
 * definition the CUDA path is checked against.  Only tests/, the smoke() check
 * in __graft_entry__.py and the cpu_baseline / --impl reference legs of
 * bench.py may load it.  The product library (paper_2304_13398_b200/) never
 * links, imports or calls it, and it shares no code, header, table or helper
 * with the product: the truth tables below are typed in from the paper, the
 * gate functions are composed from them as the paper says, and the simulation
 * loop is Algorithm 2 written out line by line.
 *
 * Single-threaded, int64 picosecond times, values coded 0,1,X=2,Z=3.
 *
 * Citations: PAPER.md line numbers (P:n), with the section / equation /
 * algorithm they fall in.  Readings of points the paper leaves open are listed
 * in DESIGN.md §3 ("readings") and referenced here as R1..R16.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { V0 = 0, V1 = 1, VX = 2, VZ = 3 };
enum { G_BUF = 0, G_NOT, G_AND, G_NAND, G_OR, G_NOR, G_XOR, G_XNOR, G_MUX2 };
enum { RISE = 0, FALL = 1 };

enum { OR_OK = 0, OR_EINVAL = -1, OR_ECYCLE = -2, OR_ENOMEM = -3 };

/* ---------------------------------------------------------------------------
 * §2.2 4-value logic.  Table 1, typed in row by row:
 * TT[a][b], a = row operand, b = column operand, over the order 0,1,X,Z.
 * ------------------------------------------------------------------------- */
static const uint8_t TT_AND[4][4] = {
    /*        0   1   X   Z */
    /* 0 */ {V0, V0, V0, V0},
    /* 1 */ {V0, V1, VX, VX},
    /* X */ {V0, VX, VX, VX},
    /* Z */ {V0, VX, VX, VX},
};
static const uint8_t TT_OR[4][4] = {
    /* 0 */ {V0, V1, VX, VX},
    /* 1 */ {V1, V1, V1, V1},
    /* X */ {VX, V1, VX, VX},
    /* Z */ {VX, V1, VX, VX},
};
static const uint8_t TT_XOR[4][4] = {
    /* 0 */ {V0, V1, VX, VX},
    /* 1 */ {V1, V0, VX, VX},
    /* X */ {VX, VX, VX, VX},
    /* Z */ {VX, VX, VX, VX},
};

/* "value Z is regarded as X". */
static uint8_t norm_z(uint8_t v) { return v == VZ ? VX : v; }

/* NOT: 0->1, 1->0, X->X; Z is regarded as X. */
static uint8_t not4(uint8_t v)
{
    v = norm_z(v);
    return v == V0 ? V1 : (v == V1 ? V0 : VX);
}

/* n-ary AND/OR/XOR: left fold of the binary Table-1 operator (reading R10). */
static uint8_t fold(const uint8_t tt[4][4], const uint8_t *v, int n)
{
    uint8_t acc = norm_z(v[0]);
    for (int i = 1; i < n; i++) acc = tt[acc][v[i]];
    return acc;
}

/* Module function of a basic gate (§3.3: cell functions are
 * compositions of basic-gate functions).  N-gates = NOT of the base gate;
 * MUX2(a,b,s) = OR(AND(a,NOT s), AND(b,s)) (reading R11). */
static uint8_t eval_gate(int type, const uint8_t *v, int n)
{
    switch (type) {
    case G_BUF: return norm_z(v[0]);
    case G_NOT: return not4(v[0]);
    case G_AND: return fold(TT_AND, v, n);
    case G_NAND: return not4(fold(TT_AND, v, n));
    case G_OR: return fold(TT_OR, v, n);
    case G_NOR: return not4(fold(TT_OR, v, n));
    case G_XOR: return fold(TT_XOR, v, n);
    case G_XNOR: return not4(fold(TT_XOR, v, n));
    case G_MUX2: {
        uint8_t a = v[0], b = v[1], s = v[2];
        uint8_t l = TT_AND[a][not4(s)];
        uint8_t r = TT_AND[b][s];
        return TT_OR[l][r];
    }
    }
    return VX;
}

/* Exported for the truth-table tests. */
int oracle_eval_gate(int type, const uint8_t *v, int n)
{
    return eval_gate(type, v, n);
}

/* Edge of an input transition (P:145 posedge/negedge; reading R2: after Z->X,
 * order 0 < X < 1, RISE iff the new value ranks higher). */
static int rank01x(uint8_t v) { return v == V0 ? 0 : (v == V1 ? 2 : 1); }

/* ---------------------------------------------------------------------------
 * Waveforms: list of (t, v), strictly increasing t (§2.1).
 * ------------------------------------------------------------------------- */
typedef struct {
    int64_t *t;
    uint8_t *v;
    int64_t n, cap;
} wave_t;

static int wave_push(wave_t *w, int64_t t, uint8_t v)
{
    if (w->n == w->cap) {
        int64_t nc = w->cap ? 2 * w->cap : 16;
        int64_t *nt = (int64_t *)realloc(w->t, (size_t)nc * sizeof(int64_t));
        if (!nt) return OR_ENOMEM;
        w->t = nt;
        uint8_t *nv = (uint8_t *)realloc(w->v, (size_t)nc);
        if (!nv) return OR_ENOMEM;
        w->v = nv;
        w->cap = nc;
    }
    w->t[w->n] = t;
    w->v[w->n] = v;
    w->n++;
    return OR_OK;
}

/* addSignalChange (Alg. 2 line "addSignalChange") with the glitch-eaten
 * rule of Eq. 1: the new schedule (determined later, t_d > t_d')
 * denies every pending schedule whose appearance time t_r' >= t_r.  If the new
 * value then equals the signal it would follow, nothing changes (Fig. 3
 * caption).  The signal before any transition is X (Alg. 2 line 1,
 * P:437; reading R6).  Recursive denial in 4-value logic: P:508. */
static int add_signal_change(wave_t *out, int64_t tr, uint8_t v)
{
    while (out->n > 0 && out->t[out->n - 1] >= tr) out->n--;
    uint8_t prev = out->n > 0 ? out->v[out->n - 1] : VX;
    if (prev == v) return OR_OK;
    return wave_push(out, tr, v);
}

typedef struct {
    int64_t gate_evals;   /* distinct input timestamps swept (one per calculateSignals) */
    int64_t events;       /* output changes of the zero-delay evaluation */
    int64_t out_trans;    /* transitions stored on gate outputs after clipping */
} ostats_t;

/* Algorithm 2 for one single-output basic gate.
 *   in[i]      input waveform W_in^i
 *   d[i*4 + e*2 + o] = Delay[i][e][o], e in {RISE,FALL}, o in {0,1};
 *     for an output change to X the delay is min over o (reading R1).
 *   duration   transitions appearing after it are dropped (reading R7). */
static int process_cell(int type, int k, const wave_t *const *in, const uint32_t *d,
                        int64_t duration, wave_t *out, ostats_t *st)
{
    uint8_t cur[4];       /* currentSignals of the inputs, Z kept as read     */
    int edge[4];          /* transition edge e_i recorded at this timestamp   */
    int64_t idx[4];       /* earliestIndex                                    */
    for (int i = 0; i < k; i++) {
        cur[i] = VX;      /* currentSignals = {X, X, ..., X}          */
        idx[i] = 0;       /* earliestIndex = {1, ..., 1} (0-based here)       */
    }
    uint8_t out_sig = VX; /* the output's currentSignals entry  */
    const int64_t INF = INT64_MAX;

    for (;;) {
        /* t_earliest = min over earliestTimestamp */
        int64_t te = INF;
        for (int i = 0; i < k; i++)
            if (idx[i] < in[i]->n && in[i]->t[idx[i]] < te) te = in[i]->t[idx[i]];
        if (te == INF) break;
        st->gate_evals++;

        /* apply every input transition at t_earliest, record its edge
         * (P:452-469).  Only inputs whose value (Z read as X) changes at this
         * timestamp take part in the delay minimum (reading R3). */
        int changed[4] = {0, 0, 0, 0};
        for (int i = 0; i < k; i++) {
            if (idx[i] < in[i]->n && in[i]->t[idx[i]] == te) {
                uint8_t nv = in[i]->v[idx[i]];
                uint8_t a = norm_z(cur[i]), b = norm_z(nv);
                if (a != b) {
                    changed[i] = 1;
                    edge[i] = rank01x(b) > rank01x(a) ? RISE : FALL;
                }
                cur[i] = nv;
                idx[i]++;
            }
        }
        /* newSignals = calculateSignals(currentSignals) */
        uint8_t o = eval_gate(type, cur, k);
        /* "if o_k.v is changed" — relative to the previous evaluation
         * (reading R4a) */
        if (o != out_sig) {
            st->events++;
            /* del_k = min over inputs of Delay[i][k][e_i][o_k.v] (P:475-479,
             * P:210 "the minimal one ... shall be chosen") */
            int64_t del = INF;
            for (int i = 0; i < k; i++) {
                if (!changed[i]) continue;
                const uint32_t *di = d + i * 4 + edge[i] * 2;
                int64_t x = (o == VX) ? (di[0] < di[1] ? di[0] : di[1]) : di[o];
                if (x < del) del = x;
            }
            /* o_k.t = t_earliest + del_k; addSignalChange */
            int rc = add_signal_change(out, te + del, o);
            if (rc) return rc;
        }
        out_sig = o; /* currentSignals = newSignals */
    }
    /* waveforms live within the duration (reading R7) */
    while (out->n > 0 && out->t[out->n - 1] > duration) out->n--;
    st->out_trans += out->n;
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Multi-output cells (§3.2 Delay P:329-333, §3.3 Module Function P:335-339).
 *
 * A cell template is a small DAG of basic gates over the cell's input pins (the
 * paper's standard cell template / UDP: "implement the logic functions of all basic
 * logic gates and combine them according to the requirement of any standard cell
 * template"); its outputs are some of the DAG's nodes, evaluated with zero
 * internal delay.  Node ids: 0..n_in-1 the cell inputs, n_in + j basic gate j (its
 * fan-in nodes < n_in + j).  Delays: the 5-D matrix Delay[cell][in][out][edge][value]
 * (P:331), one [n_in][n_out][2][2] block per cell instance; DELAY_INF = "no relation"
 * (P:331-333): such pins do not enter the minimum, and an output change whose changed
 * pins are all unrelated is not scheduled (reading R9: literal Alg. 2 — the evaluation
 * still advances, "currentSignals = newSignals").
 * ------------------------------------------------------------------------- */
#define DELAY_INF 0xFFFFFFFFu
enum { CELL_MAX_IN = 4, CELL_MAX_OUT = 8, CELL_MAX_GATES = 64 };

typedef struct {
    int32_t n_in, n_out, n_gates;
    const uint8_t *gate_type;      /* [n_gates] */
    const int32_t *gate_fanin_off; /* [n_gates + 1] */
    const int32_t *gate_fanin;     /* node ids */
    const int32_t *output_node;    /* [n_out] */
} oracle_template_t;

/* the template's outputs for input values v[0..n_in-1] (Table 1 per basic gate) */
static void eval_template(const oracle_template_t *t, const uint8_t *v, uint8_t *o)
{
    uint8_t node[CELL_MAX_IN + CELL_MAX_GATES];
    for (int i = 0; i < t->n_in; i++) node[i] = v[i];
    for (int j = 0; j < t->n_gates; j++) {
        uint8_t x[4];
        int k = t->gate_fanin_off[j + 1] - t->gate_fanin_off[j];
        for (int q = 0; q < k; q++) x[q] = node[t->gate_fanin[t->gate_fanin_off[j] + q]];
        node[t->n_in + j] = eval_gate(t->gate_type[j], x, k);
    }
    for (int q = 0; q < t->n_out; q++) o[q] = norm_z(node[t->output_node[q]]);
}

/* Algorithm 2 for one cell: all its outputs from one sweep of its inputs.
 *   d[((i * n_out + q) * 2 + e) * 2 + o] = Delay[i][q][e][o]  (DELAY_INF: no relation) */
static int process_multi(const oracle_template_t *t, const wave_t *const *in, const uint32_t *d,
                         int64_t duration, wave_t *const *out, ostats_t *st)
{
    const int k = t->n_in, m = t->n_out;
    uint8_t cur[CELL_MAX_IN];
    int edge[CELL_MAX_IN];
    int64_t idx[CELL_MAX_IN];
    uint8_t out_sig[CELL_MAX_OUT], o[CELL_MAX_OUT];
    for (int i = 0; i < k; i++) { cur[i] = VX; idx[i] = 0; }
    for (int q = 0; q < m; q++) out_sig[q] = VX;
    const int64_t INF = INT64_MAX;
    for (;;) {
        int64_t te = INF;
        for (int i = 0; i < k; i++)
            if (idx[i] < in[i]->n && in[i]->t[idx[i]] < te) te = in[i]->t[idx[i]];
        if (te == INF) break;
        st->gate_evals += m;               /* one calculateSignals per output */
        int changed[CELL_MAX_IN] = {0, 0, 0, 0};
        for (int i = 0; i < k; i++) {
            if (idx[i] < in[i]->n && in[i]->t[idx[i]] == te) {
                uint8_t nv = in[i]->v[idx[i]];
                uint8_t a = norm_z(cur[i]), b = norm_z(nv);
                if (a != b) {
                    changed[i] = 1;
                    edge[i] = rank01x(b) > rank01x(a) ? RISE : FALL;
                }
                cur[i] = nv;
                idx[i]++;
            }
        }
        eval_template(t, cur, o);
        for (int q = 0; q < m; q++) {
            if (o[q] != out_sig[q]) {                  /* P:473, reading R4a */
                st->events++;
                int64_t del = INF;                      /* min over related changed pins */
                for (int i = 0; i < k; i++) {
                    if (!changed[i]) continue;
                    const uint32_t *di = d + ((i * m + q) * 2 + edge[i]) * 2;
                    uint32_t x = (o[q] == VX) ? (di[0] < di[1] ? di[0] : di[1]) : di[o[q]];
                    if (x != DELAY_INF && (int64_t)x < del) del = x;
                }
                if (del != INF) {                       /* reading R9: unrelated -> not scheduled */
                    int rc = add_signal_change(out[q], te + del, o[q]);
                    if (rc) return rc;
                }
            }
            out_sig[q] = o[q];
        }
    }
    for (int q = 0; q < m; q++) {
        while (out[q]->n > 0 && out[q]->t[out[q]->n - 1] > duration) out[q]->n--;   /* reading R7 */
        st->out_trans += out[q]->n;
    }
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Whole netlist: §2.1 objective.  Nets 0..P-1 are the given
 * waveforms (primary / pseudo-primary inputs); net P+g is the output of gate
 * g.  Gates are processed once all their input waveforms are known (Alg. 1's
 * unlock rule), here in a plain Kahn topological order since the
 * oracle is serial (the paper's t_serial baseline).
 * ------------------------------------------------------------------------- */
typedef struct {
    int32_t P, G;
    wave_t *w;       /* [P+G] */
    ostats_t st;
} oracle_result_t;

static uint64_t splitmix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

void oracle_free(oracle_result_t *r)
{
    if (!r) return;
    if (r->w) {
        for (int64_t i = 0; i < (int64_t)r->P + r->G; i++) {
            free(r->w[i].t);
            free(r->w[i].v);
        }
        free(r->w);
    }
    free(r);
}

static int arity_ok(int type, int64_t k)
{
    if (type == G_BUF || type == G_NOT) return k == 1;
    if (type == G_MUX2) return k == 3;
    if (type >= G_AND && type <= G_XNOR) return k >= 2 && k <= 4;
    return 0;
}

/* Returns 0 and *out on success; negative error otherwise. */
int oracle_simulate(int32_t P, int32_t G, const uint8_t *type, const int64_t *fanin_off,
                    const int32_t *fanin_net, const uint32_t *pin_delay,
                    const int64_t *in_off, const uint64_t *in_trans, int64_t duration,
                    oracle_result_t **out)
{
    *out = NULL;
    if (P < 0 || G < 0 || duration < 0) return OR_EINVAL;
    int64_t N = (int64_t)P + G;
    oracle_result_t *r = (oracle_result_t *)calloc(1, sizeof(*r));
    if (!r) return OR_ENOMEM;
    r->P = P;
    r->G = G;
    r->w = (wave_t *)calloc((size_t)(N ? N : 1), sizeof(wave_t));
    if (!r->w) { oracle_free(r); return OR_ENOMEM; }

    /* given waveforms, unpacked from (t << 2) | v */
    for (int32_t p = 0; p < P; p++) {
        for (int64_t j = in_off[p]; j < in_off[p + 1]; j++) {
            int64_t t = (int64_t)(in_trans[j] >> 2);
            uint8_t v = (uint8_t)(in_trans[j] & 3);
            if (wave_push(&r->w[p], t, v)) { oracle_free(r); return OR_ENOMEM; }
        }
    }

    for (int32_t g = 0; g < G; g++) {
        int64_t k = fanin_off[g + 1] - fanin_off[g];
        if (!arity_ok(type[g], k)) { oracle_free(r); return OR_EINVAL; }
        for (int64_t e = fanin_off[g]; e < fanin_off[g + 1]; e++)
            if (fanin_net[e] < 0 || fanin_net[e] >= N) { oracle_free(r); return OR_EINVAL; }
    }

    /* Kahn's algorithm over gates: pending[g] = number of fan-in pins driven
     * by not-yet-known gate outputs. */
    int64_t *pending = (int64_t *)calloc((size_t)(G ? G : 1), sizeof(int64_t));
    int64_t *cons_off = (int64_t *)calloc((size_t)N + 1, sizeof(int64_t));
    int64_t E = G ? fanin_off[G] : 0;
    int32_t *cons = (int32_t *)malloc((size_t)(E ? E : 1) * sizeof(int32_t));
    int32_t *queue = (int32_t *)malloc((size_t)(G ? G : 1) * sizeof(int32_t));
    if (!pending || !cons_off || !cons || !queue) {
        free(pending); free(cons_off); free(cons); free(queue);
        oracle_free(r);
        return OR_ENOMEM;
    }
    for (int32_t g = 0; g < G; g++)
        for (int64_t e = fanin_off[g]; e < fanin_off[g + 1]; e++) {
            cons_off[fanin_net[e] + 1]++;
            if (fanin_net[e] >= P) pending[g]++;
        }
    for (int64_t n = 0; n < N; n++) cons_off[n + 1] += cons_off[n];
    {
        int64_t *fill = (int64_t *)malloc((size_t)(N ? N : 1) * sizeof(int64_t));
        if (!fill) { free(pending); free(cons_off); free(cons); free(queue); oracle_free(r); return OR_ENOMEM; }
        memcpy(fill, cons_off, (size_t)N * sizeof(int64_t));
        for (int32_t g = 0; g < G; g++)
            for (int64_t e = fanin_off[g]; e < fanin_off[g + 1]; e++) cons[fill[fanin_net[e]]++] = g;
        free(fill);
    }
    int64_t qh = 0, qt = 0;
    for (int32_t g = 0; g < G; g++)
        if (pending[g] == 0) queue[qt++] = g;

    int rc = OR_OK;
    while (qh < qt) {
        int32_t g = queue[qh++];
        int k = (int)(fanin_off[g + 1] - fanin_off[g]);
        const wave_t *in[4];
        for (int i = 0; i < k; i++) in[i] = &r->w[fanin_net[fanin_off[g] + i]];
        rc = process_cell(type[g], k, in, pin_delay + 4 * fanin_off[g], duration,
                          &r->w[P + g], &r->st);
        if (rc) break;
        int64_t n = (int64_t)P + g;
        for (int64_t c = cons_off[n]; c < cons_off[n + 1]; c++)
            if (--pending[cons[c]] == 0) queue[qt++] = cons[c];
    }
    if (rc == OR_OK && qt != G) rc = OR_ECYCLE; /* combinational loop */
    free(pending); free(cons_off); free(cons); free(queue);
    if (rc) { oracle_free(r); return rc; }
    *out = r;
    return OR_OK;
}

/* Cell netlist: nets 0..P-1 given; the outputs of cell c are nets P + first[c] + q
 * (first[c] = outputs of the cells before c).  Cells in Kahn order as above. */
int oracle_simulate_cells(int32_t P, int32_t T, const int32_t *tpl_nin, const int32_t *tpl_nout,
                          const int32_t *tpl_ngates, const int32_t *tpl_gate_off, const uint8_t *tpl_gate_type,
                          const int32_t *tpl_fanin_off, const int32_t *tpl_fanin, const int32_t *tpl_out_off,
                          const int32_t *tpl_out_node, int32_t C, const int32_t *cell_tpl,
                          const int32_t *cell_fanin, const uint32_t *cell_delay, const int64_t *in_off,
                          const uint64_t *in_trans, int64_t duration, oracle_result_t **out)
{
    *out = NULL;
    if (P < 0 || T < 0 || C < 0 || duration < 0) return OR_EINVAL;
    oracle_template_t *tp = (oracle_template_t *)calloc((size_t)(T ? T : 1), sizeof(oracle_template_t));
    if (!tp) return OR_ENOMEM;
    for (int32_t i = 0; i < T; i++) {
        tp[i].n_in = tpl_nin[i];
        tp[i].n_out = tpl_nout[i];
        tp[i].n_gates = tpl_ngates[i];
        tp[i].gate_type = tpl_gate_type + tpl_gate_off[i];
        tp[i].gate_fanin_off = tpl_fanin_off + tpl_gate_off[i] + i;   /* n_gates + 1 entries each */
        tp[i].gate_fanin = tpl_fanin;
        tp[i].output_node = tpl_out_node + tpl_out_off[i];
        if (tp[i].n_in < 1 || tp[i].n_in > CELL_MAX_IN || tp[i].n_out < 1 || tp[i].n_out > CELL_MAX_OUT ||
            tp[i].n_gates < 0 || tp[i].n_gates > CELL_MAX_GATES) { free(tp); return OR_EINVAL; }
    }
    int64_t *first = (int64_t *)calloc((size_t)C + 1, sizeof(int64_t));
    int64_t *pin0 = (int64_t *)calloc((size_t)C + 1, sizeof(int64_t));
    int64_t *dly0 = (int64_t *)calloc((size_t)C + 1, sizeof(int64_t));
    if (!first || !pin0 || !dly0) { free(tp); free(first); free(pin0); free(dly0); return OR_ENOMEM; }
    for (int32_t c = 0; c < C; c++) {
        if (cell_tpl[c] < 0 || cell_tpl[c] >= T) { free(tp); free(first); free(pin0); free(dly0); return OR_EINVAL; }
        const oracle_template_t *t = &tp[cell_tpl[c]];
        first[c + 1] = first[c] + t->n_out;
        pin0[c + 1] = pin0[c] + t->n_in;
        dly0[c + 1] = dly0[c] + (int64_t)t->n_in * t->n_out * 4;
    }
    const int64_t G = first[C], N = (int64_t)P + G;
    oracle_result_t *r = (oracle_result_t *)calloc(1, sizeof(*r));
    int64_t *pending = (int64_t *)calloc((size_t)(C ? C : 1), sizeof(int64_t));
    int64_t *cons_off = (int64_t *)calloc((size_t)N + 1, sizeof(int64_t));
    int32_t *cons = (int32_t *)malloc((size_t)(pin0[C] ? pin0[C] : 1) * sizeof(int32_t));
    int32_t *queue = (int32_t *)malloc((size_t)(C ? C : 1) * sizeof(int32_t));
    int32_t *owner = (int32_t *)malloc((size_t)(G ? G : 1) * sizeof(int32_t));
    int rc = OR_OK;
    if (!r || !pending || !cons_off || !cons || !queue || !owner) rc = OR_ENOMEM;
    if (!rc) {
        r->P = P;
        r->G = (int32_t)G;
        r->w = (wave_t *)calloc((size_t)(N ? N : 1), sizeof(wave_t));
        if (!r->w) rc = OR_ENOMEM;
    }
    for (int32_t p = 0; !rc && p < P; p++)
        for (int64_t j = in_off[p]; j < in_off[p + 1] && !rc; j++)
            rc = wave_push(&r->w[p], (int64_t)(in_trans[j] >> 2), (uint8_t)(in_trans[j] & 3));
    for (int32_t c = 0; !rc && c < C; c++) {
        for (int64_t q = first[c]; q < first[c + 1]; q++) owner[q] = c;
        for (int64_t e = pin0[c]; e < pin0[c + 1]; e++) {
            if (cell_fanin[e] < 0 || cell_fanin[e] >= N) { rc = OR_EINVAL; break; }
            cons_off[cell_fanin[e] + 1]++;
            if (cell_fanin[e] >= P) pending[c]++;
        }
    }
    if (!rc) {
        for (int64_t n = 0; n < N; n++) cons_off[n + 1] += cons_off[n];
        int64_t *fill = (int64_t *)malloc((size_t)(N ? N : 1) * sizeof(int64_t));
        if (!fill) rc = OR_ENOMEM;
        else {
            memcpy(fill, cons_off, (size_t)N * sizeof(int64_t));
            for (int32_t c = 0; c < C; c++)
                for (int64_t e = pin0[c]; e < pin0[c + 1]; e++) cons[fill[cell_fanin[e]]++] = c;
            free(fill);
        }
    }
    int64_t qh = 0, qt = 0;
    for (int32_t c = 0; !rc && c < C; c++)
        if (pending[c] == 0) queue[qt++] = c;
    while (!rc && qh < qt) {
        int32_t c = queue[qh++];
        const oracle_template_t *t = &tp[cell_tpl[c]];
        const wave_t *in[CELL_MAX_IN];
        wave_t *outs[CELL_MAX_OUT];
        for (int i = 0; i < t->n_in; i++) in[i] = &r->w[cell_fanin[pin0[c] + i]];
        for (int q = 0; q < t->n_out; q++) outs[q] = &r->w[P + first[c] + q];
        rc = process_multi(t, in, cell_delay + dly0[c], duration, outs, &r->st);
        /* the cell's outputs are known: unlock the consumers (once per consuming pin) */
        for (int q = 0; !rc && q < t->n_out; q++) {
            int64_t n = (int64_t)P + first[c] + q;
            for (int64_t e = cons_off[n]; e < cons_off[n + 1]; e++)
                if (--pending[cons[e]] == 0) queue[qt++] = cons[e];
        }
    }
    if (!rc && qt != C) rc = OR_ECYCLE;
    free(tp); free(first); free(pin0); free(dly0); free(pending); free(cons_off); free(cons); free(queue); free(owner);
    if (rc) { oracle_free(r); return rc; }
    *out = r;
    return OR_OK;
}

/* Results ------------------------------------------------------------------ */
int64_t oracle_total(const oracle_result_t *r)
{
    int64_t s = 0;
    for (int64_t i = 0; i < (int64_t)r->P + r->G; i++) s += r->w[i].n;
    return s;
}

void oracle_stats(const oracle_result_t *r, int64_t *out3)
{
    out3[0] = r->st.gate_evals;
    out3[1] = r->st.events;
    out3[2] = r->st.out_trans;
}

/* Canonical CSR in net order: offsets[P+G+1], trans[total] packed (t<<2)|v. */
void oracle_get(const oracle_result_t *r, int64_t *offsets, uint64_t *trans)
{
    int64_t o = 0;
    for (int64_t i = 0; i < (int64_t)r->P + r->G; i++) {
        offsets[i] = o;
        for (int64_t j = 0; j < r->w[i].n; j++)
            trans[o++] = ((uint64_t)r->w[i].t[j] << 2) | r->w[i].v[j];
    }
    offsets[(int64_t)r->P + r->G] = o;
}

/* Per-net 64-bit results checksum (not part of the method):
 * h = splitmix64(C ^ n) XOR the XOR over positions j = 0..n-1 of
 * splitmix64(e_j + (j + 1) * K), e_j the j-th packed entry (t << 2 | v),
 * C = 0x9E3779B97F4A7C15, K = 0xD1B54A32D192ED03, arithmetic mod 2^64. */
void oracle_hashes(const oracle_result_t *r, uint64_t *h)
{
    for (int64_t i = 0; i < (int64_t)r->P + r->G; i++) {
        uint64_t x = splitmix64(0x9E3779B97F4A7C15ull ^ (uint64_t)r->w[i].n);
        for (int64_t j = 0; j < r->w[i].n; j++) {
            const uint64_t e = ((uint64_t)r->w[i].t[j] << 2) | r->w[i].v[j];
            x ^= splitmix64(e + (uint64_t)(j + 1) * 0xD1B54A32D192ED03ull);
        }
        h[i] = x;
    }
}
