/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the optimal persistent
 * checkpointing DP of arXiv 1911.13214 ("Rotor"), written from PAPER.md:
 *   - discretisation of sizes into S slots ........ §5.2
 *   - limits m_null(s,t), m_all(s,t) ............... §4.2
 *   - Theorem 1, Eq. (1) leaf and Eq. (2) .......... P:717-739
 *   - Algorithm 1 (table fill + top query) .......... P:809-826
 *   - Algorithm 2 OptRec (schedule reconstruction) .. P:829-847
 * with the readings Q3-Q13 of DESIGN.md §3.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / the
 * --impl reference arm) may load this library.  It shares no code, header,
 * table or constant with the CUDA product path (paper_1911_13214_b200/).
 *
 * Conventions (1-based stage indices as in the paper, n = L+1 stages):
 *   uf[l], ub[l], wbx[l], of[l], ob[l]   l = 1..n
 *   wx[l]                                 l = 0..L   (a^l)
 *   wy[l]                                 l = 0..n   (delta^l)
 * Memory index m = 0..S (Q6).  +inf is IEEE +INFINITY (Q13).
 * Exported table layout ("canonical", documented in include/rotor.h):
 *   cell(s,t) = (s-1)*n - (s-1)*(s-2)/2 + (t-s)  (s-major);  value at cell*(S+1) + m.
 * D (argmin) codes: k = s'-s in 1..d for an F_ck split, 0 for F_all / leaf,
 *   0xFFFF when C = +inf.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 *
 * Threads: oracle_fill_threads() runs the very same per-cell
 * computation with the cells of one diagonal d spread over OpenMP threads.  The
 * cells of a diagonal read only shorter diagonals and each cell's
 * candidate loop is unchanged, so the table is bit-identical to oracle_fill's
 * (tests/test_oracle_pins.py::test_threaded_fill_bit_identical).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_FALL 0
#define OR_FCK 1
#define OR_FNULL 2
#define OR_BWD 3
#define OR_NONE 0xFFFF

typedef struct {
    int L, n, S, restricted;
    uint64_t M;
    /* discretised sizes (slots), 1-based where the paper is */
    int64_t *wx, *wbx, *wy, *of, *ob;
    double *uf, *ub;
    double *P; /* P[k] = uf[1] + ... + uf[k] (sequential), k = 0..n   (Q12) */
    double *w; /* w[s] = uf[s] + ub[s]                                  (Q12) */
    int64_t *mnull, *mall; /* [(n+1)*(n+1)], index s*(n+1)+t */
    double *C;             /* [cells*(S+1)] */
    uint16_t *D;           /* [cells*(S+1)] */
    int64_t cells;
    /* window: only cells with s0 <= s <= t <= s0+nw-1 are stored and filled
     * (default: the whole chain, s0 = 1, nw = n).  Every such cell depends only
     * on cells of the same window, and the prefix sums P stay those
     * of the whole chain, so windowed values are bit-identical to full ones. */
    int s0, nw;
    int filled;
    int keep_d; /* store the fill's argmin table D (default 1) */
    /* reconstruction output */
    int32_t *ops;
    int64_t ops_cap, ops_n;
    int truncated;
} oracle_ctx;

/* ---- §5.2 discretisation: slots(x) = ceil(x / (M/S)) = ceil(x*S/M), exact (Q7) ---- */
static int64_t slots_of(uint64_t x, uint64_t M, int S)
{
    unsigned __int128 num = (unsigned __int128)x * (unsigned __int128)(unsigned)S;
    unsigned __int128 q = (num + M - 1) / M;
    const unsigned __int128 cap = (unsigned __int128)1 << 40; /* any value > S behaves alike; avoids overflow */
    return (int64_t)(q > cap ? cap : q);
}

static int64_t cell_index(const oracle_ctx *c, int s, int t)
{
    int64_t r = s - c->s0; /* s-major: row r holds cells (s, s..s0+nw-1) */
    return r * c->nw - r * (r - 1) / 2 + (t - s);
}

static double *Cp(oracle_ctx *c, int s, int t) { return c->C + cell_index(c, s, t) * (int64_t)(c->S + 1); }
static uint16_t *Dp(oracle_ctx *c, int s, int t) { return c->D + cell_index(c, s, t) * (int64_t)(c->S + 1); }

/* C[s,t,m] with the Q6 convention: a lookup below m = 0 is +inf. */
static double Cget(oracle_ctx *c, int s, int t, int64_t m)
{
    if (m < 0) return INFINITY;
    return Cp(c, s, t)[m];
}

static int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

void oracle_free(oracle_ctx *c)
{
    if (!c) return;
    free(c->wx); free(c->wbx); free(c->wy); free(c->of); free(c->ob);
    free(c->uf); free(c->ub); free(c->P); free(c->w);
    free(c->mnull); free(c->mall); free(c->C); free(c->D); free(c->ops);
    free(c);
}

/*
 * Build the discretised chain, the prefix sums and the two limit tables.
 * Input arrays use the rotor_chain indexing of include/rotor.h (0-based storage
 * of 1-based stages: uf[l-1] is stage l; wx[l] is a^l; wy[l] is delta^l).
 */
oracle_ctx *oracle_new(int L, int S, const double *uf, const double *ub, const uint64_t *wx,
                       const uint64_t *wbx, const uint64_t *wy, const uint64_t *of, const uint64_t *ob,
                       uint64_t M, int restricted)
{
    if (L < 1 || S < 1 || M == 0) return NULL;
    oracle_ctx *c = (oracle_ctx *)calloc(1, sizeof(oracle_ctx));
    if (!c) return NULL;
    int n = L + 1;
    c->L = L; c->n = n; c->S = S; c->M = M; c->restricted = restricted;
    c->wx = calloc(n + 2, sizeof(int64_t));
    c->wbx = calloc(n + 2, sizeof(int64_t));
    c->wy = calloc(n + 2, sizeof(int64_t));
    c->of = calloc(n + 2, sizeof(int64_t));
    c->ob = calloc(n + 2, sizeof(int64_t));
    c->uf = calloc(n + 2, sizeof(double));
    c->ub = calloc(n + 2, sizeof(double));
    c->P = calloc(n + 2, sizeof(double));
    c->w = calloc(n + 2, sizeof(double));
    c->mnull = calloc((size_t)(n + 2) * (n + 2), sizeof(int64_t));
    c->mall = calloc((size_t)(n + 2) * (n + 2), sizeof(int64_t));
    if (!c->wx || !c->wbx || !c->wy || !c->of || !c->ob || !c->uf || !c->ub || !c->P || !c->w ||
        !c->mnull || !c->mall) {
        oracle_free(c);
        return NULL;
    }
    for (int l = 0; l <= L; l++) c->wx[l] = slots_of(wx[l], M, S);
    for (int l = 0; l <= n; l++) c->wy[l] = slots_of(wy[l], M, S);
    for (int l = 1; l <= n; l++) {
        c->wbx[l] = slots_of(wbx[l - 1], M, S);
        c->of[l] = slots_of(of[l - 1], M, S);
        c->ob[l] = slots_of(ob[l - 1], M, S);
        c->uf[l] = uf[l - 1];
        c->ub[l] = ub[l - 1];
    }
    /* Q12: P[k] = fl(P[k-1] + uf[k]) sequentially; w[s] = fl(uf[s] + ub[s]). */
    c->P[0] = 0.0;
    for (int k = 1; k <= n; k++) c->P[k] = c->P[k - 1] + c->uf[k];
    for (int s = 1; s <= n; s++) c->w[s] = c->uf[s] + c->ub[s];

    /* §4.2 limits, literal maxima. */
    for (int s = 1; s <= n; s++) {
        for (int t = s; t <= n; t++) {
            /* m_all(s,t) = max(wy[t] + wbx[s] + of[s], wy[s] + wbx[s] + ob[s]) */
            c->mall[s * (n + 2) + t] = max64(c->wy[t] + c->wbx[s] + c->of[s], c->wy[s] + c->wbx[s] + c->ob[s]);
            if (t > s) {
                /* m_null(s,t) = max(wy[t] + wx[s] + of[s],
                 *                   wy[t] + max_{s+1 <= j < t} (wx[j-1] + wx[j] + of[j])) */
                int64_t v = c->wy[t] + c->wx[s] + c->of[s];
                for (int j = s + 1; j < t; j++) v = max64(v, c->wy[t] + c->wx[j - 1] + c->wx[j] + c->of[j]);
                c->mnull[s * (n + 2) + t] = v;
            }
        }
    }
    c->s0 = 1;
    c->nw = n;
    c->cells = (int64_t)n * (n + 1) / 2;
    c->keep_d = 1;
    return c;
}

/* Restrict storage and fill to the window of stages s0..t0 (call before oracle_fill). */
int oracle_set_window(oracle_ctx *c, int s0, int t0)
{
    if (c->filled || s0 < 1 || t0 > c->n || s0 > t0) return -1;
    c->s0 = s0;
    c->nw = t0 - s0 + 1;
    c->cells = (int64_t)c->nw * (c->nw + 1) / 2;
    return 0;
}

static int64_t MNULL(const oracle_ctx *c, int s, int t) { return c->mnull[s * (c->n + 2) + t]; }
static int64_t MALL(const oracle_ctx *c, int s, int t) { return c->mall[s * (c->n + 2) + t]; }

/* C_ck(s, s', t, m) = sum_{k=s}^{s'-1} uf[k] + C[s', t, m - wx[s'-1]] + C[s, s'-1, m]
 * evaluated as fl(fl(U + C[s,s'-1,m]) + C[s',t,m-wx[s'-1]]) with U = fl(P[s'-1] - P[s-1]) (Q12). */
static double C_ck(oracle_ctx *c, int s, int sp, int t, int64_t m)
{
    double U = c->P[sp - 1] - c->P[s - 1];
    double pre = Cget(c, s, sp - 1, m);
    double suf = Cget(c, sp, t, m - c->wx[sp - 1]);
    return (U + pre) + suf;
}

/* C_all(s,t,m) = uf[s] + C[s+1, t, m - wbx[s]] + ub[s], as fl(w[s] + C[...]) (Q12). */
static double C_all(oracle_ctx *c, int s, int t, int64_t m)
{
    return c->w[s] + Cget(c, s + 1, t, m - c->wbx[s]);
}

/*
 * Algorithm 1, with the fill order of Q3: by increasing d = t - s
 * (Alg. 1's s-outer loop would read C[s',t] for s' > s before it is written).
 * For each cell the candidates are visited in Alg. 2's order (Q11): F_ck with
 * s' = s+1..t ascending under strict '<' (smallest s' wins a tie), then F_all
 * only if strictly smaller.  The loop over m is innermost for speed; for every
 * fixed m the candidate order is exactly the one above, so the result is the
 * same as the literal per-cell loop.
 */
/* One cell (s, t=s+d) of Eq. (2) for every m, into C (and D when kept).
 * best/arg are caller-provided scratch rows of S+1 entries. */
static void fill_cell(oracle_ctx *c, int s, int t, double *best, int *arg)
{
    const int S = c->S;
    int64_t mn = MNULL(c, s, t), ma = MALL(c, s, t);
    for (int m = 0; m <= S; m++) { best[m] = INFINITY; arg[m] = OR_NONE; }
    /* C_1: min over s' of C_ck, only where m >= m_null(s,t) */
    for (int sp = s + 1; sp <= t; sp++) {
        for (int m = 0; m <= S; m++) {
            if (m < mn) continue;
            double v = C_ck(c, s, sp, t, m);
            if (v < best[m]) { best[m] = v; arg[m] = sp - s; }
        }
    }
    /* C_2: C_all where m >= m_all(s,t); not at s < t in restricted mode */
    if (!c->restricted) {
        for (int m = 0; m <= S; m++) {
            if (m < ma) continue;
            double v = C_all(c, s, t, m);
            if (v < best[m]) { best[m] = v; arg[m] = 0; }
        }
    }
    double *Cst = Cp(c, s, t);
    for (int m = 0; m <= S; m++) Cst[m] = best[m]; /* Eq. (2): C = min(C_1, C_2) */
    if (c->D) {
        uint16_t *Dst = Dp(c, s, t);
        for (int m = 0; m <= S; m++) Dst[m] = isinf(best[m]) ? OR_NONE : (uint16_t)arg[m];
    }
}

/*
 * Algorithm 1, with the fill order of Q3: by increasing d = t - s
 * (Alg. 1's s-outer loop would read C[s',t] for s' > s before it is written).
 * For each cell the candidates are visited in Alg. 2's order (Q11): F_ck with
 * s' = s+1..t ascending under strict '<' (smallest s' wins a tie), then F_all
 * only if strictly smaller.  The loop over m is innermost for speed; for every
 * fixed m the candidate order is exactly the one above, so the result is the
 * same as the literal per-cell loop.  nthreads > 1 spreads the independent
 * cells of one diagonal over OpenMP threads (same per-cell arithmetic).
 */
int oracle_fill_threads(oracle_ctx *c, int nthreads)
{
    const int S = c->S, W = S + 1;
    const int s_lo = c->s0, s_hi = c->s0 + c->nw - 1; /* window (whole chain by default) */
    if (nthreads < 1) nthreads = 1;
    if (!c->C) {
        c->C = (double *)malloc((size_t)c->cells * W * sizeof(double));
        if (!c->C) return -1;
        if (c->keep_d) {
            c->D = (uint16_t *)malloc((size_t)c->cells * W * sizeof(uint16_t));
            if (!c->D) return -1;
        }
    }
    /* Eq. (1): C[s,s,m] = uf[s] + ub[s] if m >= m_all(s,s) else +inf */
    for (int s = s_lo; s <= s_hi; s++) {
        double *Cs = Cp(c, s, s);
        int64_t ma = MALL(c, s, s);
        for (int m = 0; m <= S; m++) Cs[m] = (m >= ma) ? c->w[s] : INFINITY;
        if (c->D) {
            uint16_t *Ds = Dp(c, s, s);
            for (int m = 0; m <= S; m++) Ds[m] = (m >= ma) ? 0 : OR_NONE;
        }
    }
    double *best = (double *)malloc((size_t)nthreads * W * sizeof(double));
    int *arg = (int *)malloc((size_t)nthreads * W * sizeof(int));
    if (!best || !arg) { free(best); free(arg); return -1; }
    for (int d = 1; d <= s_hi - s_lo; d++) {
        int n_cells = s_hi - d - s_lo + 1;
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1) if (nthreads > 1)
        for (int i = 0; i < n_cells; i++) {
            int tid = 0;
#ifdef _OPENMP
            tid = omp_get_thread_num();
#endif
            int s = s_lo + i;
            fill_cell(c, s, s + d, best + (size_t)tid * W, arg + (size_t)tid * W);
        }
    }
    free(best);
    free(arg);
    c->filled = 1;
    return 0;
}

int oracle_fill(oracle_ctx *c) { return oracle_fill_threads(c, 1); }

/* Keep (1, default) or drop (0) the fill's argmin table D; call before filling.
 * Algorithm 2 (oracle_decision / oracle_reconstruct) needs only C. */
int oracle_set_keep_d(oracle_ctx *c, int keep)
{
    if (c->filled || c->C) return -1;
    c->keep_d = keep ? 1 : 0;
    return 0;
}

/* Borrowed pointer to the filled C table (canonical layout, cells x (S+1)). */
const double *oracle_table(const oracle_ctx *c) { return c->filled ? c->C : NULL; }

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int64_t oracle_m_top(const oracle_ctx *c) { return (int64_t)c->S - c->wx[0]; } /* Q5, Alg. 1 */

double oracle_cost(oracle_ctx *c)
{
    int64_t mt = oracle_m_top(c);
    if (mt < 0 || !c->filled || c->s0 != 1 || c->nw != c->n) return INFINITY;
    return Cget(c, 1, c->n, mt);
}

double oracle_cell(oracle_ctx *c, int s, int t, int64_t m) { return Cget(c, s, t, m); }

/*
 * The decision Algorithm 2 takes at (s,t,m): the smallest s' with
 * C[s,t,m] = C_ck(s,s',t,m) (C_1 exists only where m >= m_null), else F_all.
 * Returns k = s'-s, 0 for F_all / leaf, OR_NONE when C = +inf.
 */
int oracle_decision(oracle_ctx *c, int s, int t, int64_t m)
{
    double v = Cget(c, s, t, m);
    if (isinf(v)) return OR_NONE;
    if (s == t) return 0;
    if (m >= MNULL(c, s, t))
        for (int sp = s + 1; sp <= t; sp++)
            if (C_ck(c, s, sp, t, m) == v) return sp - s;
    return 0;
}

static void emit(oracle_ctx *c, int op, int stage)
{
    if (c->ops_n < c->ops_cap) {
        c->ops[2 * c->ops_n] = op;
        c->ops[2 * c->ops_n + 1] = stage;
    } else {
        c->truncated = 1;
    }
    c->ops_n++;
}

/* Algorithm 2, OptRec(C, s, t, m), with the F_null range of Q4: F_null^{s+1..s'-1}. */
static int opt_rec(oracle_ctx *c, int s, int t, int64_t m)
{
    if (m < 0 || isinf(Cget(c, s, t, m))) return -1; /* "Return Infeasible" */
    if (s == t) {
        emit(c, OR_FALL, s);
        emit(c, OR_BWD, s);
        return 0;
    }
    int k = oracle_decision(c, s, t, m);
    if (k >= 1) {
        int sp = s + k;
        emit(c, OR_FCK, s);
        for (int j = s + 1; j <= sp - 1; j++) emit(c, OR_FNULL, j);
        if (opt_rec(c, sp, t, m - c->wx[sp - 1])) return -1;
        return opt_rec(c, s, sp - 1, m);
    }
    if (c->restricted) return -2; /* cannot happen: restricted mode has no F_all at s < t */
    emit(c, OR_FALL, s);
    if (opt_rec(c, s + 1, t, m - c->wbx[s])) return -1;
    emit(c, OR_BWD, s);
    return 0;
}

/* Reconstruct the schedule of cell (s,t,m) into ops[2*i] = opcode, ops[2*i+1] = stage.
 * Returns the op count (may exceed cap: then only cap ops were written), -1 if infeasible. */
int64_t oracle_reconstruct(oracle_ctx *c, int s, int t, int64_t m, int32_t *ops, int64_t cap)
{
    if (!c->filled) return -3;
    c->ops = ops; /* borrowed for the duration of the call */
    c->ops_n = 0;
    c->ops_cap = ops ? cap : 0;
    c->truncated = 0;
    int r = opt_rec(c, s, t, m);
    c->ops = NULL;
    if (r) return r == -2 ? -2 : -1;
    return c->ops_n;
}

/* Export C (fp64) and D (uint16) in the canonical layout; either pointer may be NULL. */
int oracle_export(oracle_ctx *c, double *C, uint16_t *D)
{
    if (!c->filled || (D && !c->D)) return -1;
    size_t cnt = (size_t)c->cells * (c->S + 1);
    if (C) memcpy(C, c->C, cnt * sizeof(double));
    if (D) memcpy(D, c->D, cnt * sizeof(uint16_t));
    return 0;
}

/* Algorithm-2 decisions for every cell (same layout as D), for the D_fill == D_rec self-check. */
int oracle_decision_table(oracle_ctx *c, uint16_t *out)
{
    if (!c->filled) return -1;
    for (int d = 0; d < c->nw; d++)
        for (int s = c->s0; s + d <= c->s0 + c->nw - 1; s++) {
            int t = s + d;
            uint16_t *o = out + cell_index(c, s, t) * (int64_t)(c->S + 1);
            for (int m = 0; m <= c->S; m++) o[m] = (uint16_t)oracle_decision(c, s, t, m);
        }
    return 0;
}

/* Discretised sizes and limits, for the simulator / brute force and tests.
 * Arrays are 1-based like the paper: caller passes arrays of length n+2. */
void oracle_slots(const oracle_ctx *c, int64_t *wx, int64_t *wbx, int64_t *wy, int64_t *of, int64_t *ob)
{
    for (int i = 0; i <= c->n + 1; i++) {
        if (wx) wx[i] = c->wx[i];
        if (wbx) wbx[i] = c->wbx[i];
        if (wy) wy[i] = c->wy[i];
        if (of) of[i] = c->of[i];
        if (ob) ob[i] = c->ob[i];
    }
}

int64_t oracle_mnull(const oracle_ctx *c, int s, int t) { return MNULL(c, s, t); }
int64_t oracle_mall(const oracle_ctx *c, int s, int t) { return MALL(c, s, t); }
int64_t oracle_cells(const oracle_ctx *c) { return c->cells; }

/* Standalone discretisation helper for the P10 pins. */
int64_t oracle_slots_of(uint64_t x, uint64_t M, int S) { return slots_of(x, M, S); }
