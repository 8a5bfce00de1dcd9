/*
 * seqcfr_oracle.c — CPU restatement of the reference seqcfr iteration.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker for the CUDA path and the
 * `cpu_baseline` / `--impl reference` arm of bench.py; nothing in the
 * product (paper_2605_14277_b200/) links or calls it.  Parity of this file
 * with the reference is pinned by tests/test_oracle.py against the golden
 * fixtures that scripts/make_golden.py produced by running the reference
 * itself (bit-exact on every lockstep case).
 *
 * It restates, per decision point (DP) instead of per node:
 *   next_strategy            pkg/solvers.py:143-175   (≡ pkg/oracle.py:45-68)
 *   observe_utility[_plus|_dcfr] pkg/solvers.py:178-224 (≡ pkg/oracle.py:71-134)
 *   next_strategy_predictive pkg/solvers.py:227-245   (≡ pkg/oracle.py:137-148)
 *   current_strategy         pkg/solvers.py:270-291
 *   _step                    pkg/solvers.py:351-372
 *   CSR SpMV                 pkg/kernels.py:148-154
 *   scalar_best_response     pkg/oracle.py:186-221
 * with the exact association order of the reference's matrix/vector path
 * (SURVEY.md §8(a)): compile with -ffp-contract=off; sums are sequential.
 *
 * REAL selects the arithmetic of the iteration state: double (default; the
 * reference's) or float (-DREAL=float, libseqcfr_oracle_f32.so: the fp32
 * mode's checker: the same operation order with every operation rounded to
 * fp32, payoffs rounded once to fp32, schedules from fp64 libm pow rounded
 * once, avg_weight summed in fp64).  Interfaces stay fp64 (widened reads).
 * Thread parallelism (pthreads) is over independent DPs of one depth level
 * and independent SpMV rows (each output written by exactly one thread, like
 * the reference's prange backend), so results are bitwise independent of the
 * thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#ifndef REAL
#define REAL double
#endif
typedef REAL real;
#define RL(v) ((real)(v))

typedef struct {
    int64_t S, J, L;          /* |Σ| (incl. empty), |J|, number of DP levels */
    int64_t *first, *parent;  /* [J+1] action ranges, [J] parent sequence */
    int64_t *clo, *ccnt;      /* [S] child-DP range per sequence */
    int64_t *lvl;             /* [L+1] DP level starts (by process depth) */
    real *r, *b, *x, *xpost, *avg, *u, *V, *W, *g;
    double avg_weight;
} oc_player;

typedef struct {
    int64_t rows, nnz;
    int64_t *indptr, *indices;
    real* data;
} oc_csr;

typedef struct {
    oc_player p[2];
    oc_csr U, UT;
    int variant, mode; /* 0 cfr 1 cfr+ 2 dcfr 3 pcfr 4 pcfr+ ; 0 sim 1 alt */
    double alpha, beta, gamma;
    int64_t t; /* reference RegretState.t (starts at 1) */
    int threads;
} oc_state;

static void* xcalloc(size_t n, size_t s) { return calloc(n ? n : 1, s); }

/* Contiguous-chunk parallel for over [lo, hi); serial below `grain`. */
typedef void (*range_fn)(void* ctx, int64_t lo, int64_t hi);
typedef struct { range_fn fn; void* ctx; int64_t lo, hi; } chunk_t;
static void* chunk_main(void* p) {
    chunk_t* c = (chunk_t*)p;
    c->fn(c->ctx, c->lo, c->hi);
    return NULL;
}
static void parfor(int64_t lo, int64_t hi, int threads, int64_t grain, range_fn fn, void* ctx) {
    const int64_t n = hi - lo;
    if (threads <= 1 || n < grain) {
        fn(ctx, lo, hi);
        return;
    }
    if (threads > 64) threads = 64;
    pthread_t tid[64];
    chunk_t ch[64];
    for (int k = 0; k < threads; ++k) {
        ch[k].fn = fn;
        ch[k].ctx = ctx;
        ch[k].lo = lo + n * k / threads;
        ch[k].hi = lo + n * (k + 1) / threads;
    }
    for (int k = 1; k < threads; ++k) pthread_create(&tid[k], NULL, chunk_main, &ch[k]);
    chunk_main(&ch[0]);
    for (int k = 1; k < threads; ++k) pthread_join(tid[k], NULL);
}

static int build_player(oc_player* P, int64_t num_nodes, int64_t S, int64_t J, const int64_t* depth,
                        const int64_t* dp_node, const int64_t* first, const int64_t* nact,
                        const int64_t* parent) {
    (void)num_nodes;
    P->S = S;
    P->J = J;
    P->first = xcalloc(J + 1, 8);
    P->parent = xcalloc(J, 8);
    P->clo = xcalloc(S, 8);
    P->ccnt = xcalloc(S, 8);
    P->lvl = xcalloc(J + 2, 8);
    int64_t L = 0, prev = -1;
    for (int64_t j = 0; j < J; ++j) {
        P->first[j] = first[j];
        P->parent[j] = parent[j];
        int64_t s = parent[j];
        if (P->ccnt[s] == 0) P->clo[s] = j;
        else if (P->clo[s] + P->ccnt[s] != j) return -1;
        P->ccnt[s]++;
        int64_t d = depth[dp_node[j]];
        if (d < prev) return -1;
        if (d != prev) P->lvl[L++] = j;
        prev = d;
    }
    P->first[J] = J ? first[J - 1] + nact[J - 1] : 1;
    P->lvl[L] = J;
    P->L = L;
    P->r = xcalloc(S, sizeof(real));
    P->b = xcalloc(S, sizeof(real));
    P->x = xcalloc(S, sizeof(real));
    P->xpost = xcalloc(S, sizeof(real));
    P->avg = xcalloc(S, sizeof(real));
    P->u = xcalloc(S, sizeof(real));
    P->V = xcalloc(J, sizeof(real));
    P->W = xcalloc(J, sizeof(real));
    P->g = xcalloc(S, sizeof(real));
    for (int64_t j = 0; j < J; ++j)
        for (int64_t s = first[j]; s < first[j] + nact[j]; ++s) P->b[s] = RL(1.0) / (real)nact[j];
    P->x[0] = RL(1.0);
    P->xpost[0] = RL(1.0);
    P->avg_weight = 0.0;
    return 0;
}

static void copy_csr(oc_csr* M, int64_t rows, int64_t nnz, const int64_t* ip, const int64_t* ix,
                     const double* d) {
    M->rows = rows;
    M->nnz = nnz;
    M->indptr = xcalloc(rows + 1, 8);
    M->indices = xcalloc(nnz, 8);
    M->data = xcalloc(nnz, sizeof(real));
    memcpy(M->indptr, ip, (rows + 1) * 8);
    if (nnz) {
        memcpy(M->indices, ix, nnz * 8);
        for (int64_t k = 0; k < nnz; ++k) M->data[k] = (real)d[k]; /* rounded once */
    }
}

/* pkg/kernels.py:148-154 (+ backend.scale(-1.0, .) when neg). */
typedef struct { const oc_csr* M; const real* x; real* out; int neg; } spmv_ctx;
static void spmv_rows(void* p, int64_t lo, int64_t hi) {
    const spmv_ctx* c = (const spmv_ctx*)p;
    const oc_csr* M = c->M;
    for (int64_t i = lo; i < hi; ++i) {
        real acc = RL(0.0);
        for (int64_t k = M->indptr[i]; k < M->indptr[i + 1]; ++k) acc += M->data[k] * c->x[M->indices[k]];
        c->out[i] = c->neg ? RL(-1.0) * acc : acc;
    }
}
static void spmv(const oc_csr* M, const real* x, real* out, int neg, int threads) {
    spmv_ctx c = {M, x, out, neg};
    parfor(0, M->rows, threads, 1 << 14, spmv_rows, &c);
}

static real child_sum(const oc_player* P, int64_t s, const real* V) {
    const int64_t c = P->ccnt[s], lo = P->clo[s];
    if (c == 0) return RL(0.0);
    if (c == 1) return V[lo];
    real acc = RL(0.0);
    for (int64_t k = 0; k < c; ++k) acc += V[lo + k];
    return acc;
}

static real qval(const oc_player* P, const real* u, int64_t s) {
    return (RL(0.0) + u[s]) + child_sum(P, s, P->V);
}

/* observe (pkg/solvers.py:178-207) + floor (:210-214) / discount (:217-224). */
typedef struct { oc_player* P; const real* u; int post; real pf, nf; } obs_ctx;
static void observe_range(void* p, int64_t lo, int64_t hi) {
    const obs_ctx* c = (const obs_ctx*)p;
    oc_player* P = c->P;
    const real* u = c->u;
    const int post = c->post;
    const real pf = c->pf, nf = c->nf;
    {
        for (int64_t j = lo; j < hi; ++j) {
            const int64_t s0 = P->first[j], s1 = P->first[j + 1];
            real E = RL(0.0);
            for (int64_t s = s0; s < s1; ++s) E += P->b[s] * qval(P, u, s);
            P->V[j] = E;
            const real negE = RL(-1.0) * (RL(0.0) + E);
            for (int64_t s = s0; s < s1; ++s) {
                real rv = P->r[s] + (negE + qval(P, u, s));
                if (post == 1) rv = rv > RL(0.0) ? rv : RL(0.0);
                else if (post == 2) rv = rv > RL(0.0) ? rv * pf : (rv < RL(0.0) ? rv * nf : rv);
                P->r[s] = rv;
            }
        }
    }
}
static void observe(oc_player* P, const real* u, int post, double pf, double nf, int threads) {
    obs_ctx c = {P, u, post, (real)pf, (real)nf}; /* schedule factors rounded once */
    for (int64_t l = P->L - 1; l >= 0; --l) parfor(P->lvl[l], P->lvl[l + 1], threads, 1 << 13, observe_range, &c);
}

static void regret_match(const real* r, real* b, int64_t s0, int64_t s1) {
    real S = RL(0.0);
    for (int64_t s = s0; s < s1; ++s) S += r[s] > RL(0.0) ? r[s] : RL(0.0);
    for (int64_t s = s0; s < s1; ++s) {
        const real p = r[s] > RL(0.0) ? r[s] : RL(0.0);
        b[s] = S != RL(0.0) ? p / S : RL(1.0) / (real)(s1 - s0);
    }
}

/* next_strategy (pkg/solvers.py:143-175): RM into b, TD into x, avg += w x.
 * current_strategy (:270-291) when b_out is a scratch and w < 0 (no avg). */
typedef struct { oc_player* P; const real* r; real* b_out; real* x; real w; int avg; } next_ctx;
static void next_range(void* p, int64_t lo, int64_t hi) {
    const next_ctx* c = (const next_ctx*)p;
    oc_player* P = c->P;
    const real* r = c->r;
    real* b_out = c->b_out;
    real* x = c->x;
    const real w = c->w;
    {
        for (int64_t j = lo; j < hi; ++j) {
            const int64_t s0 = P->first[j], s1 = P->first[j + 1];
            regret_match(r, b_out, s0, s1);
            const real xp = x[P->parent[j]];
            for (int64_t s = s0; s < s1; ++s) {
                const real xa = b_out[s] * xp;
                x[s] = xa;
                if (c->avg) P->avg[s] = w * xa + P->avg[s];
            }
        }
    }
}
/* w < 0: no average (current_strategy).  avg_weight sums the fp64 w. */
static void next_strategy(oc_player* P, const real* r, real* b_out, real* x, double w,
                          int threads) {
    next_ctx c = {P, r, b_out, x, (real)w, w >= 0.0};
    for (int64_t l = 0; l < P->L; ++l) parfor(P->lvl[l], P->lvl[l + 1], threads, 1 << 13, next_range, &c);
    if (w >= 0.0) {
        P->avg[0] = (real)w * x[0] + P->avg[0]; /* the axpy covers the empty sequence too */
        P->avg_weight += w;
    }
}

static double factor(int64_t t, double e) {
    const double p = pow((double)t, e);
    if (isinf(p)) return 1.0;
    return p / (p + 1.0);
}

static void variant_observe(oc_state* st, oc_player* P, const real* u) {
    int post = 0;
    double pf = 1.0, nf = 1.0;
    if (st->variant == 1 || st->variant == 4) post = 1;
    if (st->variant == 2) {
        post = 2;
        pf = factor(st->t, st->alpha);
        nf = factor(st->t, st->beta);
    }
    observe(P, u, post, pf, nf, st->threads);
}

/* variant_next (pkg/solvers.py:248-256); predictive = snapshot / observe(m)
 * with the previous behaviour / next_strategy / restore (:227-245). */
static void variant_next(oc_state* st, oc_player* P, real* scratch_r) {
    const double w = pow((double)st->t, st->gamma);
    if (st->variant == 3 || st->variant == 4) {
        memcpy(scratch_r, P->r, P->S * sizeof(real));
        real* keep = P->r;
        P->r = scratch_r;
        observe(P, P->u, st->variant == 4 ? 1 : 0, 1.0, 1.0, st->threads);
        next_strategy(P, P->r, P->b, P->x, w, st->threads);
        P->r = keep;
    } else {
        next_strategy(P, P->r, P->b, P->x, w, st->threads);
    }
}

oc_state* oc_create(const int64_t* nn, const int64_t* ns, const int64_t* nj,
                    const int64_t* const* depth, const int64_t* const* dp_node,
                    const int64_t* const* first, const int64_t* const* nact,
                    const int64_t* const* parent, int64_t nnz, const int64_t* u_indptr,
                    const int64_t* u_indices, const double* u_data, const int64_t* ut_indptr,
                    const int64_t* ut_indices, const double* ut_data, int variant, int mode,
                    double alpha, double beta, double gamma, int threads) {
    oc_state* st = xcalloc(1, sizeof(oc_state));
    for (int k = 0; k < 2; ++k)
        if (build_player(&st->p[k], nn[k], ns[k], nj[k], depth[k], dp_node[k], first[k], nact[k],
                         parent[k]) != 0) {
            free(st);
            return NULL;
        }
    copy_csr(&st->U, ns[0], nnz, u_indptr, u_indices, u_data);
    copy_csr(&st->UT, ns[1], nnz, ut_indptr, ut_indices, ut_data);
    st->variant = variant;
    st->mode = mode;
    st->alpha = alpha;
    st->beta = beta;
    st->gamma = gamma;
    st->t = 1;
    st->threads = threads < 1 ? 1 : threads;
    return st;
}

/* _step (pkg/solvers.py:351-372), n times. */
void oc_step(oc_state* st, int64_t n) {
    oc_player *A = &st->p[0], *B = &st->p[1];
    int64_t smax = A->S > B->S ? A->S : B->S;
    real* scratch = xcalloc(smax, sizeof(real));
    real* peek = xcalloc(A->S, sizeof(real));
    for (int64_t it = 0; it < n; ++it) {
        variant_next(st, A, scratch);
        variant_next(st, B, scratch);
        spmv(&st->U, B->x, A->u, 0, st->threads);
        if (st->mode == 0) {
            spmv(&st->UT, A->x, B->u, 1, st->threads);
            variant_observe(st, A, A->u);
        } else {
            variant_observe(st, A, A->u);
            next_strategy(A, A->r, peek, A->xpost, -1.0, st->threads); /* current_strategy */
            spmv(&st->UT, A->xpost, B->u, 1, st->threads);
        }
        variant_observe(st, B, B->u);
        st->t += 1;
    }
    free(scratch);
    free(peek);
}

/* which: 0 regrets[S] (slot 0 unused), 1 behaviour, 2 avg_accum, 3 u, 4 x,
 * 5 xpost.  Returns the avg weight. */
double oc_read(const oc_state* st, int player, int which, double* out) {
    const oc_player* P = &st->p[player - 1];
    const real* src = which == 0 ? P->r : which == 1 ? P->b : which == 2 ? P->avg
                    : which == 3 ? P->u : which == 4 ? P->x : P->xpost;
    for (int64_t s = 0; s < P->S; ++s) out[s] = (double)src[s]; /* exact widening */
    return P->avg_weight;
}

int64_t oc_t(const oc_state* st) { return st->t; }

/* g = U x (player 1) or -Uᵀ x (player 2), then scalar_best_response
 * (pkg/oracle.py:186-221) per DP, deepest level first. */
static real* to_real(const double* x, int64_t n) {
    real* r = xcalloc(n, sizeof(real));
    for (int64_t i = 0; i < n; ++i) r[i] = (real)x[i];
    return r;
}

double oc_best_response(oc_state* st, int player, const double* x_opp) {
    oc_player* P = &st->p[player - 1];
    real* xo = to_real(x_opp, st->p[2 - player].S);
    spmv(player == 1 ? &st->U : &st->UT, xo, P->g, player == 2, st->threads);
    free(xo);
    for (int64_t l = P->L - 1; l >= 0; --l)
        for (int64_t j = P->lvl[l]; j < P->lvl[l + 1]; ++j) {
            real best = -INFINITY;
            for (int64_t s = P->first[j]; s < P->first[j + 1]; ++s) {
                const real v = P->g[s] + child_sum(P, s, P->W);
                if (v > best) best = v;
            }
            P->W[j] = best;
        }
    return P->g[0] + child_sum(P, 0, P->W);
}

void oc_spmv(oc_state* st, int transposed, const double* x, double* out, int neg) {
    const oc_csr* M = transposed ? &st->UT : &st->U;
    real* xr = to_real(x, transposed ? st->p[0].S : st->p[1].S);
    real* o = xcalloc(M->rows, sizeof(real));
    spmv(M, xr, o, neg, st->threads);
    for (int64_t i = 0; i < M->rows; ++i) out[i] = (double)o[i];
    free(xr);
    free(o);
}

void oc_free(oc_state* st) {
    if (!st) return;
    for (int k = 0; k < 2; ++k) {
        oc_player* P = &st->p[k];
        free(P->first); free(P->parent); free(P->clo); free(P->ccnt); free(P->lvl);
        free(P->r); free(P->b); free(P->x); free(P->xpost); free(P->avg); free(P->u);
        free(P->V); free(P->W); free(P->g);
    }
    free(st->U.indptr); free(st->U.indices); free(st->U.data);
    free(st->UT.indptr); free(st->UT.indices); free(st->UT.data);
    free(st);
}
