/*
 * seqcfr_tree.c — CPU restatement of the reference compile step, plus the
 * two fixture-game generators, in plain C.
 *
 * TEST INFRASTRUCTURE ONLY (like seqcfr_oracle.c).  It exists so that the
 * checker side — tests/, __graft_entry__.smoke() and bench.py's
 * `--impl reference` / cpu_baseline legs — can build any bundle, including
 * Goofspiel-5 (8.5 M game nodes), without the product library
 * (paper_2605_14277_b200/_lib/libseqcfr_b200.so).  Nothing in the product
 * links or calls it.  Its output is pinned to the reference's own arrays by
 * tests/test_oracle_tree.py (golden digests written by
 * scripts/make_golden.py and scripts/make_golden_goof5.py, which ran the
 * reference).
 *
 * Restated reference code:
 *   DecisionProcess._extract   pkg/decision_process.py:76-242
 *   Game.chance_reach          pkg/games.py:93-103
 *   build_payoff_matrix        pkg/operators.py:164-180
 *   CsrMatrix.from_coo         pkg/kernels.py:95-112  (stable lexsort,
 *                                                      bincount sums from 0.0)
 *   CsrMatrix.transposed       pkg/kernels.py:114-127 (stable argsort)
 * Generators (the reference has neither game): SURVEY.md
 * Appendix A — Liar's dice (1 die each) and Goofspiel-N, emitted in the DFS
 * pre-order of a recursive GameBuilder walk, infoset ids interned by first
 * appearance.
 *
 * Flat game layout: kind 0 chance / 1 decision / 2 terminal; parent -1 at
 * the root; children in listed order (child_ptr / child_idx); player 0 off
 * decision nodes; infoset -1 off decision nodes; prob NaN where the node
 * carries none; payoff NaN off terminals.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t n, num_infosets;
    int8_t *kind, *player;
    int64_t *parent, *child_ptr, *child_idx, *infoset;
    double *prob, *payoff;
} ot_game;

typedef struct {
    int64_t num_nodes, num_decisions, num_seqs, height, degree;
    int8_t* kind;
    int64_t *depth, *parent, *node_seq, *seq_node, *dp_node, *dp_first_seq, *dp_num_actions,
        *dp_parent_seq, *level_starts, *game_seq;
} ot_proc;

typedef struct {
    int64_t rows, cols, nnz;
    int64_t *indptr, *indices;
    double* data;
} ot_csr;

enum { G_CHANCE = 0, G_DECISION = 1, G_TERMINAL = 2 };
enum { K_DEC = 0, K_OBS = 1, K_END = 2 };

static void* zalloc(size_t n, size_t s) { return calloc(n ? n : 1, s); }

/* ------------------------------------------------------------------------
 * Growable flat-game builder + an open-addressing intern table for infosets.
 */
typedef struct {
    int64_t n, cap;
    int8_t *kind, *player;
    int64_t *parent, *infoset;
    double *prob, *payoff;
    /* intern table: key -> id, first appearance */
    int64_t tcap, nids;
    uint64_t* tkey;
    int64_t* tval;
} builder;

static int b_grow(builder* b) {
    int64_t c = b->cap ? 2 * b->cap : 1024;
    void* p;
#define GROW(f, T)                                       \
    p = realloc(b->f, (size_t)c * sizeof(T));            \
    if (!p) return -1;                                   \
    b->f = (T*)p;
    GROW(kind, int8_t) GROW(player, int8_t) GROW(parent, int64_t) GROW(infoset, int64_t)
    GROW(prob, double) GROW(payoff, double)
#undef GROW
    b->cap = c;
    return 0;
}

static uint64_t mix64(uint64_t z) { /* splitmix64 finaliser */
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static int64_t b_intern(builder* b, uint64_t key) {
    if (2 * (b->nids + 1) > b->tcap) {
        int64_t nc = b->tcap ? 2 * b->tcap : 1 << 12;
        uint64_t* nk = (uint64_t*)malloc((size_t)nc * sizeof(uint64_t));
        int64_t* nv = (int64_t*)malloc((size_t)nc * sizeof(int64_t));
        if (!nk || !nv) { free(nk); free(nv); return -1; }
        for (int64_t i = 0; i < nc; ++i) nv[i] = -1;
        for (int64_t i = 0; i < b->tcap; ++i) {
            if (b->tval[i] < 0) continue;
            uint64_t h = mix64(b->tkey[i]) & (uint64_t)(nc - 1);
            while (nv[h] >= 0) h = (h + 1) & (uint64_t)(nc - 1);
            nk[h] = b->tkey[i];
            nv[h] = b->tval[i];
        }
        free(b->tkey); free(b->tval);
        b->tkey = nk; b->tval = nv; b->tcap = nc;
    }
    uint64_t h = mix64(key) & (uint64_t)(b->tcap - 1);
    while (b->tval[h] >= 0) {
        if (b->tkey[h] == key) return b->tval[h];
        h = (h + 1) & (uint64_t)(b->tcap - 1);
    }
    b->tkey[h] = key;
    b->tval[h] = b->nids;
    return b->nids++;
}

static int64_t b_add(builder* b, int kind, int64_t parent, double prob, int player,
                     int64_t infoset, double payoff) {
    if (b->n == b->cap && b_grow(b)) return -1;
    int64_t i = b->n++;
    b->kind[i] = (int8_t)kind;
    b->player[i] = (int8_t)player;
    b->parent[i] = parent;
    b->infoset[i] = infoset;
    b->prob[i] = prob;
    b->payoff[i] = payoff;
    return i;
}

static ot_game* b_finish(builder* b) {
    ot_game* g = (ot_game*)zalloc(1, sizeof(ot_game));
    const int64_t n = b->n;
    g->n = n;
    g->num_infosets = b->nids;
    g->kind = b->kind; g->player = b->player; g->parent = b->parent;
    g->infoset = b->infoset; g->prob = b->prob; g->payoff = b->payoff;
    free(b->tkey); free(b->tval);
    /* children in creation (= increasing id) order */
    g->child_ptr = (int64_t*)zalloc((size_t)n + 1, sizeof(int64_t));
    g->child_idx = (int64_t*)zalloc((size_t)(n > 0 ? n - 1 : 0), sizeof(int64_t));
    for (int64_t i = 1; i < n; ++i) g->child_ptr[g->parent[i] + 1]++;
    for (int64_t i = 0; i < n; ++i) g->child_ptr[i + 1] += g->child_ptr[i];
    int64_t* fill = (int64_t*)zalloc((size_t)n, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) fill[i] = g->child_ptr[i];
    for (int64_t i = 1; i < n; ++i) g->child_idx[fill[g->parent[i]]++] = i;
    free(fill);
    return g;
}

void ot_game_free(ot_game* g) {
    if (!g) return;
    free(g->kind); free(g->player); free(g->parent); free(g->infoset);
    free(g->prob); free(g->payoff); free(g->child_ptr); free(g->child_idx);
    free(g);
}

/* --- Goofspiel-N (Appendix A): each round a chance node picks the prize
 * uniformly from those left (ascending), P1 bids each remaining card
 * (ascending), P2 bids without seeing P1's bid, both bids are revealed; the
 * last round's P2 bids lead to terminals, payoff = sign(point difference).
 * An infoset is (player, own hand, public history incl. the current prize);
 * the hand follows from the history, so the key is (player, history). */
typedef struct {
    builder b;
    int cards;
} goof_ctx;

static uint64_t goof_key(int player, const int* hist, int len) {
    uint64_t k = 0;
    for (int i = 0; i < len; ++i) k = k * 16u + (uint64_t)hist[i];
    return ((k * 64u + (uint64_t)len) << 1) | (uint64_t)(player - 1);
}

static int goof_round(goof_ctx* c, int64_t parent, unsigned prizes, unsigned h1, unsigned h2,
                      int score, int* hist, int len) {
    int64_t ch = b_add(&c->b, G_CHANCE, parent, NAN, 0, -1, NAN);
    if (ch < 0) return -1;
    const int left = __builtin_popcount(prizes);
    for (int p = 1; p <= c->cards; ++p) {
        if (!(prizes & (1u << p))) continue;
        const unsigned rest = prizes & ~(1u << p);
        hist[len] = p;
        const int64_t i1 = b_intern(&c->b, goof_key(1, hist, len + 1));
        const int64_t d1 = b_add(&c->b, G_DECISION, ch, 1.0 / (double)left, 1, i1, NAN);
        if (d1 < 0 || i1 < 0) return -1;
        for (int b1 = 1; b1 <= c->cards; ++b1) {
            if (!(h1 & (1u << b1))) continue;
            const int64_t i2 = b_intern(&c->b, goof_key(2, hist, len + 1));
            const int64_t d2 = b_add(&c->b, G_DECISION, d1, NAN, 2, i2, NAN);
            if (d2 < 0 || i2 < 0) return -1;
            for (int b2 = 1; b2 <= c->cards; ++b2) {
                if (!(h2 & (1u << b2))) continue;
                const int s = score + (b1 > b2 ? p : (b2 > b1 ? -p : 0));
                if (rest) {
                    hist[len + 1] = b1;
                    hist[len + 2] = b2;
                    if (goof_round(c, d2, rest, h1 & ~(1u << b1), h2 & ~(1u << b2), s, hist,
                                   len + 3))
                        return -1;
                } else {
                    if (b_add(&c->b, G_TERMINAL, d2, NAN, 0, -1, (double)((s > 0) - (s < 0))) < 0)
                        return -1;
                }
            }
        }
    }
    return 0;
}

ot_game* ot_goofspiel(int cards) {
    if (cards < 1 || cards > 5) return NULL; /* history key: 4 bits per entry */
    goof_ctx c;
    memset(&c, 0, sizeof c);
    c.cards = cards;
    const unsigned deck = ((1u << (cards + 1)) - 1u) & ~1u;
    int hist[64];
    if (goof_round(&c, -1, deck, deck, deck, 0, hist, 0)) return NULL;
    return b_finish(&c.b);
}

/* --- Liar's dice, one die each, F faces (Appendix A): chance deals P1's die
 * then P2's die (1/F each); the P2-deal edge leads into P1's first decision.
 * Bids (q, f), q in {1, 2}, f in 1..F, ordered by q then f; a player raises
 * to any higher bid or calls liar on the standing bid; face F is wild.  An
 * infoset is (actor, own die, set of bids so far). */
typedef struct {
    builder b;
    int F;
} liars_ctx;

static int liars_expand(liars_ctx* c, int64_t parent, double prob, int actor, int d1, int d2,
                        int last, uint64_t mask) {
    const int own = actor == 1 ? d1 : d2;
    const uint64_t key = ((mask * 64u + (uint64_t)own) << 1) | (uint64_t)(actor - 1);
    const int64_t inf = b_intern(&c->b, key);
    const int64_t me = b_add(&c->b, G_DECISION, parent, prob, actor, inf, NAN);
    if (me < 0 || inf < 0) return -1;
    const int nb = 2 * c->F;
    for (int k = last + 1; k < nb; ++k)
        if (liars_expand(c, me, NAN, 3 - actor, d1, d2, k, mask | (1ull << k))) return -1;
    if (last >= 0) {
        const int q = last / c->F + 1, f = last % c->F + 1;
        const int hits = (d1 == f || d1 == c->F) + (d2 == f || d2 == c->F);
        const int bidder = 3 - actor;
        const int bidder_wins = hits >= q;
        const int p1_wins = bidder_wins == (bidder == 1);
        if (b_add(&c->b, G_TERMINAL, me, NAN, 0, -1, p1_wins ? 1.0 : -1.0) < 0) return -1;
    }
    return 0;
}

ot_game* ot_liars_dice(int faces) {
    if (faces < 1 || faces > 16) return NULL;
    liars_ctx c;
    memset(&c, 0, sizeof c);
    c.F = faces;
    const int64_t root = b_add(&c.b, G_CHANCE, -1, NAN, 0, -1, NAN);
    for (int d1 = 1; d1 <= faces; ++d1) {
        const int64_t mid = b_add(&c.b, G_CHANCE, root, 1.0 / faces, 0, -1, NAN);
        for (int d2 = 1; d2 <= faces; ++d2)
            if (liars_expand(&c, mid, 1.0 / faces, 1, d1, d2, -1, 0)) return NULL;
    }
    return b_finish(&c.b);
}

int64_t ot_game_arrays(const ot_game* g, int8_t** kind, int64_t** parent, int64_t** child_ptr,
                       int64_t** child_idx, int8_t** player, int64_t** infoset, double** prob,
                       double** payoff) {
    *kind = g->kind; *parent = g->parent; *child_ptr = g->child_ptr; *child_idx = g->child_idx;
    *player = g->player; *infoset = g->infoset; *prob = g->prob; *payoff = g->payoff;
    return g->n;
}

/* ------------------------------------------------------------------------
 * DecisionProcess._extract (pkg/decision_process.py:76-242).
 * Returns 0, or -1 on a perfect-recall violation / malformed tree, -2 on OOM.
 */
void ot_proc_free(ot_proc* p) {
    if (!p) return;
    free(p->kind); free(p->depth); free(p->parent); free(p->node_seq); free(p->seq_node);
    free(p->dp_node); free(p->dp_first_seq); free(p->dp_num_actions); free(p->dp_parent_seq);
    free(p->level_starts); free(p->game_seq);
    free(p);
}

ot_proc* ot_extract(int64_t n, const int8_t* kind, const int64_t* parent,
                    const int64_t* child_ptr, const int64_t* child_idx, const int8_t* player,
                    const int64_t* infoset, int pl, int* err) {
    *err = 0;
    if (n <= 0) { *err = -1; return NULL; }
    int64_t max_inf = -1;
    for (int64_t v = 0; v < n; ++v)
        if (kind[v] == G_DECISION && infoset[v] > max_inf) max_inf = infoset[v];
    int64_t* order = (int64_t*)zalloc((size_t)n, sizeof(int64_t));
    int64_t* slot = (int64_t*)zalloc((size_t)n, sizeof(int64_t)); /* index among siblings */
    int64_t* prov = (int64_t*)zalloc((size_t)n, sizeof(int64_t));
    int64_t* pid_of = (int64_t*)zalloc((size_t)max_inf + 1, sizeof(int64_t));
    /* per pid (<= number of decision nodes of player pl) */
    int64_t npmax = 0;
    for (int64_t v = 0; v < n; ++v) npmax += (kind[v] == G_DECISION && player[v] == pl);
    int64_t* first_key = (int64_t*)zalloc((size_t)npmax, sizeof(int64_t));
    int64_t* parent_key = (int64_t*)zalloc((size_t)npmax, sizeof(int64_t));
    int64_t* nact = (int64_t*)zalloc((size_t)npmax, sizeof(int64_t));
    ot_proc* P = NULL;
    int64_t *kid_ptr = NULL, *kid_list = NULL, *j_of_pid = NULL, *fin = NULL;
    int64_t *qa = NULL, *qpar = NULL, *qd = NULL, *qx = NULL;
    int8_t* qtag = NULL;
    if (!order || !slot || !prov || !pid_of || !first_key || !parent_key || !nact) goto oom;
    for (int64_t i = 0; i <= max_inf; ++i) pid_of[i] = -1;
    for (int64_t v = 0; v < n; ++v)
        for (int64_t k = child_ptr[v]; k < child_ptr[v + 1]; ++k) slot[child_idx[k]] = k - child_ptr[v];
    /* BFS order of the game tree */
    int64_t tail = 1;
    order[0] = 0;
    for (int64_t h = 0; h < tail; ++h) {
        const int64_t v = order[h];
        for (int64_t k = child_ptr[v]; k < child_ptr[v + 1]; ++k) {
            if (tail >= n) { *err = -1; goto fail; }
            order[tail++] = child_idx[k];
        }
    }
    if (tail != n) { *err = -1; goto fail; }
    int64_t np_ = 0, next_key = 1;
    for (int64_t h = 0; h < n; ++h) {
        const int64_t v = order[h];
        if (v != 0) {
            const int64_t par = parent[v];
            int64_t key = prov[par];
            if (kind[par] == G_DECISION && player[par] == pl)
                key = first_key[pid_of[infoset[par]]] + slot[v];
            prov[v] = key;
        }
        if (kind[v] == G_DECISION && player[v] == pl) {
            const int64_t key = prov[v];
            const int64_t na = child_ptr[v + 1] - child_ptr[v];
            int64_t pid = pid_of[infoset[v]];
            if (pid < 0) {
                pid = np_++;
                pid_of[infoset[v]] = pid;
                first_key[pid] = next_key;
                parent_key[pid] = key;
                nact[pid] = na;
                next_key += na;
            } else if (parent_key[pid] != key || nact[pid] != na) {
                *err = -1;
                goto fail;
            }
        }
    }
    const int64_t J = np_, S = next_key; /* num_seqs = 1 + sum(nact) */
    /* children_of_key: pids grouped by parent key, in pid (creation) order */
    kid_ptr = (int64_t*)zalloc((size_t)S + 1, sizeof(int64_t));
    kid_list = (int64_t*)zalloc((size_t)J, sizeof(int64_t));
    j_of_pid = (int64_t*)zalloc((size_t)J, sizeof(int64_t));
    fin = (int64_t*)zalloc((size_t)S, sizeof(int64_t));
    /* queue: every sequence slot and every DP hanging under an observation
     * point is enqueued once */
    const int64_t qcap = S + J + 1;
    qtag = (int8_t*)zalloc((size_t)qcap, 1);
    qa = (int64_t*)zalloc((size_t)qcap, sizeof(int64_t));
    qpar = (int64_t*)zalloc((size_t)qcap, sizeof(int64_t));
    qd = (int64_t*)zalloc((size_t)qcap, sizeof(int64_t));
    qx = (int64_t*)zalloc((size_t)qcap, sizeof(int64_t));
    P = (ot_proc*)zalloc(1, sizeof(ot_proc));
    if (!kid_ptr || !kid_list || !j_of_pid || !fin || !qtag || !qa || !qpar || !qd || !qx || !P)
        goto oom;
    for (int64_t p = 0; p < J; ++p) kid_ptr[parent_key[p] + 1]++;
    for (int64_t k = 0; k < S; ++k) kid_ptr[k + 1] += kid_ptr[k];
    {
        int64_t* fill = (int64_t*)zalloc((size_t)S, sizeof(int64_t));
        if (!fill) goto oom;
        memcpy(fill, kid_ptr, (size_t)S * sizeof(int64_t));
        for (int64_t p = 0; p < J; ++p) kid_list[fill[parent_key[p]]++] = p;
        free(fill);
    }
    /* the process has exactly one node per queue item */
    const int64_t NN = S + (J - 0); /* upper bound: S sequence images + DPs under obs */
    P->kind = (int8_t*)zalloc((size_t)NN, 1);
    P->depth = (int64_t*)zalloc((size_t)NN, sizeof(int64_t));
    P->parent = (int64_t*)zalloc((size_t)NN, sizeof(int64_t));
    P->node_seq = (int64_t*)zalloc((size_t)NN, sizeof(int64_t));
    P->seq_node = (int64_t*)zalloc((size_t)S, sizeof(int64_t));
    P->dp_node = (int64_t*)zalloc((size_t)J, sizeof(int64_t));
    P->dp_first_seq = (int64_t*)zalloc((size_t)J, sizeof(int64_t));
    P->dp_num_actions = (int64_t*)zalloc((size_t)J, sizeof(int64_t));
    P->dp_parent_seq = (int64_t*)zalloc((size_t)J, sizeof(int64_t));
    P->game_seq = (int64_t*)zalloc((size_t)n, sizeof(int64_t));
    if (!P->kind || !P->depth || !P->parent || !P->node_seq || !P->seq_node || !P->dp_node ||
        !P->dp_first_seq || !P->dp_num_actions || !P->dp_parent_seq || !P->game_seq)
        goto oom;
    for (int64_t s = 0; s < S; ++s) P->seq_node[s] = -1;
    int64_t qh = 0, qt = 0, nn = 0, next_j = 0, next_seq = 1;
    /* ("seq", seq, par, d, key) and ("dp", pid, par, d, parent_seq) */
#define PUSH(tag, a, par, d, x) \
    do { qtag[qt] = (tag); qa[qt] = (a); qpar[qt] = (par); qd[qt] = (d); qx[qt] = (x); ++qt; } while (0)
#define NEW_NODE(k, par, d, seq, out)                       \
    do {                                                     \
        (out) = nn++;                                        \
        P->kind[out] = (int8_t)(k);                          \
        P->parent[out] = (par);                              \
        P->depth[out] = (d);                                 \
        P->node_seq[out] = (seq);                            \
        if ((seq) >= 0) P->seq_node[seq] = (out);            \
    } while (0)
    PUSH(0, 0, -1, 0, 0);
    while (qh < qt) {
        const int tag = qtag[qh];
        const int64_t a = qa[qh], par = qpar[qh], d = qd[qh], x = qx[qh];
        ++qh;
        int64_t pid = -1, parent_seq = 0, seq = -1, nid;
        if (tag == 0) {
            const int64_t cnt = kid_ptr[x + 1] - kid_ptr[x];
            if (cnt == 0) {
                NEW_NODE(K_END, par, d, a, nid);
                continue;
            }
            if (cnt > 1) {
                NEW_NODE(K_OBS, par, d, a, nid);
                for (int64_t k = kid_ptr[x]; k < kid_ptr[x + 1]; ++k) PUSH(1, kid_list[k], nid, d + 1, a);
                continue;
            }
            pid = kid_list[kid_ptr[x]];
            parent_seq = a;
            seq = a;
        } else {
            pid = a;
            parent_seq = x;
            seq = -1;
        }
        /* open_decision */
        NEW_NODE(K_DEC, par, d, seq, nid);
        const int64_t j = next_j++;
        j_of_pid[pid] = j;
        P->dp_node[j] = nid;
        P->dp_first_seq[j] = next_seq;
        P->dp_num_actions[j] = nact[pid];
        P->dp_parent_seq[j] = parent_seq;
        for (int64_t k = 0; k < nact[pid]; ++k) PUSH(0, next_seq + k, nid, d + 1, first_key[pid] + k);
        next_seq += nact[pid];
    }
#undef PUSH
#undef NEW_NODE
    P->num_nodes = nn;
    P->num_decisions = J;
    P->num_seqs = S;
    int64_t height = 0;
    for (int64_t i = 0; i < nn; ++i) if (P->depth[i] > height) height = P->depth[i];
    P->height = height;
    {
        int64_t* cnt = (int64_t*)zalloc((size_t)nn, sizeof(int64_t));
        if (!cnt) goto oom;
        for (int64_t i = 1; i < nn; ++i) cnt[P->parent[i]]++;
        int64_t deg = 0;
        for (int64_t i = 0; i < nn; ++i) if (cnt[i] > deg) deg = cnt[i];
        P->degree = deg;
        free(cnt);
    }
    /* level_starts = searchsorted(depth, arange(height + 2)) (left side) */
    P->level_starts = (int64_t*)zalloc((size_t)height + 2, sizeof(int64_t));
    if (!P->level_starts) goto oom;
    {
        int64_t i = 0;
        for (int64_t d = 0; d <= height + 1; ++d) {
            while (i < nn && P->depth[i] < d) ++i;
            P->level_starts[d] = i;
        }
    }
    /* game_seq = final_of_key[game_seq_prov] */
    for (int64_t p = 0; p < J; ++p) {
        const int64_t j = j_of_pid[p];
        for (int64_t k = 0; k < nact[p]; ++k) fin[first_key[p] + k] = P->dp_first_seq[j] + k;
    }
    for (int64_t v = 0; v < n; ++v) P->game_seq[v] = fin[prov[v]];
    goto done;
oom:
    *err = -2;
fail:
    ot_proc_free(P);
    P = NULL;
done:
    free(order); free(slot); free(prov); free(pid_of); free(first_key); free(parent_key);
    free(nact); free(kid_ptr); free(kid_list); free(j_of_pid); free(fin);
    free(qtag); free(qa); free(qpar); free(qd); free(qx);
    return P;
}

/* ------------------------------------------------------------------------
 * build_payoff_matrix + from_coo + transposed (pkg/operators.py:164-180,
 * pkg/kernels.py:95-127).
 */
void ot_csr_free(ot_csr* m) {
    if (!m) return;
    free(m->indptr); free(m->indices); free(m->data);
    free(m);
}

/* stable counting sort of idx[0..m) by key[idx[i]] in [0, K) */
static int stable_by(int64_t m, int64_t* idx, const int64_t* key, int64_t K) {
    int64_t* cnt = (int64_t*)zalloc((size_t)K + 1, sizeof(int64_t));
    int64_t* out = (int64_t*)zalloc((size_t)m, sizeof(int64_t));
    if (!cnt || !out) { free(cnt); free(out); return -1; }
    for (int64_t i = 0; i < m; ++i) cnt[key[idx[i]] + 1]++;
    for (int64_t k = 0; k < K; ++k) cnt[k + 1] += cnt[k];
    for (int64_t i = 0; i < m; ++i) out[cnt[key[idx[i]]]++] = idx[i];
    memcpy(idx, out, (size_t)m * sizeof(int64_t));
    free(cnt); free(out);
    return 0;
}

int ot_payoff(int64_t n, const int8_t* kind, const int64_t* parent, const double* prob,
              const double* payoff, const ot_proc* p1, const ot_proc* p2, ot_csr** U_out,
              ot_csr** UT_out) {
    int rc = -2;
    const int64_t R = p1->num_seqs, C = p2->num_seqs;
    double* reach = (double*)zalloc((size_t)n, sizeof(double));
    int64_t nz = 0;
    for (int64_t v = 0; v < n; ++v) nz += kind[v] == G_TERMINAL;
    int64_t *zr = (int64_t*)zalloc((size_t)nz, sizeof(int64_t)),
            *zc = (int64_t*)zalloc((size_t)nz, sizeof(int64_t)),
            *idx = (int64_t*)zalloc((size_t)nz, sizeof(int64_t));
    double* zv = (double*)zalloc((size_t)nz, sizeof(double));
    ot_csr* U = (ot_csr*)zalloc(1, sizeof(ot_csr));
    ot_csr* UT = (ot_csr*)zalloc(1, sizeof(ot_csr));
    if (!reach || !zr || !zc || !idx || !zv || !U || !UT) goto out;
    /* chance_reach: node order, parent before child */
    reach[0] = 1.0;
    for (int64_t v = 1; v < n; ++v) {
        double p = reach[parent[v]];
        if (!isnan(prob[v])) p *= prob[v];
        reach[v] = p;
    }
    {
        int64_t k = 0;
        for (int64_t v = 0; v < n; ++v) {
            if (kind[v] != G_TERMINAL) continue;
            zr[k] = p1->game_seq[v];
            zc[k] = p2->game_seq[v];
            zv[k] = payoff[v] * reach[v];
            idx[k] = k;
            ++k;
        }
    }
    /* lexsort((c, r)): stable by c, then stable by r */
    if (stable_by(nz, idx, zc, C) || stable_by(nz, idx, zr, R)) goto out;
    /* sum duplicate cells sequentially from 0.0 (np.bincount weights) */
    int64_t m = 0;
    U->indptr = (int64_t*)zalloc((size_t)R + 1, sizeof(int64_t));
    U->indices = (int64_t*)zalloc((size_t)nz, sizeof(int64_t));
    U->data = (double*)zalloc((size_t)nz, sizeof(double));
    if (!U->indptr || !U->indices || !U->data) goto out;
    for (int64_t k = 0; k < nz; ++k) {
        const int64_t i = idx[k];
        if (k == 0 || zr[i] != zr[idx[k - 1]] || zc[i] != zc[idx[k - 1]]) {
            U->indices[m] = zc[i];
            U->data[m] = 0.0;
            U->indptr[zr[i] + 1]++;
            ++m;
        }
        U->data[m - 1] += zv[i];
    }
    for (int64_t r = 0; r < R; ++r) U->indptr[r + 1] += U->indptr[r];
    U->rows = R; U->cols = C; U->nnz = m;
    /* transposed: stable argsort of indices */
    UT->indptr = (int64_t*)zalloc((size_t)C + 1, sizeof(int64_t));
    UT->indices = (int64_t*)zalloc((size_t)m, sizeof(int64_t));
    UT->data = (double*)zalloc((size_t)m, sizeof(double));
    if (!UT->indptr || !UT->indices || !UT->data) goto out;
    for (int64_t k = 0; k < m; ++k) UT->indptr[U->indices[k] + 1]++;
    for (int64_t c = 0; c < C; ++c) UT->indptr[c + 1] += UT->indptr[c];
    {
        int64_t* fill = (int64_t*)zalloc((size_t)C, sizeof(int64_t));
        if (!fill) goto out;
        memcpy(fill, UT->indptr, (size_t)C * sizeof(int64_t));
        for (int64_t r = 0; r < R; ++r)
            for (int64_t k = U->indptr[r]; k < U->indptr[r + 1]; ++k) {
                const int64_t o = fill[U->indices[k]]++;
                UT->indices[o] = r;
                UT->data[o] = U->data[k];
            }
        free(fill);
    }
    UT->rows = C; UT->cols = R; UT->nnz = m;
    rc = 0;
out:
    free(reach); free(zr); free(zc); free(idx); free(zv);
    if (rc) { ot_csr_free(U); ot_csr_free(UT); U = UT = NULL; }
    *U_out = U;
    *UT_out = UT;
    return rc;
}
