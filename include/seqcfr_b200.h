/*
 * seqcfr_b200.h — C-ABI of the B200-native sequence-form CFR hot path.
 *
 * Drop-in boundary for the reference package `seqcfr` (read-only at
 * /root/reference/pkg/src/seqcfr).  The reference has no native FFI of its
 * own: its hot path is Python driving numba loops through the `Backend`
 * object.  The entry points below replace, at the solver level (SURVEY.md
 * §8(b) boundary 2):
 *
 *   scfr_compile            GameBundle.__init__           pkg/solvers.py:314-323
 *                           (DecisionProcess._extract     pkg/decision_process.py:76-242,
 *                            build_payoff_matrix          pkg/operators.py:164-180,
 *                            CsrMatrix.from_coo/transposed pkg/kernels.py:95-127)
 *   scfr_create             RegretState x2 allocation     pkg/solvers.py:97-127, :404-405
 *   scfr_step               the `while True: _step(...)`  pkg/solvers.py:351-372, :424-434
 *   scfr_read_average       RegretState.average_strategy  pkg/solvers.py:129-134
 *   scfr_read_averages      RunResult.average (both)      pkg/solvers.py:129-134, :436-438
 *   scfr_read_current       the x1, x2 returned by _step  pkg/solvers.py:372
 *   scfr_exploitability     metrics.exploitability        pkg/metrics.py:59-75
 *                           (+ oracle.scalar_best_response pkg/oracle.py:186-221)
 *   scfr_status             FloatingPointError checks     pkg/solvers.py:154-155, :188-189
 *
 * Conventions
 *   - Every function returns an int status: 0 on success, a negative
 *     SCFR_E* code on failure; scfr_last_error() gives the message of the
 *     calling thread's most recent failure.  SCFR_EINVAL maps to the
 *     reference's ValueError, SCFR_EGAME to GameValidationError and
 *     SCFR_ENONFINITE to FloatingPointError.
 *   - Arrays use the reference's dtypes (int64 indices, float64 values) and
 *     index layout (DecisionProcess ids, Σ-indexed sequence vectors with
 *     slot 0 = the empty sequence), so a reference maintainer can pass its
 *     numpy arrays' buffers straight through.
 *   - The caller keeps ownership of every input pointer; the library copies.
 *   - Handles are independent; one host thread drives a handle at a time.
 *   - No CPU fallback: without a usable sm_100 device, scfr_create fails with
 *     SCFR_ECUDA.
 */
#ifndef SEQCFR_B200_H
#define SEQCFR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCFR_ABI_VERSION 1

#define SCFR_OK 0
#define SCFR_EINVAL (-1)     /* bad argument / dimension mismatch (ValueError) */
#define SCFR_EGAME (-2)      /* invalid game, e.g. perfect recall (GameValidationError) */
#define SCFR_ENONFINITE (-3) /* non-finite regrets or utilities (FloatingPointError) */
#define SCFR_ECUDA (-4)      /* CUDA runtime failure / no device */
#define SCFR_ENOMEM (-5)
#define SCFR_ENCCL (-6)
/* a schedule value float(t)**gamma overflowed (the reference raises
 * OverflowError from Python's float power, pkg/solvers.py:172) */
#define SCFR_EOVERFLOW (-7)

/* Variants (pkg/solvers.py:35) and update modes (pkg/solvers.py:38-44). */
#define SCFR_CFR 0
#define SCFR_CFR_PLUS 1
#define SCFR_DCFR 2
#define SCFR_PCFR 3
#define SCFR_PCFR_PLUS 4
#define SCFR_MODE_SIM 0
#define SCFR_MODE_ALT 1

/* Arithmetic of the iteration state (scfr_config.dtype). */
#define SCFR_DTYPE_F64 0
#define SCFR_DTYPE_F32 1

/* Node kinds of the input game (pkg/games.py:23-25). */
#define SCFR_NODE_CHANCE 0
#define SCFR_NODE_DECISION 1
#define SCFR_NODE_TERMINAL 2

/* Engines (scfr_config.engine). */
#define SCFR_ENGINE_AUTO 0
#define SCFR_ENGINE_LEVELS 1          /* one kernel per DP level, captured in a CUDA graph */
#define SCFR_ENGINE_PERSISTENT 2      /* whole iterations in one kernel, one CTA per solve */
#define SCFR_ENGINE_PERSISTENT_GRID 3 /* whole iterations in one cooperative grid (batch 1) */
#define SCFR_ENGINE_TILED 4           /* one kernel per pass: CTAs own whole subtrees below a split level */
#define SCFR_ENGINE_PERSISTENT_CLUSTER 5 /* whole iterations in one kernel, one 16-CTA cluster per solve */

const char* scfr_last_error(void);
int scfr_abi_version(void);

/* ------------------------------------------------------------------------
 * Tree compiler (host).  Input: the reference Game flattened to columns
 * (paper_2605_14277_b200.games.FlatGame).  Output: both players' decision
 * processes, bit-identical to DecisionProcess, plus U and Uᵀ bit-identical
 * to build_payoff_matrix(...) and CsrMatrix.transposed().
 * ---------------------------------------------------------------------- */
typedef struct scfr_game {
    int64_t num_nodes;
    const int8_t* kind;       /* SCFR_NODE_* */
    const int64_t* parent;    /* -1 at the root (node 0) */
    const int64_t* child_ptr; /* [num_nodes+1] */
    const int64_t* child_idx; /* children in GameNode.children order */
    const int8_t* player;     /* 1/2 at decision nodes */
    const int64_t* infoset;   /* interned infoset label id at decision nodes, -1 elsewhere */
    const double* prob;       /* chance-edge probability, NaN when absent */
    const double* payoff;     /* payoff to player 1 at terminals, NaN elsewhere */
} scfr_game;

/* One player's tree-form sequential decision process, in the reference
 * DecisionProcess layout (pkg/decision_process.py:48-65). */
typedef struct scfr_tfsdp {
    int64_t num_nodes, num_decisions, num_seqs, height, degree;
    const int8_t* kind;            /* [num_nodes] 0 decision / 1 observation / 2 end */
    const int64_t* depth;          /* [num_nodes] */
    const int64_t* parent;         /* [num_nodes] */
    const int64_t* node_seq;       /* [num_nodes] */
    const int64_t* seq_node;       /* [num_seqs] */
    const int64_t* dp_node;        /* [num_decisions] */
    const int64_t* dp_first_seq;   /* [num_decisions] */
    const int64_t* dp_num_actions; /* [num_decisions] */
    const int64_t* dp_parent_seq;  /* [num_decisions] */
    const int64_t* level_starts;   /* [height+2] */
    const int64_t* game_seq;       /* [game num_nodes] (compiler output only) */
    const int64_t* dp_infoset;     /* [num_decisions] infoset id (compiler output only) */
    const int64_t* dp_game_node;   /* [num_decisions] first game node of the infoset */
} scfr_tfsdp;

/* CSR over float64 (pkg/kernels.py:33-49). */
typedef struct scfr_csr {
    int64_t rows, cols, nnz;
    const int64_t* indptr;  /* [rows+1] */
    const int64_t* indices; /* [nnz] */
    const double* data;     /* [nnz] */
} scfr_csr;

typedef struct scfr_compiled scfr_compiled;

int scfr_compile(const scfr_game* game, scfr_compiled** out);
/* Views stay valid until scfr_compiled_free. player is 1 or 2. */
int scfr_compiled_tfsdp(const scfr_compiled* c, int player, scfr_tfsdp* out);
int scfr_compiled_payoff(const scfr_compiled* c, int transposed, scfr_csr* out);
void scfr_compiled_free(scfr_compiled* c);

/* Native generators for the large fixtures, emitting
 * the same trees as paper_2605_14277_b200.games.liars_dice / goofspiel. */
typedef struct scfr_flat_game {
    scfr_game game;
    int64_t num_infosets;
} scfr_flat_game;
/* Native reader of the reference's JSON-lines game file (pkg/games.py:554-648):
 * parses and validates (the checks and messages of games.load_game +
 * games.validate_game, first violation reported) straight into the compiler's
 * flat arrays, with the names: labels[label_off[i] .. label_off[i+1]) is node
 * i's label_from_parent, infoset_names[infoset_off[k] ..) infoset id k's label.
 * On SCFR_EGAME: err_line >= 1 for a file-level error (GameParseError),
 * err_node >= 0 for a tree violation (GameValidationError). */
typedef struct scfr_parsed_game {
    scfr_flat_game flat;
    const char* name;
    const char* labels;
    const int64_t* label_off;      /* [num_nodes + 1] */
    const char* infoset_names;
    const int64_t* infoset_off;    /* [num_infosets + 1] */
} scfr_parsed_game;
int scfr_parse_game_jsonl(const char* text, int64_t len, scfr_parsed_game** out, int64_t* err_line,
                          int64_t* err_node);
void scfr_parsed_game_free(scfr_parsed_game* g);
int scfr_generate_liars_dice(int faces, scfr_flat_game** out);
int scfr_generate_goofspiel(int cards, scfr_flat_game** out);
void scfr_flat_game_free(scfr_flat_game* g);

/* ------------------------------------------------------------------------
 * Solver (device).
 * ---------------------------------------------------------------------- */
typedef struct scfr_config {
    int32_t variant; /* SCFR_CFR .. SCFR_PCFR_PLUS */
    int32_t mode;    /* SCFR_MODE_SIM / SCFR_MODE_ALT */
    double alpha, beta, gamma;
    int32_t batch;   /* independent solves sharing the structure (>= 1) */
    /* Per-solve DCFR/averaging parameters, [batch] each, or NULL to use the
     * scalars above for every solve. */
    const double* batch_alpha;
    const double* batch_beta;
    const double* batch_gamma;
    int32_t engine;  /* SCFR_ENGINE_* */
    /* SCFR_DTYPE_F64 (default; bit-exact with the reference) or
     * SCFR_DTYPE_F32: iteration state and payoff values in fp32, the same
     * operation order rounded to fp32 at every step (level engine only).
     * Reads widen to fp64; exploitability runs in fp64 on the widened
     * profile. */
    int32_t dtype;
    int32_t reserved[6];
} scfr_config;

typedef struct scfr_handle scfr_handle;

/* Copies the structure to `device` and allocates the state of `batch`
 * solves, each initialised like RegretState (t=1, zero regrets, uniform
 * behaviour, zero averages).  UT must be U's stable transpose, as the
 * reference's OperatorSet holds it (CsrMatrix.transposed(), pkg/kernels.py:
 * 95-127): unsharded handles rebuild it on the device from U (bit-identical)
 * and check the caller's arrays only for shape, nnz and a sample of row
 * pointers and entries (SCFR_EINVAL "... not the transpose of U" otherwise);
 * SCFR_HOST_UT=1 in the environment uploads the caller's UT instead. */
int scfr_create(const scfr_tfsdp* p1, const scfr_tfsdp* p2, const scfr_csr* U,
                const scfr_csr* UT, const scfr_config* cfg, int device,
                scfr_handle** out);
/* Multi-GPU row-sharded payoff SpMV (BASELINE config 4).  Every rank of a
 * `world`-rank job holds the whole decision-process state of ONE solve and
 * rank k computes rows [k*c, (k+1)*c) (c = ceil(rows/world)) of U x2 and of
 * -Uᵀ x1; the slices are all-gathered in place over NCCL (loaded at run
 * time) on the handle's stream every iteration, so iterates stay bit-identical
 * to one GPU.  scfr_nccl_unique_id (rank 0) yields the 128-byte id that the
 * caller distributes (e.g. torch.distributed broadcast).  Collective: every
 * rank must call scfr_step / scfr_exploitability / scfr_expected_value
 * together. */
int scfr_nccl_unique_id(char* out128);
int scfr_create_sharded(const scfr_tfsdp* p1, const scfr_tfsdp* p2, const scfr_csr* U,
                        const scfr_csr* UT, const scfr_config* cfg, int device,
                        const char* nccl_unique_id, int rank, int world, scfr_handle** out);
/* Multi-GPU subtree-sharded tree passes (the split PAPER.md
 * :102-108 names: replicate the trunk, give each rank whole subtrees).  Each
 * player's trunk (the levels above a split level holding <= 4096 decision
 * points) is computed by every rank; below it rank r owns a contiguous range
 * of subtree roots of each player, chosen (scfr_subtree_plan) so that its
 * payoff rows read only its own subtrees' and the trunk's strategies.  Every
 * level launch covers only the rank's decision points; after each bottom-up
 * launch of a split level the roots' values are exchanged over NCCL (one
 * in-place broadcast per rank, inside the CUDA graph), so the trunk sees
 * exactly the one-GPU values and iterates stay bit-identical to one GPU.
 * Reads (state, averages, exploitability, expected value) first gather the
 * subtree state of every rank; scfr_status reports what this rank computed
 * (its subtrees and the trunk).  Fused level engine, fp64, batch 1.
 * Collective like scfr_create_sharded.  SCFR_EINVAL when the game has no such
 * split (trunk rows coupled to subtree columns, fewer closed root blocks than
 * ranks, ...). */
int scfr_create_subtree(const scfr_tfsdp* p1, const scfr_tfsdp* p2, const scfr_csr* U,
                        const scfr_csr* UT, const scfr_config* cfg, int device,
                        const char* nccl_unique_id, int rank, int world, scfr_handle** out);
/* Host-only planner of the subtree mode (no GPU needed): the split level of
 * each player (ls_out[2], merged-level index), the root boundaries of every
 * rank (cuts_out[2 * (world + 1)]: player k's rank r owns level-ls roots
 * [cuts[k*(world+1)+r], cuts[k*(world+1)+r+1])) and, if seqs_out is not NULL,
 * the subtree sequences of each rank (seqs_out[2 * world]). */
int scfr_subtree_plan(const scfr_tfsdp* p1, const scfr_tfsdp* p2, const scfr_csr* U, int world,
                      int32_t* ls_out, int64_t* cuts_out, int64_t* seqs_out);

/* Runs n full iterations (_step semantics incl. t++ for both players) on the
 * handle's stream; asynchronous. */
int scfr_step(scfr_handle* h, int64_t n_iter);
/* Caller-computed per-iteration scalars for the next n iterations (t+1 ..
 * t+n) of one solve (solve = -1: every solve): the averaging weight w_t
 * (reference float(t)**gamma, pkg/solvers.py:172) and the DCFR factors
 * pf_t / nf_t for positive / negative regrets (pkg/solvers.py:82-94).  A NULL
 * array keeps the library's values (libm pow, the reference's semantics).
 * Entries must be finite (SCFR_EINVAL). */
int scfr_set_schedule(scfr_handle* h, int solve, const double* w_t, const double* pf_t, const double* nf_t,
                      int64_t n);
/* The engine the handle runs (SCFR_ENGINE_*; AUTO resolved at creation). */
int scfr_engine(const scfr_handle* h, int* engine);
int scfr_synchronize(scfr_handle* h);
/* Saves (restore = 0) or restores (restore = 1) the whole iteration state of
 * the handle (every solve, and the iteration counters) in device memory:
 * a time-to-target search checks every K iterations and, on a hit, replays
 * the last K from the snapshot to find the first iteration that meets the
 * target (paper_2605_14277_b200.solve_to_target). */
int scfr_snapshot(scfr_handle* h, int restore);
/* Completed iterations (the reference's RegretState.t - 1). */
int scfr_iterations(const scfr_handle* h, int64_t* out);
/* Normalised average strategy avg_accum / avg_weight over Σ (player 1/2). */
int scfr_read_average(scfr_handle* h, int player, int solve, double* host_out);
/* Both players' average strategies in one call (RunResult.average, pkg/
 * solvers.py:129-134 for each RegretState, :436-438): the same values as two
 * scfr_read_average calls, with player 2's device->host copy overlapping the
 * copy out of player 1's.  host_out1 / host_out2: num_seqs of player 1 / 2. */
int scfr_read_averages(scfr_handle* h, int solve, double* host_out1, double* host_out2);
/* The sequence-form strategy emitted by the last iteration (x1/x2 of _step). */
int scfr_read_current(scfr_handle* h, int player, int solve, double* host_out);
#define SCFR_STATE_REGRETS 0  /* [num_seqs-1]  RegretState.regrets   */
#define SCFR_STATE_BEHAVIOR 1 /* [num_seqs-1]  RegretState.behavior; for non-predictive
                               * variants the behaviour the NEXT iteration plays (regret
                               * matching of the current regrets, fused into the observe
                               * pass; the reference computes the same b at the start of
                               * the next next_strategy) */
#define SCFR_STATE_ACCUM 2    /* [num_seqs]    RegretState.avg_accum */
#define SCFR_STATE_UTILITY 3  /* [num_seqs]    u of the last iteration (the next prediction) */
int scfr_read_state(scfr_handle* h, int player, int solve, int which, double* host_out);
int scfr_avg_weight(const scfr_handle* h, int player, int solve, double* out);
/* NashConv/2 of the average (which=0) or last emitted (which=1) profile,
 * computed on the device; br1/br2 may be NULL. */
int scfr_exploitability(scfr_handle* h, int solve, int which, double* expl,
                        double* br1, double* br2);
/* Player-1 expected value x1ᵀ U x2 of the average profile (metrics.expected_value). */
int scfr_expected_value(scfr_handle* h, int solve, double* out);
/* Best-response values of both players against an arbitrary host profile
 * (x1 over Σ1, x2 over Σ2): metrics.best_response_values, pkg/metrics.py:59-68. */
int scfr_best_response_values(scfr_handle* h, const double* x1, const double* x2, double* br1,
                              double* br2);
/* x1ᵀ (U x2) for an arbitrary host profile (metrics.expected_value, pkg/metrics.py:50-56). */
int scfr_expected_value_of(scfr_handle* h, const double* x1, const double* x2, double* out);
/* Non-finite flag raised by any kernel since creation (FloatingPointError). */
int scfr_status(scfr_handle* h, int* nonfinite);
/* Device bytes held by the handle (structure + state). */
int scfr_device_bytes(const scfr_handle* h, int64_t* out);
/* Number of kernel launches issued by scfr_step so far (graph nodes count
 * individually). */
int scfr_launch_count(const scfr_handle* h, int64_t* out);
/* Kernel-only device time of the last scfr_step in ms (CUDA events on the
 * handle's stream), and the summed duration of the payoff-SpMV kernels. */
int scfr_last_step_ms(scfr_handle* h, double* total_ms);

/* Runs n iterations (real ones: state advances) without the graph, timing
 * every kernel launch with CUDA events on the handle's stream; aggregates
 * per kernel kind (td_avg, td, cur, obs_rm, obs, pred, spmv, tick): launch
 * count, summed device ms and algorithmic HBM bytes. */
typedef struct scfr_kernel_stat {
    char name[16];
    int64_t launches;
    double ms;
    double bytes;
} scfr_kernel_stat;
int scfr_profile_step(scfr_handle* h, int64_t n_iter, scfr_kernel_stat* out, int cap, int* count);
/* In-graph timeline of the level engine: runs n_iter iterations (they count,
 * as with scfr_step) through a copy of the iteration graph whose kernels
 * record their first-CTA start and last-CTA end (%globaltimer).  With
 * overlapped alt iterations the recorded graph is the two-stream body
 * (n_iter >= 2: prologue, n_iter - 1 recorded bodies, epilogue).  One span
 * per launch, times in microseconds from the iteration's first start,
 * averaged; stream 0 / 1; bytes = the launch's algorithmic bytes.  Spans
 * ordered by end time partition the step: each instant belongs to the
 * launch that finishes next. */
typedef struct scfr_kernel_span {
    char name[16];
    int32_t kind;
    int32_t stream;
    double bytes;
    double start_us, end_us;
} scfr_kernel_span;
int scfr_timeline(scfr_handle* h, int64_t n_iter, scfr_kernel_span* out, int cap, int* count);
/* Process-wide bytes copied host->device and device->host by this library
 * (structure uploads, state reads); used for the end-to-end accounting. */
int scfr_transfer_bytes(int64_t* h2d, int64_t* d2h);
int scfr_destroy(scfr_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* SEQCFR_B200_H */
