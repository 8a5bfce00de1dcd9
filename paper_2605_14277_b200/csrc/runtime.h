// Device-runtime types shared by the level engine (solver.cu) and the
// persistent engine (persistent.cu).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <utility>
#include <cstdint>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges are no-ops unless a profiler injects

#include "common.h"
#include "kernels.cuh"

#define CUDA_OK(expr)                                                                      \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess)                                                             \
            ::scfr::fail(SCFR_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));     \
    } while (0)

namespace scfr {

constexpr int TPB = 128;

// NVTX range over a scope (host API entry points and create stages), so an
// nsys / ncu timeline shows where host time goes around the kernels.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Process-wide host<->device byte counters (scfr_transfer_bytes).
inline std::atomic<int64_t> g_h2d{0}, g_d2h{0};
inline void count_copy(size_t n, cudaMemcpyKind k) {
    if (k == cudaMemcpyHostToDevice) g_h2d += (int64_t)n;
    else if (k == cudaMemcpyDeviceToHost) g_d2h += (int64_t)n;
}
inline cudaError_t copy_async(void* dst, const void* src, size_t n, cudaMemcpyKind k,
                              cudaStream_t s) {
    count_copy(n, k);
    return cudaMemcpyAsync(dst, src, n, k, s);
}
inline cudaError_t copy_sync(void* dst, const void* src, size_t n, cudaMemcpyKind k) {
    count_copy(n, k);
    return cudaMemcpy(dst, src, n, k);
}

enum KernelKind : int {
    KK_TD_AVG = 0, KK_TD, KK_CUR, KK_OBS_RM, KK_OBS, KK_PRED, KK_SPMV, KK_TICK, KK_PERSIST,
    KK_COUNT
};
inline const char* kKernelNames[KK_COUNT] = {"td_avg", "td", "cur", "obs_rm", "obs",
                                             "pred", "spmv", "tick", "persistent"};
struct KernelRecord {
    int kind;
    double bytes;
    cudaEvent_t e0, e1;
};

// Device buffers come from the device's stream-ordered memory pool, kept
// resident (release threshold raised once per device), so building a second
// solver for the same game reuses memory instead of paying cudaMalloc/cudaFree.
// The allocating stream is thread-local state set by the API entry points.
inline thread_local cudaStream_t g_alloc_stream = nullptr;
struct AllocStream {
    cudaStream_t prev;
    explicit AllocStream(cudaStream_t s) : prev(g_alloc_stream) { g_alloc_stream = s; }
    ~AllocStream() { g_alloc_stream = prev; }
};

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    bool pooled = false;
    // kPad bytes past the end: bulk copies may round ranges out to 16-byte
    // granules, so the last granule may extend past n.
    static constexpr size_t kPad = 16;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;  // owns device memory: never copied
    DevBuf& operator=(const DevBuf&) = delete;
    void alloc(size_t count) {
        free();
        n = count;
        if (!count) return;
        if (g_alloc_stream) {
            CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T) + kPad, g_alloc_stream));
            pooled = true;
        } else {
            CUDA_OK(cudaMalloc(&p, count * sizeof(T) + kPad));
        }
    }
    void zero(cudaStream_t s) {
        if (n) CUDA_OK(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
    void free() {
        // callers synchronise the owning stream before buffers die
        if (p) {
            if (pooled) cudaFreeAsync(p, 0);
            else cudaFree(p);
        }
        p = nullptr;
        n = 0;
        pooled = false;
    }
    size_t bytes() const { return n * sizeof(T); }
    ~DevBuf() { free(); }
};

// State vectors are DevBuf<double>; in the fp32 mode they hold floats
// (allocated with half the doubles) and are accessed through vals<R>().
template <class R>
inline R* vals(const DevBuf<double>& b) {
    return reinterpret_cast<R*>(b.p);
}
inline size_t val_slots(size_t count, bool f32) { return f32 ? (count + 1) / 2 : count; }

struct Player {
    int S = 0, J = 0;
    int max_actions = 0;
    std::vector<int> lvl;                        // DP level starts (process depth), size L+1
    std::vector<double> lvl_ns, lvl_nj, lvl_nc;  // per level: sequences, DPs, child-DP refs
    std::vector<int> lvl_maxa;                   // per level: widest DP (actions)
    std::vector<int> lvl_pmin;                   // per level: smallest parent sequence of its DPs
    std::vector<int> lvl_s0;                     // per level: first sequence
    std::vector<DevTree> lvl_shape;              // per level: affine shape (pointers unset)
    // int32 host structure, valid only while scfr_create runs (host scratch
    // reused across creates, see HostScratch in host_par.h): the tile planner
    const std::vector<int>* h_seq_ptr = nullptr;
    const std::vector<int>* h_dp_parent = nullptr;
    DevBuf<int> seq_ptr, dp_parent;
    DevBuf<int2> child;
    DevBuf<double> r, b, x, xpost, avg, u, V;  // batched [B][...]
    DevBuf<double> g, W, xbar;                 // best-response scratch, one solve
    DevBuf<double> wide;                       // fp32 mode: a widened read of one vector
    DevBuf<double> bcur;                       // player 1, predictive alt mode: OBS's regret matching, read by CUR
    DevBuf<double> PV;                         // predictive variants: PRED's DP values (OBS keeps V), so the
                                               // two passes' levels can overlap (solver.cu body_t)
    DevTree tree() const { return DevTree{seq_ptr.p, dp_parent.p, child.p}; }
    int levels() const { return (int)lvl.size() - 1; }
};

struct DevCsr {
    int rows = 0, cols = 0, nnz = 0;  // rows / nnz held on this device (a shard if sharded)
    int full_rows = 0, row0 = 0, chunk = 0;  // global rows; first local row; rows per rank
    // indptr at selected global rows (the players' level boundaries), for the
    // per-launch byte accounting of the fused SpMV
    std::vector<int> h_rows;
    std::vector<int64_t> h_ptr;
    // per level of the row player: the non-zero count every row of the level
    // shares, else -1 (kernels.cuh FuseUT::rc; unsharded matrices only)
    std::vector<int> lvl_rowc;
    int64_t ptr_at(int row) const {
        const auto it = std::lower_bound(h_rows.begin(), h_rows.end(), row);
        return it != h_rows.end() && *it == row ? h_ptr[it - h_rows.begin()] : 0;
    }
    DevBuf<int> indptr, indices;
    DevBuf<int> indices_iter;  // iteration copy with forced-leaf columns -> parent columns (solver.cu leaf_x)
    DevBuf<double> data;
    DevBuf<float> data32;  // fp32 mode: the values rounded once
    const int* iter_indices() const { return indices_iter.p ? indices_iter.p : indices.p; }
};

// One phase of the persistent program: a DP level of one or both players
// (items [0,n1) -> player 1 DPs lo1.., [n1,n1+n2) -> player 2 DPs lo2..),
// or a payoff SpMV over rows.
struct Phase {
    int kind;  // PH_*
    int lo1, n1, lo2, n2;
    int first_avg;  // the first TD_AVG phase also averages x[0] of DP-less players
    int warp1, warp2;  // run this player's DPs warp-per-DP (small fat OBS/PRED levels)
};
enum : int { PH_TD_AVG = 0, PH_TD_POST, PH_CUR, PH_OBS, PH_PRED, PH_SPMV_U, PH_SPMV_UT,
             PH_SPMV_BOTH,
             // SMEM engine only: a whole top-down pass in one phase, each sequence's
             // x from its ancestor chain (items: sequences 1.. of each player)
             PH_TDC_AVG, PH_TDC_POST,
             // ... and player 1's current strategy (predictive alt): regret
             // matching of every DP into bm, then the chain product with bm
             PH_RMC, PH_TDC_CUR };

struct SmemSide {  // byte offsets of one player's arrays in the SMEM engine's buffer
    int r, b, x, xpost, avg, u, V, seq_ptr, dp_parent, child;
    int sdp;  // sequence -> its DP's parent sequence (the chain top-down phases; 0 when absent)
    int bm;   // player 1, chain CUR: the regret-matched strategy (0 when absent)
};
struct SmemPlan {
    SmemSide p[2];
    int prog;  // byte offset of the staged phase program
    int bytes;
    // the payoff rows staged in shared memory (0 bytes: read from global):
    // per matrix int32 row pointers, uint16 columns and uint16 ids into one
    // table of the distinct payoff values (csrc/persistent.cu compact_payoff)
    int csr, csr_bytes;
    int uptr, ucol, uvid, tptr, tcol, tvid, tab;
    int chain;  // chain phases: the longest ancestor chain (DPs)
};

struct PersistentPlan {
    bool grid = false;   // true: one solve over a cooperative grid; false: one CTA per solve
    bool cluster = false;  // one solve per thread-block cluster of csize CTAs
    int csize = 0;
    bool small = false;  // CTA mode with state + structure resident in shared memory
    const void* small_kern = nullptr;  // its kernel (k_small<MAXA>)
    SmemPlan smem{};
    int ctas = 0, threads = 0;
    std::vector<Phase> host_program;
    DevBuf<Phase> program;
    DevBuf<unsigned> barrier;  // {count, generation}
    DevBuf<unsigned char> csr_blob;  // SmemPlan::csr block, staged into shared memory
    int csr_rel[7] = {};             // uptr, ucol, uvid, tptr, tcol, tvid, tab within the blob
    bool chain = false;              // SMEM engine: one top-down phase per pass (PH_TDC_*)
};

// Programmatic Dependent Launch (sm_90+): let the next kernel in the stream
// start launching now / wait until the previous grid's writes are visible.
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool predictive(int v);
int post_of(int v);
inline bool is_persistent(int engine) {
    return engine == SCFR_ENGINE_PERSISTENT || engine == SCFR_ENGINE_PERSISTENT_GRID ||
           engine == SCFR_ENGINE_PERSISTENT_CLUSTER;
}
inline int grid_for(int n) { return n <= 0 ? 1 : (n + TPB - 1) / TPB; }
// Levels whose widest DP has at least this many actions run warp-per-DP
// (SCFR_WIDE_ACTIONS overrides; large values disable).
inline const int kWideActions = [] {
    const char* e = std::getenv("SCFR_WIDE_ACTIONS");
    return e ? std::atoi(e) : 5;
}();

// Per-iteration parameters shared by every pass kernel: host-computed
// schedules indexed by the device iteration counter, the variant's post-op.
struct KParams {
    const double* wsched;
    const double* pfsched;
    const double* nfsched;
    int cap;
    const long long* tdev;
    int post, do_rm, plus;
    int* nonfinite;
    // scfr_timeline: first-CTA start / last-CTA end (%globaltimer ns) of this
    // launch, slots [2 * tl_idx, 2 * tl_idx + 1]; null when not recording
    unsigned long long* tl;
    int tl_idx;
    // schedule index = *tdev + tofs: the overlapped alt iteration runs the
    // next iteration's PRED / TD + average before the tick (tofs = 1)
    int tofs;
};

// Timeline records of a launch (scfr_timeline): every CTA's thread 0 after
// the PDL wait (start: min) and after the CTA's last thread (end: max).
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// (the start slot holds the maximum of ~t, so both slots start at zero)
__device__ __forceinline__ void tl_start(unsigned long long* tl, int idx) {
    if (tl && threadIdx.x == 0) atomicMax(tl + 2 * idx, ~global_ns());
}
__device__ __forceinline__ void tl_end(unsigned long long* tl, int idx) {
    if (tl) {
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(tl + 2 * idx + 1, global_ns());
    }
}

// Tile engine plan of one player (tiled.cu): DPs below the split level are
// renumbered tile-major (tile, level, root-first, original order) so every
// tile is a contiguous block of DPs and of sequences.
struct TileShape {  // one (tile, level) block, or one top level
    int j_lo, s_lo, un, cn, c_lo, pc, p_lo, nroot;
};
struct TilePlayer {
    int ls = 0;           // split level: levels [0, ls) are the top, [ls, L) are tiled
    int Jtop = 0, Stop = 0;  // top DPs [0, Jtop), top sequences [0, Stop) (ids unchanged)
    int ntiles = 0, nlev = 0;
    int max_dps = 0, max_seqs = 0;  // largest tile (shared-memory sizing)
    int maxa = 1;                   // widest DP below the split
    std::vector<int> top_lvl;       // [ls+1] level starts of the top
    std::vector<TileShape> top_shape;
    unsigned top_warp = 0;          // top levels run warp-per-DP (fat)
    std::vector<int> h_off;         // [ntiles][nlev+1] device DP offsets of the level blocks
    std::vector<TileShape> h_shape; // [ntiles][nlev]
    DevBuf<int> seq_ptr, dp_parent, off, sperm, dperm;
    DevBuf<int2> child;
    DevBuf<TileShape> shape;
    DevBuf<unsigned> ticket;  // [B] last-CTA tickets
    DevBuf<double> gat;       // original-order scratch for reads
    // algorithmic bytes of one pass (host accounting)
    double bytes_obs = 0, bytes_obs_rm = 0, bytes_pred = 0, bytes_td_avg = 0, bytes_td = 0,
           bytes_cur = 0, bytes_spmv = 0;
};

// Pass kinds of the level kernels.
enum : int { LK_TD_AVG = 0, LK_TD, LK_CUR, LK_OBS, LK_PRED };

constexpr int kTopMax = 8;  // top levels

// The level engine's top (solver.cu prepare_top): top-down passes do not
// launch levels [0, ls) of a player; its level-ls launch recomputes each
// parent's x from the ancestor chain.  Lives in device memory.
struct TopInfo {
    int ls, Stop;      // top levels, top sequences [0, Stop)
    const int* anc;    // [Stop][ls] ancestor sequences top-down (-1 pad; bit 30: forced level, b = 1.0)
    int pro;           // 1: the level-ls launch also writes the top's x (top_prologue); 0: nobody reads it
};
struct TopPlayer {
    bool on = false;
    int ls = 0;
    DevBuf<int> anc;
    DevBuf<TopInfo> info;
};

}  // namespace scfr

namespace scfr {
// scfr_snapshot: saved state vectors, device iteration counter, host counters.
struct Snapshot {
    bool valid = false;
    DevBuf<double> buf[2][7];  // per player: r, b, x, xpost, avg, u, V
    DevBuf<long long> tdev;
    int64_t t = 0;
    std::vector<double> avg_weight;
};
}  // namespace scfr

struct scfr_handle {
    int device = 0;
    int B = 1;
    bool f32 = false;  // SCFR_DTYPE_F32: iteration state in fp32
    int variant = 0, mode = 0;
    int engine = SCFR_ENGINE_LEVELS;
    int num_sms = 148;
    std::vector<double> alpha, beta, gamma;
    scfr::Player P[2];
    scfr::DevCsr U, UT;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int cap = 0;                 // schedule capacity (iterations)
    std::vector<double> w_host, pf_host, nf_host;  // [B][cap] schedules (t^gamma, DCFR factors)
    scfr::DevBuf<double> wsched, pfsched, nfsched;
    scfr::DevBuf<long long> tdev;
    scfr::DevBuf<int> nonfinite;
    scfr::DevBuf<double> brout;
    int64_t t = 0;                   // completed iterations
    std::vector<double> avg_weight;  // [B]
    cudaGraphExec_t exec = nullptr;
    int64_t nodes_per_iter = 0;
    // Overlapped alt iterations (solver.cu Launcher::body_t; SCFR_NO_OVERLAP=1:
    // off): prologue (next of both players), body (observe of iteration t with
    // player 1's next of t+1 on a second stream beside player 2's observe and
    // next), epilogue (observe of the last iteration)
    bool overlap = false;
    int prio_hi = 0;  // the overlapped body's critical stream (B) launch priority (SCFR_NO_PRIO=1: 0)
    int64_t prio_nj = 1000;  // ... for its launches of at most this many DPs (the top levels)
    cudaStream_t stream2 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_a = nullptr, ev_b = nullptr;
    // player 2's observe above its deepest launch on stream3, gating PRED2
    // level by level (ev_lv[l]: OBS2 of level l done); opt-in SCFR_OBS_SIDE=1
    cudaStream_t stream3 = nullptr;
    static constexpr int kSideLevels = 16;
    cudaEvent_t ev_side = nullptr, ev_lv[kSideLevels] = {};
    static constexpr int kReadParts = 8;
    static constexpr int kReadEvents = 2 * kReadParts;  // (two segments: scfr_read_averages)
    cudaEvent_t rd_ev[kReadEvents] = {};  // chunked device->host reads (read_to_host_multi)
    cudaGraphExec_t exec_pro = nullptr, exec_body = nullptr, exec_epi = nullptr;
    int64_t nodes_pro = 0, nodes_body = 0, nodes_epi = 0;
    int64_t launches = 0;
    bool use_graph = true;
    bool pdl = true;   // programmatic dependent launch between level kernels
    bool fuse = true;  // payoff SpMV fused into the observe pass (level engine)
    bool affine_rows = true;  // fused SpMV indexes equal-length level rows without indptr (SCFR_NO_ROW_SHAPE)
    bool small_warp = true;   // warp-per-DP on small multi-action levels (SCFR_NO_SMALL_WARP=1: off)
    int64_t warp_nj = 4096;  // size limit of the fat / small warp rules (SCFR_WARP_NJ)
    bool bcur_on = false;  // predictive alt: OBS P1 writes RM(r) to P[0].bcur, CUR is a plain TD (SCFR_NO_BCUR=1: off)
    bool group = true;
    bool leaf_fuse = true;  // OBS: the forced leaf level computed in the group launch above it (SCFR_NO_LEAF_FUSE=1)
    bool pipe = true;            // big affine group levels: the cp.async-pipelined kernel (SCFR_NO_PIPE=1: off)
    int64_t pipe_nj = 65536;     // ... on levels of at least this many DPs (SCFR_PIPE_NJ)
    int pipe_kinds = 1 << 0;     // ... for these LK_* kinds (SCFR_PIPE_KINDS bit mask; TD + average only:
                                 //     OBS / PRED / CUR measured slower pipelined)
    bool pair = false;  // bottom-up group launches also compute the parent level (opt-in SCFR_PAIR=1)
    int64_t group_nj = 4096;  // group mode only above this many DPs per level (SCFR_GROUP_NJ)  // big affine 2..16-action levels run G = 32/n DPs per warp (SCFR_NO_GROUP=1: off)
    bool td_warp = true;    // top-down passes warp-per-DP on wide levels (SCFR_NO_TD_WARP=1: thread per DP)
    bool leaf_skip = true;  // PRED skips a forced deepest level (kernels.cuh leaf_note; SCFR_NO_LEAF_SKIP)
    bool leaf_x = false;    // level engine: forced leaf x / avg are parent copies (solver.cu k_expand_leaf)
    bool u_empty_skip = false;  // levels with empty payoff rows neither compute nor read u (kernels.cuh ld_u)
    std::vector<std::pair<int, int>> neg_zero_rows;  // player 2 rows {first, count} holding -0.0
    bool wave_ctas_env = false;
    int wave_ctas = 12;  // level-kernel grid cap per task, in CTAs per SM (SCFR_WAVE_CTAS)
    bool timed = false;
    scfr::PersistentPlan plan;
    scfr::Snapshot snap;
    // Multi-GPU modes: NCCL communicator (ncclComm_t) over `world` ranks,
    // this handle being `rank`; the row-sharded payoff SpMV
    // (scfr_create_sharded) or, with `subtree`, the subtree-sharded tree
    // passes (scfr_create_subtree, subtree.h): launches of levels >= sub_ls[k]
    // cover DPs [sub_jb[k][l][rank], sub_jb[k][l][rank + 1]) (sequences
    // sub_sb), the roots' V is broadcast after bottom-up split launches, and
    // reads gather the other ranks' subtrees first (sub_stale)
    void* comm = nullptr;
    void* comm2 = nullptr;  // subtree mode, overlapped alt body: stream2's communicator (ncclCommSplit)
    int world = 1, rank = 0;
    bool subtree = false, sub_stale = false;
    int sub_ls[2] = {-1, -1};
    int sub_sim = 1;    // SCFR_SUBTREE_SIM (world 1): ranks simulated by split launches
    int sub_view = -1;  // SCFR_SUBTREE_VIEW (world 1, timing): one rank's launches of a larger plan
    std::vector<std::vector<int>> sub_jb[2], sub_sb[2];
    bool rowshard() const { return comm && !subtree; }
    // Tile engine (SCFR_ENGINE_TILED): per-player plans and the payoff rows
    // in the tile numbering (rows of U for player 1, of Uᵀ for player 2).
    scfr::TilePlayer tp[2];
    scfr::DevCsr tM[2];
    int tile_threads = 256, tile_grid_up = 0, tile_grid_down = 0;
    int tile_vwin = 0;       // doubles of the up pass's V window (largest tile)
    int tile_dwin = 0;       // doubles of the down pass's x window (top + largest tile)
    int tile_staged = 1;     // SCFR_TILE_STAGE=0: no shared-memory staging (A/B)
    size_t tile_smem_up = 0, tile_smem_down = 0;
    std::vector<std::pair<const void*, int>> tile_occ;  // resident CTAs per SM, per tile kernel
    // The level engine's top (prepare_top; SCFR_NO_TOP=1: off), and player 1's
    // deeper top for its current-strategy pass (alt mode: x1' is read only by
    // player 2's payoff rows, all of which read level-ls sequences; no prologue)
    scfr::TopPlayer top[2];
    scfr::TopPlayer top_cur;
    void (*comm_destroy)(void*) = nullptr;  // set with comm (NCCL is dlopen'ed)
    ~scfr_handle() {
        // in-flight async copies / kernels may still use buffers that the
        // member destructors free: drain the stream first (also on a failed
        // create, where this destructor runs from the unique_ptr)
        if (stream) cudaStreamSynchronize(stream);
        if (comm2 && comm_destroy) comm_destroy(comm2);
        comm2 = nullptr;
        if (comm && comm_destroy) comm_destroy(comm);
        comm = nullptr;
        if (exec) cudaGraphExecDestroy(exec);
        for (cudaGraphExec_t e : {exec_pro, exec_body, exec_epi})
            if (e) cudaGraphExecDestroy(e);
        if (stream2) cudaStreamSynchronize(stream2);
        if (stream3) cudaStreamSynchronize(stream3);
        for (cudaEvent_t e : {ev_fork, ev_a, ev_b, ev_side})
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : ev_lv)
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : rd_ev)
            if (e) cudaEventDestroy(e);
        if (stream2) cudaStreamDestroy(stream2);
        if (stream3) cudaStreamDestroy(stream3);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace scfr {

// Generic launch plumbing shared by the engines: optional per-launch CUDA
// events (scfr_profile_step) and Programmatic Dependent Launch.
struct LaunchBase {
    scfr_handle* h;
    int64_t count = 0;
    cudaStream_t st = nullptr;  // launch stream (null: the handle's)
    int tofs = 0;               // KParams::tofs of the launches
    int prio = 0;               // launch priority attribute (0: none; lower = more urgent)
    unsigned long long* tl = nullptr;  // scfr_timeline buffer while capturing its graph
    struct TlRec {
        int kind;
        double bytes;
        int stream;  // 0: the handle's stream, 1: stream2 (overlapped body)
    };
    std::vector<TlRec>* tl_kinds = nullptr;  // per launch
    std::vector<KernelRecord>* prof = nullptr;  // per-launch events when profiling

    template <class F>
    void launch(int kind, double bytes, F&& f) {
        if (tl_kinds) tl_kinds->push_back(TlRec{kind, bytes * h->B, st && st != h->stream ? 1 : 0});
        if (prof) {
            KernelRecord r;
            r.kind = kind;
            r.bytes = bytes * h->B;
            CUDA_OK(cudaEventCreate(&r.e0));
            CUDA_OK(cudaEventCreate(&r.e1));
            CUDA_OK(cudaEventRecord(r.e0, h->stream));
            f();
            CUDA_OK(cudaEventRecord(r.e1, h->stream));
            prof->push_back(r);
        } else {
            f();
        }
        ++count;
    }

    // Kernel launch with Programmatic Dependent Launch allowed (the kernels
    // call griddepcontrol.launch_dependents / .wait), so the next kernel's
    // grid is set up while this one drains.  SCFR_NO_PDL=1 turns it off.
    template <class... KArgs, class... Args>
    void run_ex(void (*kern)(KArgs...), dim3 grid, int threads, size_t smem, Args... args) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st ? st : h->stream;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = h->pdl ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (prio) {  // (graphs honour it: instantiated with UseNodePriority)
            attr[1].id = cudaLaunchAttributePriority;
            attr[1].val.priority = prio;
            cfg.numAttrs = 2;
        }
        CUDA_OK(cudaLaunchKernelEx(&cfg, kern, args...));
    }
    template <class... KArgs, class... Args>
    void run_threads(void (*kern)(KArgs...), dim3 grid, int threads, Args... args) {
        run_ex(kern, grid, threads, 0, args...);
    }
    template <class... KArgs, class... Args>
    void run(void (*kern)(KArgs...), dim3 grid, Args... args) {
        run_ex(kern, grid, TPB, 0, args...);
    }
    template <class... KArgs, class... Args>
    void run1(void (*kern)(KArgs...), dim3 grid, Args... args) {
        run_ex(kern, grid, 1, 0, args...);
    }
    KParams kparams(bool do_rm) const;
};

// Tile engine (tiled.cu).
bool prepare_tiled(scfr_handle* h, const scfr_csr* U, const scfr_csr* UT, bool required);
void tiled_iteration(LaunchBase& L);
// Device pointer to `buf` (a [B][S] vector of `player` in the engine's
// numbering) for `solve`, in the reference's sequence order.
const double* orig_order(scfr_handle* h, int player, const double* buf, int solve);
__global__ void k_tick(long long* tdev, unsigned long long* tl, int tl_idx);

// solver.cu helpers
bool leaf_single(const scfr_handle* h, const Player& P);
bool warp_level(const scfr_handle* h, const Player& P, int l);

int choose_engine(scfr_handle* h);
void prepare_persistent(scfr_handle* h);
// Enqueues n iterations; returns the number of kernel launches issued.
int64_t launch_persistent(scfr_handle* h, int64_t n);
double persistent_bytes_per_iter(const scfr_handle* h);
}  // namespace scfr
