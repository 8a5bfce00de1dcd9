// Persistent engine: whole CFR iterations inside ONE kernel launch.
//
// The level engine pays one kernel launch (~2-4 µs of graph-node latency)
// per DP level and pass, which is all of the time for games whose levels
// hold a few hundred DPs (Kuhn, Leduc, batched sweeps) and most of it for
// Liar's dice.  Here the iteration is a host-built program of phases; a
// phase is one DP level of one or both players (independent players share a
// phase: both next() passes, both observe passes in simultaneous mode) or a
// payoff SpMV, and phases are separated by a barrier:
//
//   CTA mode   one CTA per solve (batch = grid), barrier = __syncthreads,
//              plain L1-cacheable loads — the whole solve lives on one SM.
//   grid mode  one solve over a cooperative grid (co-residency guaranteed by
//              cudaLaunchCooperativeKernel), barrier = atomic arrive +
//              generation spin with gpu-scope fences, mutable state read
//              L2-only (ld.global.cg) because producers are other SMs.
//
// The per-DP arithmetic is the same code as the level engine
// (kernels.cuh), so iterates are bit-identical across engines.

#include <algorithm>
#include <cstring>
#include <type_traits>

#include <cooperative_groups.h>

#include "runtime.h"

namespace scfr {

struct PArgs {
    DevTree T[2];
    double* r[2];
    double* b[2];
    double* x[2];
    double* xpost[2];
    double* avg[2];
    double* u[2];
    double* V[2];
    int S[2], J[2];
    const int* Uip;
    const int* Uix;
    const double* Ud;
    int Urows;
    const int* Tip;
    const int* Tix;
    const double* Td;
    int Trows;
    const double* wsched;
    const double* pfsched;
    const double* nfsched;
    int cap;
    const Phase* prog;
    int nphase;
    long long t0;
    int n_iter;
    int post, pred, plus, alt;
    int* nonfinite;
    long long* tdev;
    unsigned* barrier;
    long long* trace;  // SCFR_PHASE_TRACE=1: per-phase clock64 deltas (CTA 0, thread 0)
    const unsigned char* csr;  // SmemPlan::csr block (SMEM engine)
};

__device__ __forceinline__ void grid_sync(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// One phase's share of DPs for player-K, run by this thread: items
// begin, begin+stride, ... < n of the level starting at DP lo.  Out of line
// (one call per phase per thread) so each pass is register-allocated on its
// own instead of every pass being inlined into the persistent loop.
template <int MAXA, class Ld>
__device__ __noinline__ void phase_dps(int kind, DevTree T, int lo, int n, int begin, int stride,
                                       const double* u, double* r, double* b, double* x,
                                       double* xpost, double* avg, double* V, double w, int post,
                                       double pf, double nf, int pred, int plus, int* nonfinite,
                                       bool warp) {
    if (warp && (kind == PH_OBS || kind == PH_PRED)) {
        // warp-per-DP (fat / wide levels): begin and stride count warps
        const int lane = threadIdx.x & 31;
        for (int i = begin; i < n; i += stride) {
            const int j = lo + i;
            if (kind == PH_OBS)
                obs_dp_warp<Ld>(T, j, u, r, b, V, post, pf, nf, pred == 0, nonfinite, lane);
            else
                pred_dp_warp<Ld>(T, j, u, r, b, V, plus != 0, lane);
        }
        return;
    }
    for (int i = begin; i < n; i += stride) {
        const int j = lo + i;
        switch (kind) {
            case PH_TD_AVG:
                if (j == 0) avg[0] = dadd(dmul(w, Ld::ld(x)), Ld::ld(avg));
                td_dp<Ld>(T, j, b, x, avg, w);
                break;
            case PH_TD_POST:
                td_dp<Ld>(T, j, b, xpost, nullptr, 0.0);
                break;
            case PH_CUR:
                cur_dp<MAXA, Ld>(T, j, r, xpost);
                break;
            case PH_OBS:
                obs_dp<MAXA, Ld>(T, j, u, r, b, V, post, pf, nf, pred == 0, nonfinite);
                break;
            case PH_PRED:
                pred_dp<MAXA, Ld>(T, j, u, r, b, V, plus != 0);
                break;
        }
    }
}

// Payoff SpMV share: rows [begin, n) step stride of M applied to x into out
// (optionally scaled by -1).
template <class Ld>
__device__ __noinline__ void phase_spmv(const int* ip, const int* ix, const double* d, int n,
                                        int begin, int stride, const double* x, double* out,
                                        bool neg, int* nonfinite) {
    for (int i = begin; i < n; i += stride) {
        double acc = spmv_row<Ld>(ip, ix, d, x, i);
        if (neg) acc = dmul(-1.0, acc);
        if (!isfinite(acc)) atomicOr(nonfinite, 1);
        out[i] = acc;
    }
}

template <int K, int MAXA, class Ld>
__device__ __forceinline__ void player_phase(const PArgs& a, const Phase& ph, int lo, int n,
                                             int begin, int stride, int solve, double w,
                                             double pf, double nf, bool warp) {
    if (n <= 0) return;
    const size_t o = (size_t)solve * a.S[K];
    phase_dps<MAXA, Ld>(ph.kind, a.T[K], lo, n, begin, stride, a.u[K] + o, a.r[K] + o,
                        a.b[K] + o, a.x[K] + o, a.xpost[K] + o, a.avg[K] + o,
                        a.V[K] + (size_t)solve * (a.J[K] > 0 ? a.J[K] : 1), w, a.post, pf, nf,
                        a.pred, a.plus, a.nonfinite, warp);
}

// MODE: PM_CTA (one CTA per solve, __syncthreads), PM_GRID (one solve over
// a cooperative grid, atomic grid barrier), PM_CLUSTER (one solve per
// thread-block cluster of up to 16 SMs, hardware cluster barrier; a batch is
// one cluster per solve).  Grid and cluster modes read mutable state from L2
// (ld.global.cg): the producers are other SMs.
enum : int { PM_CTA = 0, PM_GRID = 1, PM_CLUSTER = 2 };

template <int MODE, int MAXA, int THREADS>
__global__ void __launch_bounds__(THREADS) k_persistent(const __grid_constant__ PArgs a) {
    constexpr bool GRID = MODE == PM_GRID;
    using Ld = std::conditional_t<MODE != PM_CTA, LdL2, LdL1>;
    int solve = 0, rank = 0, size = 0;
    if constexpr (MODE == PM_CLUSTER) {
        const cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
        solve = blockIdx.x / (int)cl.num_blocks();
        rank = (int)cl.block_rank() * blockDim.x + threadIdx.x;
        size = (int)cl.num_blocks() * blockDim.x;
    } else {
        solve = GRID ? 0 : blockIdx.x;
        rank = GRID ? blockIdx.x * blockDim.x + threadIdx.x : threadIdx.x;
        size = GRID ? gridDim.x * blockDim.x : blockDim.x;
    }
    const size_t o1 = (size_t)solve * a.S[0], o2 = (size_t)solve * a.S[1];
    for (int it = 0; it < a.n_iter; ++it) {
        const size_t si = (size_t)solve * a.cap + (size_t)(a.t0 + it);
        const double w = a.wsched[si];
        const double pf = a.post == POST_DCFR ? a.pfsched[si] : 1.0;
        const double nf = a.post == POST_DCFR ? a.nfsched[si] : 1.0;
        for (int p = 0; p < a.nphase; ++p) {
            const Phase ph = a.prog[p];
            if (ph.kind < PH_SPMV_U) {
                // items [0,n1) are player-1 DPs, [n1,n1+n2) player-2 DPs; in
                // warp mode an item is a warp (lanes = actions)
                const int wr = rank >> 5, ws = size >> 5;
                const bool w1 = ph.warp1 && ws > 0, w2 = ph.warp2 && ws > 0;
                player_phase<0, MAXA, Ld>(a, ph, ph.lo1, ph.n1, w1 ? wr : rank, w1 ? ws : size, solve,
                                          w, pf, nf, w1);
                const int r2 = w2 ? wr : rank, s2 = w2 ? ws : size;
                const int n1u = w1 == w2 ? ph.n1 : 0;  // continue after player 1's items
                const int b2 = ((r2 - n1u) % s2 + s2) % s2;
                player_phase<1, MAXA, Ld>(a, ph, ph.lo2, ph.n2, b2, s2, solve, w, pf, nf, w2);
            } else {
                // payoff SpMV: rows of U (-> u1), then rows of Uᵀ (-> u2 = -Uᵀ x1)
                const double* x1 = (a.alt ? a.xpost[0] : a.x[0]) + o1;
                if (ph.kind != PH_SPMV_UT)
                    phase_spmv<Ld>(a.Uip, a.Uix, a.Ud, a.Urows, rank, size, a.x[1] + o2,
                                   a.u[0] + o1, false, a.nonfinite);
                if (ph.kind != PH_SPMV_U) {
                    const int b2 = ph.kind == PH_SPMV_BOTH ? ((rank - a.Urows) % size + size) % size : rank;
                    phase_spmv<Ld>(a.Tip, a.Tix, a.Td, a.Trows, b2, size, x1, a.u[1] + o2, true,
                                   a.nonfinite);
                }
            }
            // a player without decision points still averages x[0] = 1
            if (ph.first_avg && rank == 0) {
                if (a.J[0] == 0) a.avg[0][o1] = dadd(dmul(w, Ld::ld(a.x[0] + o1)), Ld::ld(a.avg[0] + o1));
                if (a.J[1] == 0) a.avg[1][o2] = dadd(dmul(w, Ld::ld(a.x[1] + o2)), Ld::ld(a.avg[1] + o2));
            }
            if constexpr (MODE == PM_CLUSTER) cooperative_groups::this_cluster().sync();
            else if constexpr (GRID) grid_sync(a.barrier);
            else __syncthreads();
        }
    }
    if (rank == 0 && (GRID || (MODE == PM_CLUSTER ? solve == 0 : blockIdx.x == 0))) *a.tdev = a.t0 + a.n_iter;
}

// ---------------------------------------------------------------------------
// SMEM-resident CTA engine: when one solve's state and structure fit in
// shared memory (Kuhn, Leduc, ...), each CTA stages them in once per launch,
// runs every phase of every iteration against shared memory (LdS: ~30-cycle
// loads instead of L1/L2 round trips on the per-phase critical path), and
// writes the state back at the end.  U and Uᵀ stay in global memory behind
// the read-only path.

struct SPtrs {
    double *r, *b, *x, *xpost, *avg, *u, *V;
    DevTree T;
};

__device__ __forceinline__ SPtrs carve(unsigned char* sm, const SmemSide& o, bool has_xpost) {
    SPtrs p;
    p.r = reinterpret_cast<double*>(sm + o.r);
    p.b = reinterpret_cast<double*>(sm + o.b);
    p.x = reinterpret_cast<double*>(sm + o.x);
    p.xpost = has_xpost ? reinterpret_cast<double*>(sm + o.xpost) : nullptr;
    p.avg = reinterpret_cast<double*>(sm + o.avg);
    p.u = reinterpret_cast<double*>(sm + o.u);
    p.V = reinterpret_cast<double*>(sm + o.V);
    p.T.seq_ptr = reinterpret_cast<const int*>(sm + o.seq_ptr);
    p.T.dp_parent = reinterpret_cast<const int*>(sm + o.dp_parent);
    p.T.child = reinterpret_cast<const int2*>(sm + o.child);
    return p;
}

// Copies one player's state (and, when `structure`, its index arrays)
// between global memory (solve slice) and shared memory.
template <int K>
__device__ __forceinline__ void stage(const PArgs& a, const SPtrs& s, int solve, bool in) {
    const size_t o = (size_t)solve * a.S[K];
    const int S = a.S[K];
    for (int i = threadIdx.x; i < S; i += blockDim.x) {
        if (in) {
            s.r[i] = a.r[K][o + i];
            s.b[i] = a.b[K][o + i];
            s.x[i] = a.x[K][o + i];
            if (s.xpost) s.xpost[i] = a.xpost[K][o + i];
            s.avg[i] = a.avg[K][o + i];
            s.u[i] = a.u[K][o + i];
            const_cast<int2*>(s.T.child)[i] = __ldg(a.T[K].child + i);
        } else {
            a.r[K][o + i] = s.r[i];
            a.b[K][o + i] = s.b[i];
            a.x[K][o + i] = s.x[i];
            if (s.xpost) a.xpost[K][o + i] = s.xpost[i];
            a.avg[K][o + i] = s.avg[i];
            a.u[K][o + i] = s.u[i];
        }
    }
    if (in) {
        const int J = a.J[K];
        for (int i = threadIdx.x; i <= J; i += blockDim.x) {
            const_cast<int*>(s.T.seq_ptr)[i] = __ldg(a.T[K].seq_ptr + i);
            if (i < J) const_cast<int*>(s.T.dp_parent)[i] = __ldg(a.T[K].dp_parent + i);
        }
    }
}

// Shared-memory pointers of player K, derived at the point of use from the
// layout (a kernel parameter in the constant bank) so they do not stay live
// in registers across the whole persistent loop.
extern __shared__ __align__(16) unsigned char g_smem[];

template <int K>
__device__ __forceinline__ SPtrs sptrs(const SmemPlan& sp) {
    return carve(g_smem, sp.p[K], K == 0);
}

// One DP (thread mode) of a phase in the SMEM engine, fully inlined.
template <int K, int MAXA>
__device__ __forceinline__ void small_item(int kind, const SmemPlan& sp, int j, double w,
                                           const PArgs& a, double pf, double nf) {
    const SPtrs P = sptrs<K>(sp);
    switch (kind) {
        case PH_TD_AVG:
            if (j == 0) P.avg[0] = dadd(dmul(w, P.x[0]), P.avg[0]);
            td_dp<LdS>(P.T, j, P.b, P.x, P.avg, w);
            break;
        case PH_TD_POST: td_dp<LdS>(P.T, j, P.b, P.xpost, nullptr, 0.0); break;
        case PH_CUR: cur_dp<MAXA, LdS>(P.T, j, P.r, P.xpost); break;
        case PH_OBS:
            obs_dp<MAXA, LdS>(P.T, j, P.u, P.r, P.b, P.V, a.post, pf, nf, a.pred == 0, a.nonfinite);
            break;
        case PH_PRED: pred_dp<MAXA, LdS>(P.T, j, P.u, P.r, P.b, P.V, a.plus != 0); break;
    }
}

// A whole top-down pass in one phase (PH_TDC_*): sequence s's x from its
// ancestor chain, x = b_a·(…·(b_0·x[0])), the products td_dp forms level by
// level, in the same order (x[0] = 1.0 is never written).
constexpr int kChainMax = 8;
// PH_RMC: cur_dp's regret matching of DP j (S summed in action order), into bm.
__device__ __forceinline__ void small_rm_item(const SmemPlan& sp, int j) {
    const SPtrs P = sptrs<0>(sp);
    double* bm = reinterpret_cast<double*>(g_smem + sp.p[0].bm);
    const int s0 = P.T.seq_ptr[j], n = P.T.seq_ptr[j + 1] - s0;
    double S = 0.0;
    for (int s = s0; s < s0 + n; ++s) {
        const double v = P.r[s];
        S = dadd(S, v > 0.0 ? v : 0.0);
    }
    for (int s = s0; s < s0 + n; ++s) bm[s] = rm_prob(P.r[s], S, n);
}

template <int K>
__device__ __forceinline__ void small_chain_item(int kind, const SmemPlan& sp, int s, double w) {
    const SPtrs P = sptrs<K>(sp);
    const int* pseq = reinterpret_cast<const int*>(g_smem + sp.p[K].sdp);  // parent sequence, pseq[0] = 0
    const int depth = sp.chain;  // the longest chain (uniform: no divergence)
    int anc[kChainMax];
    int q = s;
#pragma unroll
    for (int i = 0; i < kChainMax; ++i) {  // s, its parent sequence, ... (0 past the root)
        anc[i] = q;
        if (i < depth) q = pseq[q];
    }
    const double* bsrc = kind == PH_TDC_CUR ? reinterpret_cast<const double*>(g_smem + sp.p[K].bm) : P.b;
    double x = 1.0;
#pragma unroll
    for (int i = kChainMax - 1; i >= 0; --i)
        if (i < depth && anc[i] != 0) x = dmul(bsrc[anc[i]], x);
    if (kind == PH_TDC_AVG) {
        P.x[s] = x;
        P.avg[s] = dadd(dmul(w, x), P.avg[s]);
    } else {
        P.xpost[s] = x;
    }
}

// One DP of a top-down phase (thread mode), inline.
template <int K>
__device__ __forceinline__ void small_td_item(int kind, const SmemPlan& sp, int j, double w) {
    const SPtrs P = sptrs<K>(sp);
    if (kind == PH_TD_AVG) {
        if (j == 0) P.avg[0] = dadd(dmul(w, P.x[0]), P.avg[0]);
        td_dp<LdS>(P.T, j, P.b, P.x, P.avg, w);
    } else {
        td_dp<LdS>(P.T, j, P.b, P.xpost, nullptr, 0.0);
    }
}

// One DP of a fat OBS/PRED phase, warp-wide (lane = action).
template <int K>
__device__ __forceinline__ void small_warp_item(int kind, const SmemPlan& sp, int j,
                                                const PArgs& a, double pf, double nf, int lane) {
    const SPtrs P = sptrs<K>(sp);
    if (kind == PH_OBS)
        obs_dp_warp<LdS>(P.T, j, P.u, P.r, P.b, P.V, a.post, pf, nf, a.pred == 0, a.nonfinite,
                         lane);
    else
        pred_dp_warp<LdS>(P.T, j, P.u, P.r, P.b, P.V, a.plus != 0, lane);
}

// Payoff row from the shared-memory copy: the same products and the same
// left-to-right sum as spmv_range (((0 + d0*x0) + d1*x1) + ...), d = the
// value table entry of the non-zero.
__device__ __forceinline__ double spmv_row_smem(const SmemPlan& sp, int ptr, int col, int vid, const double* x,
                                                int row) {
    const int* p = reinterpret_cast<const int*>(g_smem + ptr);
    const unsigned short* c = reinterpret_cast<const unsigned short*>(g_smem + col);
    const unsigned short* v = reinterpret_cast<const unsigned short*>(g_smem + vid);
    const double* tab = reinterpret_cast<const double*>(g_smem + sp.tab);
    double acc = 0.0;
    const int k1 = p[row + 1];
    for (int k = p[row]; k < k1; ++k) acc = dadd(acc, dmul(tab[v[k]], x[c[k]]));
    return acc;
}

template <int MAXA, int THREADS, bool OOL = false>
__global__ void __launch_bounds__(THREADS, 1) k_small(const __grid_constant__ PArgs a,
                                                   const __grid_constant__ SmemPlan sp) {
    const int solve = blockIdx.x;
    Phase* prog = reinterpret_cast<Phase*>(g_smem + sp.prog);
    for (int i = threadIdx.x; i < a.nphase; i += blockDim.x) prog[i] = a.prog[i];
    stage<0>(a, sptrs<0>(sp), solve, true);
    stage<1>(a, sptrs<1>(sp), solve, true);
    if (sp.csr_bytes) {
        const int4* src = reinterpret_cast<const int4*>(a.csr);
        int4* dst = reinterpret_cast<int4*>(g_smem + sp.csr);
        for (int i = threadIdx.x; i < sp.csr_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    if (sp.p[0].sdp) {  // chain phases: each sequence's parent sequence (0 -> 0)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int* spt = reinterpret_cast<const int*>(g_smem + sp.p[k].seq_ptr);
            const int* dpp = reinterpret_cast<const int*>(g_smem + sp.p[k].dp_parent);
            int* pseq = reinterpret_cast<int*>(g_smem + sp.p[k].sdp);
            if (threadIdx.x == 0) pseq[0] = 0;
            for (int j = threadIdx.x; j < a.J[k]; j += blockDim.x)
                for (int s = spt[j]; s < spt[j + 1]; ++s) pseq[s] = dpp[j];
        }
        __syncthreads();
    }
    const int rank = threadIdx.x, size = blockDim.x;
    const int warp = rank >> 5, lane = rank & 31, nwarps = size >> 5;
    long long t_last = clock64();
    for (int it = 0; it < a.n_iter; ++it) {
        const size_t si = (size_t)solve * a.cap + (size_t)(a.t0 + it);
        const double w = a.wsched[si];
        const double pf = a.post == POST_DCFR ? a.pfsched[si] : 1.0;
        const double nf = a.post == POST_DCFR ? a.nfsched[si] : 1.0;
#pragma unroll 1
        for (int p = 0; p < a.nphase; ++p) {
            const Phase ph = prog[p];
            const int total = ph.n1 + ph.n2;
            if (ph.kind == PH_RMC) {  // regret matching of every player-1 DP (no level order)
#pragma unroll 1
                for (int i = rank; i < ph.n1; i += size) small_rm_item(sp, ph.lo1 + i);
            } else if (ph.kind >= PH_TDC_AVG) {  // a whole top-down pass (sequences 1.. of each player)
#pragma unroll 1
                for (int i = rank; i < total; i += size) {
                    if (i < ph.n1) small_chain_item<0>(ph.kind, sp, ph.lo1 + i, w);
                    else small_chain_item<1>(ph.kind, sp, ph.lo2 + (i - ph.n1), w);
                }
                if (ph.kind == PH_TDC_AVG && rank == 0) {  // td_dp's avg[0] update at DP 0
                    const SPtrs P0 = sptrs<0>(sp), P1 = sptrs<1>(sp);
                    if (a.J[0] > 0) P0.avg[0] = dadd(dmul(w, P0.x[0]), P0.avg[0]);
                    if (a.J[1] > 0) P1.avg[0] = dadd(dmul(w, P1.x[0]), P1.avg[0]);
                }
            } else if (ph.kind < PH_SPMV_U) {
                if constexpr (OOL) {  // out of line: one call per player and phase
                    const bool wp = ph.warp1 | ph.warp2;  // fat OBS/PRED level: warps over the DPs
                    if (ph.kind == PH_TD_AVG || ph.kind == PH_TD_POST) {  // short: stay inline
#pragma unroll 1
                        for (int i = rank; i < total; i += size) {
                            if (i < ph.n1) small_td_item<0>(ph.kind, sp, ph.lo1 + i, w);
                            else small_td_item<1>(ph.kind, sp, ph.lo2 + (i - ph.n1), w);
                        }
                        goto phase_done;
                    }
                    const int who = wp ? warp : rank, many = wp ? nwarps : size;
                    if (ph.n1 > 0) {
                        const SPtrs P = sptrs<0>(sp);
                        phase_dps<MAXA, LdS>(ph.kind, P.T, ph.lo1, ph.n1, who, many, P.u, P.r, P.b, P.x, P.xpost,
                                             P.avg, P.V, w, a.post, pf, nf, a.pred, a.plus, a.nonfinite, wp);
                    }
                    if (ph.n2 > 0) {
                        const SPtrs P = sptrs<1>(sp);
                        const int b1 = (who + many - ph.n1 % many) % many;  // continue the combined item order
                        phase_dps<MAXA, LdS>(ph.kind, P.T, ph.lo2, ph.n2, b1, many, P.u, P.r, P.b, P.x, P.xpost,
                                             P.avg, P.V, w, a.post, pf, nf, a.pred, a.plus, a.nonfinite, wp);
                    }
                } else if (ph.warp1 | ph.warp2) {  // fat OBS/PRED level: one warp per DP, lane = action
#pragma unroll 1
                    for (int i = warp; i < total; i += nwarps) {
                        if (i < ph.n1) small_warp_item<0>(ph.kind, sp, ph.lo1 + i, a, pf, nf, lane);
                        else small_warp_item<1>(ph.kind, sp, ph.lo2 + (i - ph.n1), a, pf, nf, lane);
                    }
                } else {
#pragma unroll 1
                    for (int i = rank; i < total; i += size) {
                        if (i < ph.n1) small_item<0, MAXA>(ph.kind, sp, ph.lo1 + i, w, a, pf, nf);
                        else small_item<1, MAXA>(ph.kind, sp, ph.lo2 + (i - ph.n1), w, a, pf, nf);
                    }
                }
            } else {
#pragma unroll 1
                for (int i = rank; i < total; i += size) {
                    const bool first = ph.kind == PH_SPMV_U || (ph.kind == PH_SPMV_BOTH && i < a.Urows);
                    double acc;
                    if (first) {
                        acc = sp.csr_bytes ? spmv_row_smem(sp, sp.uptr, sp.ucol, sp.uvid, sptrs<1>(sp).x, i)
                                           : spmv_row<LdS>(a.Uip, a.Uix, a.Ud, sptrs<1>(sp).x, i);
                        sptrs<0>(sp).u[i] = acc;
                    } else {
                        const SPtrs P0 = sptrs<0>(sp);
                        const int row = ph.kind == PH_SPMV_BOTH ? i - a.Urows : i;
                        const double* x1 = a.alt ? P0.xpost : P0.x;
                        acc = dmul(-1.0, sp.csr_bytes ? spmv_row_smem(sp, sp.tptr, sp.tcol, sp.tvid, x1, row)
                                                      : spmv_row<LdS>(a.Tip, a.Tix, a.Td, x1, row));
                        sptrs<1>(sp).u[row] = acc;
                    }
                    if (!isfinite(acc)) atomicOr(a.nonfinite, 1);
                }
            }
        phase_done:
            if (ph.first_avg && rank == 0) {
                const SPtrs P0 = sptrs<0>(sp), P1 = sptrs<1>(sp);
                if (a.J[0] == 0) P0.avg[0] = dadd(dmul(w, P0.x[0]), P0.avg[0]);
                if (a.J[1] == 0) P1.avg[0] = dadd(dmul(w, P1.x[0]), P1.avg[0]);
            }
            __syncthreads();
            if (a.trace && rank == 0 && blockIdx.x == 0) {
                const long long now = clock64();
                a.trace[p] += now - t_last;
                t_last = now;
            }
        }
    }
    stage<0>(a, sptrs<0>(sp), solve, false);
    stage<1>(a, sptrs<1>(sp), solve, false);
    if (rank == 0 && blockIdx.x == 0) *a.tdev = a.t0 + a.n_iter;
}

// --- host side ---------------------------------------------------------------

// CTA mode: 256 threads, 4 actions in registers; grid mode: 128 threads x
// all SMs, 8 actions in registers (Liar's dice has up to 12-way DPs).
static constexpr auto kCta = k_persistent<PM_CTA, 4, 256>;
static constexpr auto kGrid = k_persistent<PM_GRID, 8, 128>;
// Cluster mode: 16 CTAs (the non-portable maximum) x 256 threads per solve.
static constexpr int kClusterThreads = 256;
static constexpr auto kClu = k_persistent<PM_CLUSTER, 8, kClusterThreads>;
static constexpr int kSmallThreads = 256;
static constexpr auto kSmall2 = k_small<2, kSmallThreads>;
static constexpr auto kSmall3 = k_small<3, kSmallThreads>;
static constexpr auto kSmallO2 = k_small<2, kSmallThreads, true>;
static constexpr auto kSmallO3 = k_small<3, kSmallThreads, true>;
static constexpr int kSmemLimit = 220 * 1024;

// Byte layout of one solve in the SMEM engine; returns the total size.
static int plan_smem(const scfr_handle* h, SmemPlan& sp, bool chain = false) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const int at = (int)off;
        off += (bytes + 15) & ~size_t(15);
        return at;
    };
    for (int k = 0; k < 2; ++k) {
        const Player& P = h->P[k];
        const size_t S = P.S, J = std::max(P.J, 1);
        SmemSide& o = sp.p[k];
        o.r = take(8 * S);
        o.b = take(8 * S);
        o.x = take(8 * S);
        o.xpost = k == 0 ? take(8 * S) : 0;
        o.avg = take(8 * S);
        o.u = take(8 * S);
        o.V = take(8 * J);
        o.child = take(8 * S);
        o.seq_ptr = take(4 * (J + 1));
        o.dp_parent = take(4 * J);
        o.sdp = chain ? take(4 * S) : 0;
        o.bm = chain && k == 0 && predictive(h->variant) && h->mode == SCFR_MODE_ALT ? take(8 * S) : 0;
    }
    sp.prog = take(sizeof(Phase) * h->plan.host_program.size());
    sp.csr_bytes = 0;
    const size_t blob = h->plan.csr_blob.n;
    if (blob && off + blob <= (size_t)kSmemLimit) {  // the payoff rows too, when they fit
        sp.csr = take(blob);
        sp.csr_bytes = (int)blob;
        const int* rel = h->plan.csr_rel;
        sp.uptr = sp.csr + rel[0];
        sp.ucol = sp.csr + rel[1];
        sp.uvid = sp.csr + rel[2];
        sp.tptr = sp.csr + rel[3];
        sp.tcol = sp.csr + rel[4];
        sp.tvid = sp.csr + rel[5];
        sp.tab = sp.csr + rel[6];
    }
    sp.bytes = off > (size_t)INT32_MAX ? INT32_MAX : (int)off;
    return sp.bytes;
}

// The SMEM engine's copy of U and Uᵀ (offsets into the blob set in sp):
// int32 row pointers, uint16 columns, uint16 ids into a table of the
// distinct values (Leduc: 5 520 non-zeros, 12 distinct values; 2 x 26 KB
// instead of 2 x 70 KB).  Empty when a matrix has >= 65 536 columns or the
// values >= 65 536 distinct entries.
static void compact_payoff(scfr_handle* h) {
    PersistentPlan& pl = h->plan;
    const DevCsr* M[2] = {&h->U, &h->UT};
    std::vector<int> ip[2], ix[2];
    std::vector<double> d[2];
    for (int k = 0; k < 2; ++k) {
        if (M[k]->cols >= 65536 || M[k]->nnz >= (1 << 24)) return;
        ip[k].resize(M[k]->rows + 1);
        ix[k].resize(M[k]->nnz);
        d[k].resize(M[k]->nnz);
        CUDA_OK(cudaMemcpyAsync(ip[k].data(), M[k]->indptr.p, ip[k].size() * 4, cudaMemcpyDeviceToHost, h->stream));
        if (M[k]->nnz) {
            CUDA_OK(cudaMemcpyAsync(ix[k].data(), M[k]->indices.p, ix[k].size() * 4, cudaMemcpyDeviceToHost, h->stream));
            CUDA_OK(cudaMemcpyAsync(d[k].data(), M[k]->data.p, d[k].size() * 8, cudaMemcpyDeviceToHost, h->stream));
        }
    }
    CUDA_OK(cudaStreamSynchronize(h->stream));
    std::vector<double> tab;  // distinct values, by bit pattern (-0.0 and 0.0 stay apart)
    std::vector<std::pair<uint64_t, int>> seen;
    std::vector<unsigned short> vid[2];
    for (int k = 0; k < 2; ++k) {
        vid[k].resize(d[k].size());
        for (size_t e = 0; e < d[k].size(); ++e) {
            uint64_t bits;
            std::memcpy(&bits, &d[k][e], 8);
            int id = -1;
            for (const auto& s : seen)
                if (s.first == bits) {
                    id = s.second;
                    break;
                }
            if (id < 0) {
                if (tab.size() >= 4096) return;  // (linear probe: keep the table small)
                id = (int)tab.size();
                tab.push_back(d[k][e]);
                seen.emplace_back(bits, id);
            }
            vid[k][e] = (unsigned short)id;
        }
    }
    std::vector<unsigned char> blob;
    auto put = [&](const void* p, size_t bytes) {
        const int at = (int)blob.size();
        blob.resize((blob.size() + bytes + 15) & ~size_t(15));
        if (bytes) std::memcpy(blob.data() + at, p, bytes);
        return at;
    };
    std::vector<unsigned short> col[2];
    for (int k = 0; k < 2; ++k) col[k].assign(ix[k].begin(), ix[k].end());
    int* rel = pl.csr_rel;
    rel[0] = put(ip[0].data(), ip[0].size() * 4);
    rel[1] = put(col[0].data(), col[0].size() * 2);
    rel[2] = put(vid[0].data(), vid[0].size() * 2);
    rel[3] = put(ip[1].data(), ip[1].size() * 4);
    rel[4] = put(col[1].data(), col[1].size() * 2);
    rel[5] = put(vid[1].data(), vid[1].size() * 2);
    rel[6] = put(tab.data(), tab.size() * 8);
    pl.csr_blob.alloc(blob.size());
    CUDA_OK(copy_async(pl.csr_blob.p, blob.data(), blob.size(), cudaMemcpyHostToDevice, h->stream));
}

// Same rule as the level engine: few DPs, >= 8 child-DP references per DP.
static bool fat_level(const Player& P, int l) {
    static const bool off = [] {  // SCFR_SMALL_NO_WARP=1: thread per DP everywhere (A/B)
        const char* e = std::getenv("SCFR_SMALL_NO_WARP");
        return e && e[0] == '1';
    }();
    if (off) return false;
    return (P.lvl_nj[l] <= 4096 && P.lvl_nc[l] >= 8.0 * P.lvl_nj[l]) ||
           (P.lvl_maxa[l] >= kWideActions && P.lvl_maxa[l] <= 32);
}

static void push_levels(std::vector<Phase>& prog, int kind, const Player* A, const Player* B,
                        bool deep_first) {
    const int LA = A ? A->levels() : 0, LB = B ? B->levels() : 0;
    const int L = std::max(LA, LB);
    for (int k = 0; k < L; ++k) {
        Phase ph{kind, 0, 0, 0, 0, 0};
        const int la = deep_first ? LA - 1 - k : k, lb = deep_first ? LB - 1 - k : k;
        const bool sums = kind == PH_OBS || kind == PH_PRED;
        if (A && la >= 0 && la < LA) {
            ph.lo1 = A->lvl[la];
            ph.n1 = A->lvl[la + 1] - A->lvl[la];
            ph.warp1 = sums && fat_level(*A, la);
        }
        if (B && lb >= 0 && lb < LB) {
            ph.lo2 = B->lvl[lb];
            ph.n2 = B->lvl[lb + 1] - B->lvl[lb];
            ph.warp2 = sums && fat_level(*B, lb);
        }
        prog.push_back(ph);
    }
}

// Longest ancestor chain of a sequence (DP levels above it, inclusive), from
// the host structure of this create.
static int chain_depth(const scfr_handle* h) {
    int worst = 0;
    for (const Player& P : h->P) {
        if (!P.h_seq_ptr || !P.h_dp_parent) return INT32_MAX;
        const std::vector<int>& sp = *P.h_seq_ptr;
        const std::vector<int>& par = *P.h_dp_parent;
        std::vector<int> sdepth(P.S, 0);  // DPs on the chain of each sequence
        for (int j = 0; j < P.J; ++j) {
            const int d = sdepth[par[j]] + 1;  // (parents precede their DPs)
            for (int s = sp[j]; s < sp[j + 1]; ++s) sdepth[s] = d;
            worst = std::max(worst, d);
        }
    }
    return worst;
}

static std::vector<Phase> build_program(const scfr_handle* h, bool chain = false) {
    const Player* A = &h->P[0];
    const Player* Bp = &h->P[1];
    const bool pr = predictive(h->variant);
    std::vector<Phase> prog;
    if (pr) push_levels(prog, PH_PRED, A, Bp, true);
    const size_t first_td = prog.size();
    if (chain)
        prog.push_back(Phase{PH_TDC_AVG, 1, A->S - 1, 1, Bp->S - 1, 0});
    else
        push_levels(prog, PH_TD_AVG, A, Bp, false);
    if (prog.size() == first_td) prog.push_back(Phase{PH_TD_AVG, 0, 0, 0, 0, 0});
    prog[first_td].first_avg = 1;
    if (h->mode == SCFR_MODE_SIM) {
        prog.push_back(Phase{PH_SPMV_BOTH, 0, h->U.rows + h->UT.rows, 0, 0, 0});
        push_levels(prog, PH_OBS, A, Bp, true);
    } else {
        prog.push_back(Phase{PH_SPMV_U, 0, h->U.rows, 0, 0, 0});
        push_levels(prog, PH_OBS, A, nullptr, true);
        if (chain && !pr) {
            prog.push_back(Phase{PH_TDC_POST, 1, A->S - 1, 0, 0, 0});
        } else if (chain) {
            prog.push_back(Phase{PH_RMC, 0, A->J, 0, 0, 0});
            prog.push_back(Phase{PH_TDC_CUR, 1, A->S - 1, 0, 0, 0});
        } else {
            push_levels(prog, pr ? PH_CUR : PH_TD_POST, A, nullptr, false);
        }
        prog.push_back(Phase{PH_SPMV_UT, 0, h->UT.rows, 0, 0, 0});
        push_levels(prog, PH_OBS, nullptr, Bp, true);
    }
    return prog;
}

// Engine choice by size (sequences of both players, per solve): batches of
// small games -> one CTA per solve; one small game -> one CTA; medium ->
// cooperative grid; large (every level fills the GPU) -> level kernels.
int choose_engine(scfr_handle* h) {
    const int64_t S = (int64_t)h->P[0].S + h->P[1].S;
    if (h->B > 1) return S <= 262144 ? SCFR_ENGINE_PERSISTENT : SCFR_ENGINE_LEVELS;
    // The grid-persistent engine measured slower than PDL-chained level
    // kernels on Liar's dice (468 vs 184 µs/iter), so medium games use levels.
    return S <= 8192 ? SCFR_ENGINE_PERSISTENT : SCFR_ENGINE_LEVELS;
}

void prepare_persistent(scfr_handle* h) {
    PersistentPlan& pl = h->plan;
    pl.host_program = build_program(h);
    pl.grid = h->engine == SCFR_ENGINE_PERSISTENT_GRID;
    pl.cluster = h->engine == SCFR_ENGINE_PERSISTENT_CLUSTER;
    pl.threads = pl.grid ? 128 : 256;  // must match kGrid / kCta / kClu
    if (pl.cluster) {
        int want = 16;
        if (const char* e = std::getenv("SCFR_CLUSTER_SIZE")) want = std::max(1, std::min(16, std::atoi(e)));
        CUDA_OK(cudaFuncSetAttribute(kClu, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        for (; want >= 1; want /= 2) {  // largest cluster the device can co-schedule
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(want * h->B);
            cfg.blockDim = dim3(kClusterThreads);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = want;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, kClu, &cfg) == cudaSuccess && nclusters >= 1) break;
            cudaGetLastError();
        }
        if (want < 1) fail(SCFR_ECUDA, "cluster-persistent kernel cannot be scheduled");
        pl.csize = want;
        pl.ctas = want * h->B;
        pl.threads = kClusterThreads;
    } else if (pl.grid) {
        int occ = 0;
        CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kGrid, pl.threads, 0));
        if (occ < 1) fail(SCFR_ECUDA, "persistent kernel cannot be resident");
        int want = h->num_sms;
        const char* env_ctas = std::getenv("SCFR_PERSIST_CTAS");
        if (env_ctas) want = std::max(1, std::atoi(env_ctas));
        pl.ctas = std::min(want, h->num_sms * occ);
    } else {
        pl.ctas = h->B;
        const char* env_small = std::getenv("SCFR_NO_SMEM");
        const char* env_csr = std::getenv("SCFR_NO_SMEM_PAYOFF");  // A/B: payoff rows from global memory
        if (!(env_csr && env_csr[0] == '1')) compact_payoff(h);
        pl.small = plan_smem(h, pl.smem) <= kSmemLimit && !(env_small && env_small[0] == '1');
        // one top-down phase per pass from ancestor chains (SCFR_SMALL_NO_CHAIN=1: per level)
        const char* nch = std::getenv("SCFR_SMALL_NO_CHAIN");
        const int depth = pl.small && !(nch && nch[0] == '1') ? chain_depth(h) : INT32_MAX;
        if (depth <= kChainMax) {
            pl.smem.chain = depth;
            pl.host_program = build_program(h, true);
            if (plan_smem(h, pl.smem, true) <= kSmemLimit) {
                pl.chain = true;
            } else {
                pl.host_program = build_program(h, false);
                plan_smem(h, pl.smem, false);
            }
        }
        if (pl.small) {
            pl.threads = kSmallThreads;
            // OBS / PRED / CUR phases out of line with 3 actions in registers
            // (Leduc's DPs have 2 or 3: no divergent generic path), top-down
            // phases inline.  SCFR_SMALL_OOL=0 / SCFR_SMALL_MAXA=2: the fully
            // inlined kernel / 2 actions in registers (A/B).
            // Games of at most 2 actions (Kuhn) keep the inlined kernel: the
            // calls cost more than the divergence they remove (7.0 vs 6.1 us).
            const bool two = std::max(h->P[0].max_actions, h->P[1].max_actions) <= 2;
            int maxa = two ? 2 : 3;
            if (const char* e = std::getenv("SCFR_SMALL_MAXA")) maxa = std::atoi(e) == 2 ? 2 : 3;
            const char* ool = std::getenv("SCFR_SMALL_OOL");
            if (ool ? ool[0] != '0' : !two)
                pl.small_kern = maxa == 3 ? (const void*)kSmallO3 : (const void*)kSmallO2;
            else
                pl.small_kern = maxa == 3 ? (const void*)kSmall3 : (const void*)kSmall2;
            CUDA_OK(cudaFuncSetAttribute(pl.small_kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         pl.smem.bytes));
        }
    }
    pl.program.alloc(pl.host_program.size());
    CUDA_OK(copy_async(pl.program.p, pl.host_program.data(), pl.host_program.size() * sizeof(Phase),
                       cudaMemcpyHostToDevice, h->stream));
    pl.barrier.alloc(2);
    pl.barrier.zero(h->stream);
    CUDA_OK(cudaStreamSynchronize(h->stream));
}

int64_t launch_persistent(scfr_handle* h, int64_t n) {
    PersistentPlan& pl = h->plan;
    PArgs a;
    for (int k = 0; k < 2; ++k) {
        Player& P = h->P[k];
        a.T[k] = P.tree();
        a.r[k] = P.r.p;
        a.b[k] = P.b.p;
        a.x[k] = P.x.p;
        a.xpost[k] = P.xpost.p;
        a.avg[k] = P.avg.p;
        a.u[k] = P.u.p;
        a.V[k] = P.V.p;
        a.S[k] = P.S;
        a.J[k] = P.J;
    }
    a.Uip = h->U.indptr.p;
    a.Uix = h->U.indices.p;
    a.Ud = h->U.data.p;
    a.Urows = h->U.rows;
    a.Tip = h->UT.indptr.p;
    a.Tix = h->UT.indices.p;
    a.Td = h->UT.data.p;
    a.Trows = h->UT.rows;
    a.wsched = h->wsched.p;
    a.pfsched = h->pfsched.p;
    a.nfsched = h->nfsched.p;
    a.cap = h->cap;
    a.prog = pl.program.p;
    a.nphase = (int)pl.host_program.size();
    a.post = post_of(h->variant);
    a.pred = predictive(h->variant) ? 1 : 0;
    a.plus = h->variant == SCFR_PCFR_PLUS ? 1 : 0;
    a.alt = h->mode == SCFR_MODE_ALT ? 1 : 0;
    a.nonfinite = h->nonfinite.p;
    a.tdev = h->tdev.p;
    a.barrier = pl.barrier.p;
    a.trace = nullptr;
    a.csr = pl.csr_blob.p;
    const char* tr = std::getenv("SCFR_PHASE_TRACE");
    DevBuf<long long> trace_buf;
    if (tr && tr[0] == '1' && pl.small) {
        trace_buf.alloc(pl.host_program.size());
        trace_buf.zero(h->stream);
        a.trace = trace_buf.p;
    }
    int64_t launches = 0;
    // Chunk long requests so one launch stays well under the watchdog-free
    // but still bounded duration, and the schedule index fits in int.
    const int64_t chunk = 1 << 16;
    for (int64_t done = 0; done < n; done += chunk) {
        a.t0 = h->t + done;
        a.n_iter = (int)std::min<int64_t>(chunk, n - done);
        if (pl.cluster) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(pl.ctas);
            cfg.blockDim = dim3(pl.threads);
            cfg.stream = h->stream;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = pl.csize;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            CUDA_OK(cudaLaunchKernelEx(&cfg, kClu, a));
        } else if (pl.grid) {
            void* args[] = {&a};
            CUDA_OK(cudaLaunchCooperativeKernel((const void*)kGrid, dim3(pl.ctas),
                                                dim3(pl.threads), args, 0, h->stream));
        } else {
            if (pl.small) {
                void* args[] = {&a, &pl.smem};
                CUDA_OK(cudaLaunchKernel(pl.small_kern, dim3(pl.ctas), dim3(pl.threads), args, pl.smem.bytes,
                                         h->stream));
            } else {
                kCta<<<pl.ctas, pl.threads, 0, h->stream>>>(a);
            }
            CUDA_OK(cudaGetLastError());
        }
        ++launches;
    }
    if (a.trace) {  // debug: average cycles per phase per iteration, on stderr
        std::vector<long long> cyc(pl.host_program.size());
        CUDA_OK(cudaMemcpyAsync(cyc.data(), a.trace, cyc.size() * sizeof(long long),
                                cudaMemcpyDeviceToHost, h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));
        static const char* names[] = {"td_avg", "td_post", "cur", "obs", "pred", "spmv_u", "spmv_ut", "spmv_both",
                                      "tdc_avg", "tdc_post", "rmc", "tdc_cur"};
        for (size_t p = 0; p < cyc.size(); ++p) {
            const Phase& ph = pl.host_program[p];
            std::fprintf(stderr, "[phase %2zu] %-9s n1=%6d n2=%6d  %9.1f cycles/iter\n", p,
                         names[ph.kind], ph.n1, ph.n2, (double)cyc[p] / (double)n);
        }
    }
    return launches;
}

double persistent_bytes_per_iter(const scfr_handle* h) {
    // Same algorithmic-byte model as the level engine (solver.cu LevelBytes).
    double total = 0.0;
    for (const Phase& ph : h->plan.host_program) {
        for (int k = 0; k < 2; ++k) {
            const int lo = k == 0 ? ph.lo1 : ph.lo2, n = k == 0 ? ph.n1 : ph.n2;
            if (n == 0 || ph.kind >= PH_SPMV_U) continue;
            const Player& P = h->P[k];
            int l = (int)(std::upper_bound(P.lvl.begin(), P.lvl.end(), lo) - P.lvl.begin()) - 1;
            if (l < 0 || l >= P.levels()) continue;
            const double ns = P.lvl_ns[l], nj = P.lvl_nj[l], nc = P.lvl_nc[l];
            switch (ph.kind) {
                case PH_TD_AVG: total += 32 * ns + 16 * nj; break;
                case PH_TD_POST:
                case PH_CUR: total += 16 * ns + 16 * nj; break;
                case PH_OBS: total += (predictive(h->variant) ? 40 : 48) * ns + 12 * nj + 8 * nc; break;
                case PH_PRED: total += 40 * ns + 12 * nj + 8 * nc; break;
            }
        }
        if (ph.kind >= PH_SPMV_U) {
            const DevCsr* ms[2] = {&h->U, &h->UT};
            for (int k = 0; k < 2; ++k) {
                if ((ph.kind == PH_SPMV_U && k == 1) || (ph.kind == PH_SPMV_UT && k == 0)) continue;
                const DevCsr& M = *ms[k];
                total += 4.0 * (M.rows + 1) + 12.0 * M.nnz + 8.0 * M.cols + 8.0 * M.rows;
            }
        }
    }
    return total * h->B;
}

}  // namespace scfr
