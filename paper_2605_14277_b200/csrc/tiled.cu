// Tile engine: one kernel launch per pass of a CFR iteration.
//
// The level engine launches one kernel per DP level and pass.  On
// Goofspiel-5 that is 26 launches per iteration.  The small top levels are
// dependent-load chains, and every level sends its V through HBM to the next
// launch (profiles/r01/SUMMARY.md).  Here a pass is ONE launch:
//
//   * A split level `ls` cuts each player's decision process into a small
//     top (levels < ls, unchanged ids) and a forest below.  Its roots are
//     the DPs whose parent sequence lies in the top.
//   * Roots are grouped into tiles.  Siblings never straddle a tile.  A tile
//     owns its roots' whole subtrees.  DPs and sequences below the split are
//     renumbered tile-major.  Within a tile they are ordered by level, then
//     roots first, then original order.  So every tile is one contiguous
//     block of DPs and of sequences, and every (tile, level) block is a
//     contiguous range with an exact affine shape where one exists.
//   * Bottom-up passes (OBS, PRED): a CTA walks its tile's levels deep to
//     shallow and keeps V in shared memory.  Only the roots' V goes to HBM.
//     The CTA that completes a player's last tile (a ticket) then runs the
//     top levels.  Those are few DPs, warp-per-DP where fat.
//   * Top-down passes (TD+avg, TD, CUR): every CTA recomputes the top's x
//     into shared memory, a handful of DPs.  The first tile's CTA also
//     writes them out.  Then the CTA walks its tile shallow to deep, and x
//     flows parent to child through shared memory.
//
// Per-DP arithmetic is the same code as the other engines (kernels.cuh, or
// the same intrinsic sequence for the top-down products), so iterates are
// bit-identical to the reference.  The payoff rows are permuted into the
// tile numbering, keeping their CSR nnz order.  Reads scatter state back to
// the reference's order (orig_order).

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "runtime.h"

namespace scfr {

__global__ void k_derive_child(int J, const int* __restrict__ dp_parent, int2* __restrict__ child);
template <class R>
__global__ void k_derive_uniform(int J, int S, int B, const int* __restrict__ seq_ptr,
                                 R* __restrict__ b);

constexpr int kTileThreads = 256;
constexpr int kTileMinBlocks = 3;  // <= 80 registers; shared memory allows ~3 CTAs per SM anyway
constexpr int kMaxTop = 12;          // top levels carried in the kernel parameters
constexpr int kMaxStop = 4096;       // top sequences (recomputed per CTA in shared memory)
constexpr int kMaxEntries = 12288;   // DPs + sequences of one tile (≤ 96 KB of fp64)

struct TileTask {
    const int* seq_ptr;      // tile numbering
    const int* dp_parent;
    const int2* child;
    const int* top_seq_ptr;  // original numbering (the top and the roots' V)
    const int* top_dp_parent;
    const int2* top_child;
    const int* dperm;        // tile DP id -> original DP id (roots publish V there)
    const int* off;          // [ntiles][nlev+1]
    const TileShape* shp;    // [ntiles][nlev]
    int ntiles, nlev, ls, Stop;
    int top_lvl[kMaxTop + 1];
    TileShape top_shp[kMaxTop];
    unsigned top_warp;
    int S, J;                // per-solve strides
    const double* u;         // utility (OBS, fused: written) / prediction (PRED)
    double* r;
    double* b;
    double* x;               // TD output (x or xpost)
    double* avg;
    double* V;               // global V: roots and top DPs only
    FuseU fu;
    int fu_sx;
    unsigned* ticket;        // [B]
    int vwin;                // shared-memory V window (doubles) of the launch
    int staged;              // stage affine blocks through shared memory
};

__device__ __forceinline__ DevTree tree_of(const TileTask& t, const TileShape& sh, bool top = false) {
    DevTree T = top ? DevTree{t.top_seq_ptr, t.top_dp_parent, t.top_child}
                    : DevTree{t.seq_ptr, t.dp_parent, t.child};
    T.j_lo = sh.j_lo;
    T.s_lo = sh.s_lo;
    T.un = sh.un;
    T.cn = sh.cn;
    T.c_lo = sh.c_lo;
    T.pc = sh.pc;
    T.p_lo = sh.p_lo;
    return T;
}

// Generic pointer p - base elements (shared-memory window indexed by global id).
__device__ __forceinline__ double* shifted(double* p, int base) {
    return reinterpret_cast<double*>(reinterpret_cast<uintptr_t>(p) - (uintptr_t)base * sizeof(double));
}

enum : int { TK_OBS = 0, TK_PRED, TK_TD_AVG, TK_TD, TK_CUR };

// ---------------------------------------------------------------------------
// Bottom-up: OBS (counterfactual values, regret update, [RM]) or PRED.

// Staging: every thread keeps kStageDepth independent loads in flight, so a
// block's inputs arrive in about one HBM round trip instead of one per DP.
constexpr int kStageDepth = 4;
constexpr int kUCH = 1024;  // sequences staged per chunk
constexpr int kPCH = 1024;  // payoff nnz per product chunk

template <class T>
__device__ __forceinline__ void stage(T* dst, const T* __restrict__ src, int n) {
    for (int i = threadIdx.x; i < n; i += kStageDepth * blockDim.x) {
        T v[kStageDepth];
#pragma unroll
        for (int q = 0; q < kStageDepth; ++q) {
            const int k = i + q * (int)blockDim.x;
            if (k < n) v[q] = src[k];
        }
#pragma unroll
        for (int q = 0; q < kStageDepth; ++q) {
            const int k = i + q * (int)blockDim.x;
            if (k < n) dst[k] = v[q];
        }
    }
}

// Shared-memory staging buffers of the up pass (after the tile's V window).
struct UpStage {
    double* u;   // [kUCH] utility (fused rows) / prediction
    double* b;   // [kUCH]
    double* r;   // [kUCH]
    double* p;   // [kPCH] payoff products
    int* ip;     // [kUCH + 1] row pointers
};

// u[s0 .. s0+ns) = (±) rows of the payoff matrix applied to x, computed by
// the whole CTA: row pointers staged, products d*x[c] gathered with several
// loads in flight per thread, then each row summed sequentially in CSR
// order from 0.0 (pkg/kernels.py:149-154; the same roundings as spmv_row).
__device__ __forceinline__ void fused_rows(const FuseU& f, int s0, int ns, const UpStage& st,
                                           double* __restrict__ u_out, int* nonfinite) {
    stage(st.ip, f.ip + s0, ns + 1);
    for (int i = threadIdx.x; i < ns; i += blockDim.x) st.u[i] = 0.0;
    __syncthreads();
    const int k0 = st.ip[0], k1 = st.ip[ns];
    for (int kb = k0; kb < k1; kb += kPCH) {
        const int ke = min(k1, kb + kPCH);
        for (int i = kb + (int)threadIdx.x; i < ke; i += kStageDepth * blockDim.x) {
            int c[kStageDepth];
            double d[kStageDepth], xv[kStageDepth];
#pragma unroll
            for (int q = 0; q < kStageDepth; ++q) {
                const int k = i + q * (int)blockDim.x;
                if (k < ke) {
                    c[q] = __ldg(f.ix + k);
                    d[q] = __ldg(f.d + k);
                }
            }
#pragma unroll
            for (int q = 0; q < kStageDepth; ++q)
                if (i + q * (int)blockDim.x < ke) xv[q] = f.x[c[q]];
#pragma unroll
            for (int q = 0; q < kStageDepth; ++q) {
                const int k = i + q * (int)blockDim.x;
                if (k < ke) st.p[k - kb] = dmul(d[q], xv[q]);
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < ns; i += blockDim.x) {
            const int a = max(st.ip[i], kb), e = min(st.ip[i + 1], ke);
            if (a < e) {
                double acc = st.u[i];
                for (int k = a; k < e; ++k) acc = dadd(acc, st.p[k - kb]);
                st.u[i] = acc;
            }
        }
        __syncthreads();
    }
    bool bad = false;
    for (int i = threadIdx.x; i < ns; i += blockDim.x) {
        double v = st.u[i];
        if (f.neg) v = dmul(-1.0, v);
        bad |= !isfinite(v);
        st.u[i] = v;
        u_out[s0 + i] = v;
    }
    if (bad) atomicOr(nonfinite, 1);
}

// One affine (tile, level) block, chunk by chunk: stage u / b / r into
// shared memory, run the per-DP code on the staged copies (V lives in
// shared memory too), write r / b back with coalesced stores.
template <int KIND, int MAXA>
__device__ __forceinline__ void up_block_staged(const TileTask& t, const DevTree& T, const TileShape& sh,
                                                int lo, int hi, double* Vs, double* Vg,
                                                const KParams& kp, double pf, double nf,
                                                const FuseU& fu, const UpStage& st, size_t so) {
    const int un = sh.un;
    const bool single = un == 1;
    const bool write_b = KIND == TK_PRED || kp.do_rm != 0;
    const int CH = max(1, kUCH / un);
    for (int c0 = lo; c0 < hi; c0 += CH) {
        const int c1 = min(hi, c0 + CH);
        const int s0 = sh.s_lo + (c0 - lo) * un, ns = (c1 - c0) * un;
        if (!single) {
            stage(st.b, t.b + so + s0, ns);
            stage(st.r, t.r + so + s0, ns);
        }
        if (KIND == TK_OBS && fu.ip) fused_rows(fu, s0, ns, st, const_cast<double*>(t.u) + so, kp.nonfinite);
        else stage(st.u, t.u + so + s0, ns);
        __syncthreads();
        double* us = shifted(st.u, s0);
        double* bs = shifted(st.b, s0);
        double* rs = shifted(st.r, s0);
        for (int j = c0 + (int)threadIdx.x; j < c1; j += blockDim.x) {
            if constexpr (KIND == TK_OBS)
                obs_dp<MAXA, LdL1>(T, j, us, rs, bs, Vs, kp.post, pf, nf, kp.do_rm != 0, kp.nonfinite);
            else
                pred_dp<MAXA, LdL1>(T, j, us, rs, bs, Vs, kp.plus != 0);
            if (j - lo < sh.nroot) Vg[t.dperm[j]] = Vs[j];  // a root: the top pass reads it
        }
        __syncthreads();
        if (!single) {
            for (int i = threadIdx.x; i < ns; i += blockDim.x) {
                if (KIND == TK_OBS) t.r[so + s0 + i] = st.r[i];
                if (write_b) t.b[so + s0 + i] = st.b[i];
            }
            __syncthreads();
        }
    }
}

template <int KIND, int MAXA>
__device__ __forceinline__ void up_tile(const TileTask& t, int tile, const KParams& kp, double* sm,
                                        const UpStage& st, double pf, double nf, const FuseU& fu) {
    const size_t so = (size_t)blockIdx.y * t.S;
    double* Vg = t.V + (size_t)blockIdx.y * t.J;
    const int* o = t.off + (size_t)tile * (t.nlev + 1);
    double* Vs = shifted(sm, o[0]);
    for (int k = t.nlev - 1; k >= 0; --k) {
        const int lo = o[k], hi = o[k + 1];
        if (lo == hi) continue;  // CTA-uniform
        const TileShape sh = t.shp[(size_t)tile * t.nlev + k];
        const DevTree T = tree_of(t, sh);
        if (sh.un > 0 && t.staged) {
            up_block_staged<KIND, MAXA>(t, T, sh, lo, hi, Vs, Vg, kp, pf, nf, fu, st, so);
            continue;
        }
        for (int j = lo + (int)threadIdx.x; j < hi; j += blockDim.x) {
            if constexpr (KIND == TK_OBS)
                obs_dp<MAXA, LdL1>(T, j, t.u + so, t.r + so, t.b + so, Vs, kp.post, pf, nf,
                                   kp.do_rm != 0, kp.nonfinite, fu);
            else
                pred_dp<MAXA, LdL1>(T, j, t.u + so, t.r + so, t.b + so, Vs, kp.plus != 0);
            if (j - lo < sh.nroot) Vg[t.dperm[j]] = Vs[j];  // a root: the top pass reads it
        }
        __syncthreads();
    }
}

// The top levels, deep to shallow, by the CTA that completed the player's
// last tile.  The top runs in the ORIGINAL numbering (its ids are unchanged
// and its child ranges reach the roots, which published V at their original
// ids), so sibling roots may sit in different tiles.  V of the roots comes
// from other CTAs: L2 loads.
template <int KIND>
__device__ __noinline__ void up_top(const TileTask& t, const KParams& kp, double pf, double nf,
                                    const FuseU& fu) {
    const size_t so = (size_t)blockIdx.y * t.S;
    double* Vg = t.V + (size_t)blockIdx.y * t.J;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    if (KIND == TK_OBS && fu.ip && threadIdx.x == 0) {  // row 0: u[0] (the next prediction)
        bool bad = false;
        fused_u<LdL2s>(fu, const_cast<double*>(t.u) + so, 0, bad);
        if (bad) atomicOr(kp.nonfinite, 1);
    }
    for (int l = t.ls - 1; l >= 0; --l) {
        const int lo = t.top_lvl[l], hi = t.top_lvl[l + 1];
        const DevTree T = tree_of(t, t.top_shp[l], true);
        if (t.top_warp >> l & 1) {
            for (int j = lo + warp; j < hi; j += nwarps) {
                if constexpr (KIND == TK_OBS)
                    obs_dp_warp<LdL2s>(T, j, t.u + so, t.r + so, t.b + so, Vg, kp.post, pf, nf,
                                      kp.do_rm != 0, kp.nonfinite, lane, fu);
                else
                    pred_dp_warp<LdL2s>(T, j, t.u + so, t.r + so, t.b + so, Vg, kp.plus != 0, lane);
            }
        } else {
            for (int j = lo + (int)threadIdx.x; j < hi; j += blockDim.x) {
                if constexpr (KIND == TK_OBS)
                    obs_dp<4, LdL2s>(T, j, t.u + so, t.r + so, t.b + so, Vg, kp.post, pf, nf,
                                    kp.do_rm != 0, kp.nonfinite, fu);
                else
                    pred_dp<4, LdL2s>(T, j, t.u + so, t.r + so, t.b + so, Vg, kp.plus != 0);
            }
        }
        __syncthreads();
    }
}

template <int KIND, int MAXA>
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks) k_tile_up(const __grid_constant__ TileTask t0,
                                                          const __grid_constant__ TileTask t1,
                                                          const __grid_constant__ KParams kp) {
    pdl_launch_dependents();
    pdl_wait();
    extern __shared__ double sm[];
    __shared__ int s_last;
    UpStage st;
    {
        double* q = sm + t0.vwin;  // staging after the V window (vwin: largest tile's DPs)
        st.u = q;
        st.b = q + kUCH;
        st.r = q + 2 * kUCH;
        st.p = q + 3 * kUCH;
        st.ip = reinterpret_cast<int*>(q + 3 * kUCH + kPCH);
    }
    double pf = 1.0, nf = 1.0;
    if (KIND == TK_OBS && kp.post == POST_DCFR) {
        const size_t k = (size_t)blockIdx.y * kp.cap + *kp.tdev;
        pf = kp.pfsched[k];
        nf = kp.nfsched[k];
    }
    const int total = t0.ntiles + t1.ntiles;
    for (int g = blockIdx.x; g < total; g += gridDim.x) {
        const bool second = g >= t0.ntiles;
        const TileTask& t = second ? t1 : t0;
        FuseU fu = t.fu;
        if (fu.ip) fu.x += (size_t)blockIdx.y * t.fu_sx;
        up_tile<KIND, MAXA>(t, second ? g - t0.ntiles : g, kp, sm, st, pf, nf, fu);
        __threadfence();  // every thread publishes its root V / r / b / u ...
        __syncthreads();
        if (threadIdx.x == 0) {  // ... before the ticket
            s_last = atomicAdd(t.ticket + blockIdx.y, 1u) == (unsigned)t.ntiles - 1u;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            up_top<KIND>(t, kp, pf, nf, fu);
            if (threadIdx.x == 0) t.ticket[blockIdx.y] = 0u;  // re-armed for the next launch
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Top-down: x[(j,a)] = b[(j,a)] * x[parent(j)] (+ avg = w*x + avg), or CUR
// (regret matching of r on the fly).  Same intrinsic sequence as td_dp /
// cur_dp in kernels.cuh; x of parents comes from shared memory: the top's
// (xs, indexed by id) or the tile's (xt, indexed by id - tile's first seq).

template <int KIND, int MAXA>
__device__ __forceinline__ void down_dp(const DevTree& T, int j, double xp,
                                        const double* __restrict__ bsrc, double* __restrict__ x,
                                        double* __restrict__ avg, double w, double* xt, bool keep) {
    int s0, n;
    dp_range<LdL1>(T, j, s0, n);
    if (T.un == 1) {  // single-action: b == 1.0 and r == +0.0 (kernels.cuh single_action_note)
        const double xa = dmul(1.0, xp);
        x[s0] = xa;
        if (KIND == TK_TD_AVG) avg[s0] = dadd(dmul(w, xa), avg[s0]);
        if (keep) xt[s0] = xa;
        return;
    }
    if constexpr (KIND == TK_CUR) {
        double S = 0.0;
        if (n <= MAXA) {
            double rr[MAXA];
#pragma unroll
            for (int a = 0; a < MAXA; ++a)
                if (a < n) {
                    rr[a] = bsrc[s0 + a];
                    S = dadd(S, rr[a] > 0.0 ? rr[a] : 0.0);
                }
#pragma unroll
            for (int a = 0; a < MAXA; ++a)
                if (a < n) {
                    const double xa = dmul(rm_prob(rr[a], S, n), xp);
                    x[s0 + a] = xa;
                    if (keep) xt[s0 + a] = xa;
                }
        } else {
            for (int s = s0; s < s0 + n; ++s) {
                const double v = bsrc[s];
                S = dadd(S, v > 0.0 ? v : 0.0);
            }
            for (int s = s0; s < s0 + n; ++s) {
                const double xa = dmul(rm_prob(bsrc[s], S, n), xp);
                x[s] = xa;
                if (keep) xt[s] = xa;
            }
        }
    } else {
        for (int s = s0; s < s0 + n; ++s) {
            const double xa = dmul(bsrc[s], xp);
            x[s] = xa;
            if (KIND == TK_TD_AVG) avg[s] = dadd(dmul(w, xa), avg[s]);
            if (keep) xt[s] = xa;
        }
    }
}

// One affine (tile, level) block of a top-down pass, chunk by chunk: b (or
// r) and avg staged into shared memory, parents' x from shared memory, avg
// written back with coalesced stores.
template <int KIND, int MAXA>
__device__ __forceinline__ void down_block_staged(const DevTree& T, const TileShape& sh, int lo, int hi,
                                                  const double* xs, double* xt, int Stop,
                                                  const double* __restrict__ bsrc, double* __restrict__ x,
                                                  double* __restrict__ avg, double w, bool keep,
                                                  double* sb, double* sa) {
    const int un = sh.un;
    const bool single = un == 1;
    const int CH = max(1, kUCH / un);
    for (int c0 = lo; c0 < hi; c0 += CH) {
        const int c1 = min(hi, c0 + CH);
        const int s0 = sh.s_lo + (c0 - lo) * un, ns = (c1 - c0) * un;
        if (!single) stage(sb, bsrc + s0, ns);
        if (KIND == TK_TD_AVG) stage(sa, avg + s0, ns);
        __syncthreads();
        double* bs = shifted(sb, s0);
        double* as = shifted(sa, s0);
        for (int j = c0 + (int)threadIdx.x; j < c1; j += blockDim.x) {
            const int ps = parent_of<LdL1>(T, j);
            const double xp = ps < Stop ? xs[ps] : xt[ps];
            down_dp<KIND, MAXA>(T, j, xp, bs, x, as, w, xt, keep);
        }
        __syncthreads();
        if (KIND == TK_TD_AVG) {
            for (int i = threadIdx.x; i < ns; i += blockDim.x) avg[s0 + i] = sa[i];
            __syncthreads();
        }
    }
}

template <int KIND, int MAXA>
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks) k_tile_down(const __grid_constant__ TileTask t0,
                                                            const __grid_constant__ TileTask t1,
                                                            const __grid_constant__ KParams kp) {
    pdl_launch_dependents();
    pdl_wait();
    extern __shared__ double sm[];
    const double w = KIND == TK_TD_AVG ? kp.wsched[(size_t)blockIdx.y * kp.cap + *kp.tdev] : 0.0;
    const int total = t0.ntiles + t1.ntiles;
    for (int g = blockIdx.x; g < total; g += gridDim.x) {
        const bool second = g >= t0.ntiles;
        const TileTask& t = second ? t1 : t0;
        const int tile = second ? g - t0.ntiles : g;
        const size_t so = (size_t)blockIdx.y * t.S;
        const double* bsrc = (KIND == TK_CUR ? t.r : t.b) + so;
        double* x = t.x + so;
        double* avg = t.avg + so;
        const bool writer = tile == 0;  // the first tile's CTA also writes the top
        double* xs = sm;                // [Stop]
        double* xt0 = sm + t.Stop;      // tile sequences
        // top, shallow -> deep (tiny: recomputed by every CTA)
        if (threadIdx.x == 0) {
            xs[0] = x[0];
            if (KIND == TK_TD_AVG && writer) avg[0] = dadd(dmul(w, x[0]), avg[0]);
        }
        __syncthreads();
        for (int l = 0; l < t.ls; ++l) {
            const int lo = t.top_lvl[l], hi = t.top_lvl[l + 1];
            const DevTree T = tree_of(t, t.top_shp[l], true);
            for (int j = lo + (int)threadIdx.x; j < hi; j += blockDim.x) {
                const double xp = xs[parent_of<LdL1>(T, j)];
                if (writer)
                    down_dp<KIND, MAXA>(T, j, xp, bsrc, x, avg, w, xs, true);
                else
                    down_dp<KIND == TK_TD_AVG ? TK_TD : KIND, MAXA>(T, j, xp, bsrc, xs, nullptr, 0.0,
                                                                  xs, false);
            }
            __syncthreads();
        }
        // the tile, shallow -> deep
        const int* o = t.off + (size_t)tile * (t.nlev + 1);
        const int sbase = t.shp[(size_t)tile * t.nlev].s_lo;
        double* xt = shifted(xt0, sbase);
        for (int k = 0; k < t.nlev; ++k) {
            const int lo = o[k], hi = o[k + 1];
            if (lo == hi) continue;
            const TileShape sh = t.shp[(size_t)tile * t.nlev + k];
            const DevTree T = tree_of(t, sh);
            const bool keep = k + 1 < t.nlev;  // the deepest level has no children
            if (sh.un > 0 && t.staged) {
                down_block_staged<KIND, MAXA>(T, sh, lo, hi, xs, xt, t.Stop, bsrc, x, avg, w, keep,
                                              sm + t.vwin, sm + t.vwin + kUCH);
                continue;
            }
            for (int j = lo + (int)threadIdx.x; j < hi; j += blockDim.x) {
                const int ps = parent_of<LdL1>(T, j);
                const double xp = ps < t.Stop ? xs[ps] : xt[ps];
                down_dp<KIND, MAXA>(T, j, xp, bsrc, x, avg, w, xt, keep);
            }
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// Host: planning.

// Exact affine shape of DPs [j0, j1) in the given numbering (cf. the level
// engine's detection in upload_player).
static TileShape detect_shape(const std::vector<int>& sp, const std::vector<int>& par,
                              const std::vector<int>& cfirst, const std::vector<int>& ccnt,
                              int j0, int j1) {
    TileShape sh{};
    sh.j_lo = j0;
    sh.s_lo = sp[j0];
    sh.cn = -1;
    if (j1 <= j0) return sh;
    const int n0 = sp[j0 + 1] - sp[j0];
    bool uni = true;
    for (int j = j0; j < j1 && uni; ++j) uni = sp[j + 1] - sp[j] == n0;
    sh.un = uni ? n0 : 0;
    const int s0 = sp[j0], s1 = sp[j1];
    const int c0 = ccnt[s0];
    bool aff = true;
    for (int q = s0; q < s1 && aff; ++q)
        aff = ccnt[q] == c0 && (c0 == 0 || cfirst[q] == cfirst[s0] + (q - s0) * c0);
    sh.cn = aff ? c0 : -1;
    sh.c_lo = aff && c0 > 0 ? cfirst[s0] : 0;
    int pc = 1;
    while (j0 + pc < j1 && par[j0 + pc] == par[j0]) ++pc;
    bool pr = true;
    for (int j = j0; j < j1 && pr; ++j) pr = par[j] == par[j0] + (j - j0) / pc;
    sh.pc = pr ? pc : 0;
    sh.p_lo = par[j0];
    return sh;
}

// Renumbering of one player: perm (device DP -> original DP) and sperm
// (device sequence -> original sequence), plus the tile tables.
struct PlayerPlan {
    std::vector<int> perm, sperm, sinv;
    std::vector<int> sp, par;  // device numbering
};

static bool plan_player(const scfr_handle* h, const Player& P, TilePlayer& tp, PlayerPlan& pp) {
    const int J = P.J, S = P.S, L = P.levels();
    if (J == 0 || L < 2) return false;
    if (!P.h_seq_ptr || !P.h_dp_parent) return false;
    const std::vector<int>& sp = *P.h_seq_ptr;
    const std::vector<int>& par = *P.h_dp_parent;
    std::vector<int> seq_dp(S, -1), lev(J);
    for (int j = 0; j < J; ++j)
        for (int s = sp[j]; s < sp[j + 1]; ++s) seq_dp[s] = j;
    for (int l = 0; l < L; ++l)
        for (int j = P.lvl[l]; j < P.lvl[l + 1]; ++j) lev[j] = l;
    // subtree sizes (DPs + sequences), children folded into their parent DP
    std::vector<int64_t> sub(J, 0);
    for (int j = J - 1; j >= 0; --j) {
        sub[j] += 1 + (sp[j + 1] - sp[j]);
        if (par[j] != 0) sub[seq_dp[par[j]]] += sub[j];
    }
    auto is_root = [&](int j, int Jtop) { return par[j] == 0 || seq_dp[par[j]] < Jtop; };
    // split level: the smallest one whose roots fit a tile and give >= 2
    // tiles per SM; else the feasible one with the most roots
    int best = -1;
    int64_t best_roots = 0;
    for (int ls = 1; ls < L && ls <= kMaxTop; ++ls) {
        const int Jtop = P.lvl[ls];
        if (sp[Jtop] > kMaxStop || Jtop > 8192) break;
        int64_t roots = 0, maxsub = 0;
        for (int j = Jtop; j < J; ++j)
            if (is_root(j, Jtop)) {
                ++roots;
                maxsub = std::max(maxsub, sub[j]);
            }
        if (maxsub > kMaxEntries) continue;
        if (roots >= 2 * h->num_sms) {
            best = ls;
            break;
        }
        if (roots > best_roots) {
            best_roots = roots;
            best = ls;
        }
    }
    if (best < 0) return false;
    const int ls = best, Jtop = P.lvl[ls];
    tp.ls = ls;
    tp.Jtop = Jtop;
    tp.Stop = sp[Jtop];
    tp.nlev = L - ls;
    // group roots into tiles (siblings together), ~2 tiles per SM or fewer if they are big
    int64_t forest = 0;
    for (int j = Jtop; j < J; ++j)
        if (is_root(j, Jtop)) forest += sub[j];
    const int64_t target = std::min<int64_t>(kMaxEntries, std::max<int64_t>(1, forest / (2 * h->num_sms)));
    std::vector<int> tile_of(J, -1);
    int ntiles = 0;
    int64_t acc = 0;
    for (int j = Jtop; j < J; ++j) {
        if (is_root(j, Jtop)) {
            if (ntiles == 0 || acc + sub[j] > target) {
                ++ntiles;
                acc = 0;
            }
            acc += sub[j];
            tile_of[j] = ntiles - 1;
        } else {
            tile_of[j] = tile_of[seq_dp[par[j]]];
        }
    }
    tp.ntiles = ntiles;
    const int nl = tp.nlev;
    // buckets (tile, level, non-root) in original order
    const size_t nb = (size_t)ntiles * nl * 2;
    std::vector<int> bcount(nb + 1, 0);
    auto bucket = [&](int j) {
        return ((size_t)tile_of[j] * nl + (lev[j] - ls)) * 2 + (is_root(j, Jtop) ? 0 : 1);
    };
    for (int j = Jtop; j < J; ++j) bcount[bucket(j) + 1]++;
    for (size_t q = 0; q < nb; ++q) bcount[q + 1] += bcount[q];
    pp.perm.resize(J);
    std::iota(pp.perm.begin(), pp.perm.begin() + Jtop, 0);
    {
        std::vector<int> fill(bcount.begin(), bcount.end() - 1);
        for (int j = Jtop; j < J; ++j) pp.perm[Jtop + fill[bucket(j)]++] = j;
    }
    tp.h_off.assign((size_t)ntiles * (nl + 1), 0);
    std::vector<int> nroot((size_t)ntiles * nl, 0);
    for (int t = 0; t < ntiles; ++t) {
        for (int k = 0; k <= nl; ++k)  // k == nl: the start of the next tile
            tp.h_off[(size_t)t * (nl + 1) + k] = Jtop + bcount[((size_t)t * nl + k) * 2];
        for (int k = 0; k < nl; ++k) {
            const size_t q = ((size_t)t * nl + k) * 2;
            nroot[(size_t)t * nl + k] = bcount[q + 1] - bcount[q];
        }
    }
    // sequences follow their DPs
    pp.sperm.assign(S, 0);
    pp.sinv.assign(S, 0);
    pp.sp.assign(J + 1, 0);
    int next = 1;
    for (int d = 0; d < J; ++d) {
        const int j = pp.perm[d];
        pp.sp[d] = next;
        for (int s = sp[j]; s < sp[j + 1]; ++s) {
            pp.sperm[next] = s;
            pp.sinv[s] = next;
            ++next;
        }
    }
    pp.sp[J] = S;
    pp.par.assign(J, 0);
    for (int d = 0; d < J; ++d) pp.par[d] = pp.sinv[par[pp.perm[d]]];
    // child ranges in the new numbering; below the split the child DPs of a
    // sequence stay contiguous (the top keeps its original child ranges)
    std::vector<int> cfirst(S, -1), ccnt(S, 0);
    for (int d = Jtop; d < J; ++d) {
        const int ps = pp.par[d];
        if (ps < tp.Stop) continue;
        if (cfirst[ps] < 0) cfirst[ps] = d;
        else if (pp.par[d - 1] != ps) return false;
        ccnt[ps]++;
    }
    tp.h_shape.assign((size_t)ntiles * nl, TileShape{});
    tp.max_dps = tp.max_seqs = 0;
    tp.maxa = 1;
    for (int t = 0; t < ntiles; ++t) {
        const int* o = &tp.h_off[(size_t)t * (nl + 1)];
        tp.max_dps = std::max(tp.max_dps, o[nl] - o[0]);
        tp.max_seqs = std::max(tp.max_seqs, pp.sp[o[nl]] - pp.sp[o[0]]);
        for (int k = 0; k < nl; ++k) {
            TileShape sh = detect_shape(pp.sp, pp.par, cfirst, ccnt, o[k], o[k + 1]);
            sh.nroot = nroot[(size_t)t * nl + k];
            tp.h_shape[(size_t)t * nl + k] = sh;
        }
    }
    for (int d = Jtop; d < J; ++d) tp.maxa = std::max(tp.maxa, pp.sp[d + 1] - pp.sp[d]);
    tp.top_lvl.assign(P.lvl.begin(), P.lvl.begin() + ls + 1);
    tp.top_shape.clear();
    tp.top_warp = 0;
    for (int l = 0; l < ls; ++l) {  // the level engine's exact shapes (original numbering)
        const DevTree& o = P.lvl_shape[l];
        tp.top_shape.push_back(TileShape{o.j_lo, o.s_lo, o.un, o.cn, o.c_lo, o.pc, o.p_lo, 0});
        if (P.lvl_nj[l] <= 4096 && P.lvl_nc[l] >= 8.0 * P.lvl_nj[l]) tp.top_warp |= 1u << l;
    }
    // Algorithmic HBM bytes per pass (fp64 values, int32 indices, every array
    // touched once; structure only where a block is not affine; V only where
    // it leaves shared memory: the roots' V, and V / child V of the top).
    tp.bytes_obs = tp.bytes_obs_rm = tp.bytes_pred = tp.bytes_td_avg = tp.bytes_td = tp.bytes_cur = 0;
    auto add_block = [&](const TileShape& sh, int lo, int hi, bool top) {
        if (hi <= lo) return;
        const double nj = hi - lo, ns = pp.sp[hi] - pp.sp[lo];
        double nc = 0;
        if (top) {
            for (int l = 0; l < ls; ++l)
                if (P.lvl[l] == lo) nc = P.lvl_nc[l];
        } else {
            for (int q = pp.sp[lo]; q < pp.sp[hi]; ++q) nc += ccnt[q];
        }
        const bool single = sh.un == 1;
        const double st_up = (sh.un > 0 ? 0 : 4 * nj) + (sh.cn >= 0 ? 0 : 8 * ns);
        const double st_dn = (sh.un > 0 ? 0 : 4 * nj) + (sh.pc > 0 ? 0 : 4 * nj);
        const double vg = top ? 8 * nj + 8 * nc : 8.0 * sh.nroot;
        const double rb = single ? 0 : 24 * ns;
        tp.bytes_obs += 8 * ns + rb + vg + st_up;
        tp.bytes_obs_rm += 8 * ns + rb + (single ? 0 : 8 * ns) + vg + st_up;
        tp.bytes_pred += 8 * ns + rb + vg + st_up;
        const double bread = single ? 0 : 8 * ns;
        tp.bytes_td_avg += bread + 8 * ns + 16 * ns + st_dn;
        tp.bytes_td += bread + 8 * ns + st_dn;
        tp.bytes_cur += bread + 8 * ns + st_dn;
    };
    for (int l = 0; l < ls; ++l) add_block(tp.top_shape[l], P.lvl[l], P.lvl[l + 1], true);
    for (int t = 0; t < ntiles; ++t)
        for (int k = 0; k < nl; ++k) {
            const int* o = &tp.h_off[(size_t)t * (nl + 1)];
            add_block(tp.h_shape[(size_t)t * nl + k], o[k], o[k + 1], false);
        }
    tp.bytes_td_avg += 16;  // avg[0]
    return true;
}

bool prepare_tiled(scfr_handle* h, const scfr_csr* U, const scfr_csr* UT, bool required) {
    if (h->comm) {
        if (required) fail(SCFR_EINVAL, "the tile engine does not run the row-sharded mode");
        return false;
    }
    if (h->P[0].J == 0 || h->P[1].J == 0) {
        if (required) fail(SCFR_EINVAL, "the tile engine needs decision points for both players");
        return false;
    }
    PlayerPlan pp[2];
    for (int k = 0; k < 2; ++k)
        if (!plan_player(h, h->P[k], h->tp[k], pp[k])) {
            if (required) fail(SCFR_EINVAL, "no tile plan for player %d (tree shape)", k + 1);
            return false;
        }
    cudaStream_t s = h->stream;
    for (int k = 0; k < 2; ++k) {
        TilePlayer& tp = h->tp[k];
        Player& P = h->P[k];
        const int J = P.J, S = P.S;
        tp.seq_ptr.alloc(J + 1);
        tp.dp_parent.alloc(J);
        tp.child.alloc(S);
        tp.off.alloc(tp.h_off.size());
        tp.shape.alloc(tp.h_shape.size());
        tp.sperm.alloc(S);
        tp.dperm.alloc(J);
        tp.ticket.alloc(h->B);
        tp.gat.alloc(S);
        CUDA_OK(copy_async(tp.seq_ptr.p, pp[k].sp.data(), (J + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
        CUDA_OK(copy_async(tp.dp_parent.p, pp[k].par.data(), J * sizeof(int), cudaMemcpyHostToDevice, s));
        CUDA_OK(copy_async(tp.off.p, tp.h_off.data(), tp.h_off.size() * sizeof(int), cudaMemcpyHostToDevice, s));
        CUDA_OK(copy_async(tp.shape.p, tp.h_shape.data(), tp.h_shape.size() * sizeof(TileShape),
                           cudaMemcpyHostToDevice, s));
        CUDA_OK(copy_async(tp.sperm.p, pp[k].sperm.data(), S * sizeof(int), cudaMemcpyHostToDevice, s));
        CUDA_OK(copy_async(tp.dperm.p, pp[k].perm.data(), J * sizeof(int), cudaMemcpyHostToDevice, s));
        tp.child.zero(s);
        tp.ticket.zero(s);
        k_derive_child<<<grid_for(J), TPB, 0, s>>>(J, tp.dp_parent.p, tp.child.p);
        // initial behaviour in the tile numbering (uniform per DP)
        k_derive_uniform<<<grid_for(J), TPB, 0, s>>>(J, S, h->B, tp.seq_ptr.p, P.b.p);
        CUDA_OK(cudaGetLastError());
    }
    // payoff rows in the tile numbering: rows of U by player 1's order,
    // columns by player 2's (and the reverse for Uᵀ); nnz order kept per row
    for (int k = 0; k < 2; ++k) {
        const scfr_csr* m = k == 0 ? U : UT;
        const std::vector<int>& rperm = pp[k].sperm;
        const std::vector<int>& cinv = pp[1 - k].sinv;
        DevCsr& D = h->tM[k];
        D.rows = D.full_rows = D.chunk = (int)m->rows;
        D.cols = (int)m->cols;
        D.nnz = (int)m->nnz;
        D.row0 = 0;
        std::vector<int> ip(m->rows + 1), ix(std::max<int64_t>(m->nnz, 1));
        std::vector<double> dv(std::max<int64_t>(m->nnz, 1));
        ip[0] = 0;
        for (int64_t i = 0; i < m->rows; ++i) {
            const int64_t r = rperm[i], k0 = m->indptr[r], k1 = m->indptr[r + 1];
            int q = ip[i];
            for (int64_t e = k0; e < k1; ++e, ++q) {
                ix[q] = cinv[m->indices[e]];
                dv[q] = m->data[e];
            }
            ip[i + 1] = q;
        }
        D.indptr.alloc(ip.size());
        D.indices.alloc(ix.size());
        D.data.alloc(dv.size());
        CUDA_OK(copy_async(D.indptr.p, ip.data(), ip.size() * sizeof(int), cudaMemcpyHostToDevice, s));
        CUDA_OK(copy_async(D.indices.p, ix.data(), ix.size() * sizeof(int), cudaMemcpyHostToDevice, s));
        CUDA_OK(copy_async(D.data.p, dv.data(), dv.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaStreamSynchronize(s));  // staging vectors die here
        // the fused payoff rows: indptr, indices + data, x gathers (u write counted per block)
        const double spmv = 4.0 * (D.rows + 1) + 20.0 * D.nnz;
        h->tp[k].bytes_obs += spmv;
        h->tp[k].bytes_obs_rm += spmv;
    }
    // launch geometry: a persistent-style grid, tiles strided over the CTAs
    size_t up = 0, down = 0;
    for (int k = 0; k < 2; ++k) {
        h->tile_vwin = std::max(h->tile_vwin, h->tp[k].max_dps);
        up = std::max(up, (size_t)(h->tp[k].max_dps + 3 * kUCH + kPCH) * sizeof(double) +
                              (kUCH + 1) * sizeof(int));
        }
    for (int k = 0; k < 2; ++k) h->tile_dwin = std::max(h->tile_dwin, h->tp[k].Stop + h->tp[k].max_seqs);
    down = (size_t)(h->tile_dwin + 2 * kUCH) * sizeof(double);
    if (const char* e = std::getenv("SCFR_TILE_STAGE")) h->tile_staged = std::atoi(e) != 0;
    h->tile_smem_up = up;
    h->tile_smem_down = down;
    h->tile_threads = kTileThreads;
    CUDA_OK(cudaStreamSynchronize(s));
    return true;
}

// ---------------------------------------------------------------------------
// Host: per-iteration launches.

static TileTask make_task(scfr_handle* h, int k, const double* u, double* x) {
    TilePlayer& tp = h->tp[k];
    Player& P = h->P[k];
    TileTask t{};
    t.seq_ptr = tp.seq_ptr.p;
    t.dp_parent = tp.dp_parent.p;
    t.child = tp.child.p;
    t.top_seq_ptr = P.seq_ptr.p;
    t.top_dp_parent = P.dp_parent.p;
    t.top_child = P.child.p;
    t.dperm = tp.dperm.p;
    t.off = tp.off.p;
    t.shp = tp.shape.p;
    t.ntiles = tp.ntiles;
    t.nlev = tp.nlev;
    t.ls = tp.ls;
    t.Stop = tp.Stop;
    for (int l = 0; l <= tp.ls; ++l) t.top_lvl[l] = tp.top_lvl[l];
    for (int l = 0; l < tp.ls; ++l) t.top_shp[l] = tp.top_shape[l];
    t.top_warp = tp.top_warp;
    t.S = P.S;
    t.J = P.J;
    t.u = u;
    t.r = P.r.p;
    t.b = P.b.p;
    t.x = x;
    t.avg = P.avg.p;
    t.V = P.V.p;
    t.ticket = tp.ticket.p;
    t.vwin = h->tile_vwin;
    t.staged = h->tile_staged;
    return t;
}

using TileKernel = void (*)(TileTask, TileTask, KParams);

template <int KIND>
static TileKernel pick_up(int maxa) {
    if (maxa <= 1) return k_tile_up<KIND, 1>;
    if (maxa <= 2) return k_tile_up<KIND, 2>;
    if (maxa <= 4) return k_tile_up<KIND, 4>;
    return k_tile_up<KIND, 8>;
}
template <int KIND>
static TileKernel pick_down(int maxa) {
    if (maxa <= 1) return k_tile_down<KIND, 1>;
    if (maxa <= 2) return k_tile_down<KIND, 2>;
    if (maxa <= 4) return k_tile_down<KIND, 4>;
    return k_tile_down<KIND, 8>;
}

// Resident CTAs of `kern` at `smem` bytes (cached per handle), capping the grid.
static int resident_grid(scfr_handle* h, TileKernel kern, size_t smem, int tiles) {
    const void* key = reinterpret_cast<const void*>(kern);
    int occ = 0;
    for (const auto& e : h->tile_occ)
        if (e.first == key) occ = e.second;
    if (!occ) {
        CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTileThreads, smem));
        if (occ < 1) fail(SCFR_ECUDA, "tile kernel cannot be resident (%zu B shared memory)", smem);
        h->tile_occ.emplace_back(key, occ);
    }
    int cap = occ * h->num_sms;
    if (const char* e = std::getenv("SCFR_TILE_CTAS")) cap = std::max(1, std::min(cap, std::atoi(e)));
    return std::max(1, std::min(tiles, cap));
}

// One pass over player tasks a (and optionally b) as one launch.
static void pass(LaunchBase& L, int kk, bool up, int kind, bool do_rm, TileTask a, const TileTask* b,
                 int maxa, double bytes) {
    scfr_handle* h = L.h;
    TileTask t1 = b ? *b : TileTask{};
    if (!b) t1.ntiles = 0;
    TileKernel kern;
    if (up) kern = kind == TK_OBS ? pick_up<TK_OBS>(maxa) : pick_up<TK_PRED>(maxa);
    else kern = kind == TK_TD_AVG ? pick_down<TK_TD_AVG>(maxa)
              : kind == TK_TD ? pick_down<TK_TD>(maxa) : pick_down<TK_CUR>(maxa);
    const size_t smem = up ? h->tile_smem_up : h->tile_smem_down;
    a.vwin = t1.vwin = up ? h->tile_vwin : h->tile_dwin;  // staging sits after this window
    const int grid = resident_grid(h, kern, smem, a.ntiles + t1.ntiles);
    const KParams kp = L.kparams(do_rm);
    L.launch(kk, bytes, [&] { L.run_ex(kern, dim3(grid, h->B), kTileThreads, smem, a, t1, kp); });
}

void tiled_iteration(LaunchBase& L) {
    scfr_handle* h = L.h;
    Player& A = h->P[0];
    Player& Bp = h->P[1];
    const bool pr = predictive(h->variant);
    const int maxa = std::max(h->tp[0].maxa, h->tp[1].maxa);
    const bool alt = h->mode == SCFR_MODE_ALT;
    // next(): [PRED] then TD + average, both players per launch
    if (pr) {
        TileTask a = make_task(h, 0, A.u.p, A.x.p), b = make_task(h, 1, Bp.u.p, Bp.x.p);
        pass(L, KK_PRED, true, TK_PRED, false, a, &b, maxa,
             h->tp[0].bytes_pred + h->tp[1].bytes_pred);
    }
    {
        TileTask a = make_task(h, 0, nullptr, A.x.p), b = make_task(h, 1, nullptr, Bp.x.p);
        pass(L, KK_TD_AVG, false, TK_TD_AVG, false, a, &b, maxa,
             h->tp[0].bytes_td_avg + h->tp[1].bytes_td_avg);
    }
    // observe(): OBS with the payoff rows fused (u1 = U x2, u2 = -Uᵀ x1 / x1')
    TileTask o1 = make_task(h, 0, A.u.p, A.x.p), o2 = make_task(h, 1, Bp.u.p, Bp.x.p);
    o1.fu = FuseU{h->tM[0].indptr.p, h->tM[0].indices.p, h->tM[0].data.p, Bp.x.p, 0};
    o1.fu_sx = Bp.S;
    o2.fu = FuseU{h->tM[1].indptr.p, h->tM[1].indices.p, h->tM[1].data.p, alt ? A.xpost.p : A.x.p, 1};
    o2.fu_sx = A.S;
    const int kobs = pr ? KK_OBS : KK_OBS_RM;
    const double ob1 = pr ? h->tp[0].bytes_obs : h->tp[0].bytes_obs_rm;
    const double ob2 = pr ? h->tp[1].bytes_obs : h->tp[1].bytes_obs_rm;
    if (!alt) {
        pass(L, kobs, true, TK_OBS, !pr, o1, &o2, maxa, ob1 + ob2);
    } else {
        pass(L, kobs, true, TK_OBS, !pr, o1, nullptr, maxa, ob1);
        // current_strategy of player 1 into xpost: RM on the fly (predictive)
        // or TD of the b that OBS already regret-matched
        TileTask c = make_task(h, 0, nullptr, A.xpost.p);
        pass(L, pr ? KK_CUR : KK_TD, false, pr ? TK_CUR : TK_TD, false, c, nullptr, maxa,
             pr ? h->tp[0].bytes_cur : h->tp[0].bytes_td);
        pass(L, kobs, true, TK_OBS, !pr, o2, nullptr, maxa, ob2);
    }
    L.launch(KK_TICK, 0.0, [&] { L.run1(k_tick, dim3(1), h->tdev.p, L.tl, (int)L.count); });
}

__global__ void k_scatter_seq(int S, const int* __restrict__ sperm, const double* __restrict__ src,
                              double* __restrict__ dst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < S) dst[sperm[i]] = src[i];
}

__global__ void k_widen_f32(int n, const float* __restrict__ f, double* __restrict__ d) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) d[i] = (double)f[i];
}

const double* orig_order(scfr_handle* h, int player, const double* buf, int solve) {
    Player& P = h->P[player - 1];
    if (h->f32) {  // fp32 state (level engine, reference order): widen exactly
        const float* f = reinterpret_cast<const float*>(buf) + (size_t)solve * P.S;
        k_widen_f32<<<grid_for(P.S), TPB, 0, h->stream>>>(P.S, f, P.wide.p);
        CUDA_OK(cudaGetLastError());
        return P.wide.p;
    }
    const double* src = buf + (size_t)solve * P.S;
    if (h->engine != SCFR_ENGINE_TILED) return src;
    TilePlayer& tp = h->tp[player - 1];
    k_scatter_seq<<<grid_for(P.S), TPB, 0, h->stream>>>(P.S, tp.sperm.p, src, tp.gat.p);
    CUDA_OK(cudaGetLastError());
    return tp.gat.p;
}

}  // namespace scfr
