// Device runtime behind the C-ABI: structure upload, the level engine (one
// kernel per DP level, captured once as a CUDA graph), on-device best
// response, and the C entry points.  The persistent engine is in
// persistent.cu.
//
// One iteration is the reference _step (pkg/solvers.py:351-372):
//   sim:  next1, next2, u1 = U x2, u2 = -Uᵀ x1, observe1(u1), observe2(u2)
//   alt:  next1, next2, u1 = U x2, observe1(u1), x1' = current1(),
//         u2 = -Uᵀ x1', observe2(u2)
// mapped onto fused per-level kernels (kernels.cuh):
//   next    = [PRED levels deep→shallow, if predictive] + TD levels (+avg)
//   observe = OBS levels deep→shallow (+ RM into b for non-predictive)
//   current = CUR levels (predictive) / TD levels without avg (otherwise:
//             b was already regret-matched by OBS)
// Per-iteration scalars (t^gamma, DCFR factors) come from host-computed
// schedules indexed by a device-side iteration counter, so one captured
// graph serves every iteration.

#include <algorithm>
#include <exception>
#include <thread>
#include <atomic>
#include <chrono>
#include <memory>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>  // types only: the library is dlopen'ed by the multi-GPU modes

#include "host_par.h"
#include "runtime.h"
#include "subtree.h"

namespace scfr {

bool predictive(int v) { return v == SCFR_PCFR || v == SCFR_PCFR_PLUS; }
int post_of(int v) {
    if (v == SCFR_CFR_PLUS || v == SCFR_PCFR_PLUS) return POST_PLUS;
    if (v == SCFR_DCFR) return POST_DCFR;
    return POST_NONE;
}

// ---------------------------------------------------------------------------
// Level kernels.  One launch covers one DP level of up to two players (the
// passes of player 1 and player 2 are independent in next() and, in
// simultaneous mode, in observe()): blocks [0, t0.nblk) serve task t0, the
// rest t1; blockIdx.y is the solve within a batch.  Producers of every value
// read here ran in earlier launches, so plain L1-cacheable loads are
// coherent.  Thread-per-DP for thin levels, warp-per-DP (lane = action) for
// fat ones.

template <class R>  // value type: double, or float in the fp32 mode
struct TaskT {
    DevTree T;
    int lo, n;   // DPs [lo, lo+n)
    int S, J;    // per-solve strides of seq- and dp-indexed state
    int nblk;    // blocks of the launch serving this task
    const R* u;  // utility (OBS) / prediction (PRED)
    R* r;
    R* b;
    R* x;
    R* avg;
    R* V;
    FuseUT<R> fu;  // fu.ip set: OBS computes u from the payoff rows (fused SpMV)
    int fu_sx;     // per-solve stride of fu.x
    const R* Vc;   // OBS / PRED: child values read from here (u / the prediction; kernels.cuh leaf_note), per-solve stride S
    int skip_v;    // OBS on a forced leaf level whose V nobody reads
    R* bw;         // OBS: regret matching writes here instead of b (bcur)
    // Top-down launch of level ls of a player with a top (prepare_top): the
    // parents' x come from their ancestor chains, and the launch also writes
    // the top's x (and average).
    const TopInfo* top;
    // OBS group launch over the level above a forced leaf level: the leaf's
    // fused payoff rows are computed here (lfu.ip set), u written, used as
    // the child values; the leaf launch is skipped.  Child DP c is sequence
    // c + lshift.
    FuseUT<R> lfu;
    int lshift;
    R* tu_leaf;  // the utility array the leaf rows are written to
    // Parent pair (bottom-up group launches, Launcher::pair_ok): the launch
    // also computes the parent level.  A warp takes pblk parent DPs, runs
    // their pblk*pch children (this level, contiguous) in group rounds, then
    // the parents from the children's V.
    int pair, plo, pn, pblk, pch;
    DevTree PT;       // the parent level's shape
    FuseUT<R> pfu;    // the parent level's fused payoff rows (fu.ip unset: none)
    const R* pu;      // the parent level's utility / prediction (null: empty rows)
};
using Task = TaskT<double>;

// --- the top: last-arrival completion, ancestor-chain x -----------------

// x of top sequence p from its ancestor chain: b_a0·1.0, then b_a1·that, ...
// (x[s] = b[s]·x[parent] with x[0] = 1.0; a forced level's b is 1.0 and is
// not read).  src: b (or bcur) of this solve.
template <class R>
__device__ __forceinline__ R top_x(const TopInfo* tp, const R* src, int p) {
    if (p == 0) return R(1);
    const int ls = tp->ls;
    const int* an = tp->anc + (size_t)p * ls;
    int a[kTopMax];
    R bv[kTopMax];
#pragma unroll
    for (int l = 0; l < kTopMax; ++l) a[l] = l < ls ? __ldg(an + l) : -1;
#pragma unroll
    for (int l = 0; l < kTopMax; ++l) bv[l] = a[l] >= 0 && !(a[l] & (1 << 30)) ? src[a[l]] : R(1);
    R x = R(1);
#pragma unroll
    for (int l = 0; l < kTopMax; ++l)
        if (a[l] >= 0) x = dmul(bv[l], x);
    return x;
}

// Work of a top-down level-ls launch before its DPs: the top's x (and
// average), once per solve across the task's CTAs.
template <int KIND, class R>
__device__ __forceinline__ void top_prologue(const TaskT<R>& t, int blk, R w) {
    const size_t so = (size_t)blockIdx.y * t.S;
    const TopInfo* tp = t.top;
    if (!tp->pro) return;
    const R* src = t.b + so;
    for (int s = 1 + blk * TPB + (int)threadIdx.x; s < tp->Stop; s += t.nblk * TPB) {
        const R xa = top_x(tp, src, s);
        t.x[so + s] = xa;
        if (KIND == LK_TD_AVG) t.avg[so + s] = dadd(dmul(w, xa), t.avg[so + s]);
    }
    if (KIND == LK_TD_AVG && blk == 0 && threadIdx.x == 0)  // the reference axpy also covers x[0] = 1
        t.avg[so] = dadd(dmul(w, t.x[so]), t.avg[so]);
}

// The task's blocks stride over its DPs (grid-stride): a launch is capped at
// about one resident wave, so the deep levels (10^6 DPs of a few loads each)
// are not limited by CTA scheduling.
template <int KIND, int MAXA, bool WARP, class R>
__device__ __forceinline__ void level_body(const TaskT<R>& t, int blk, const KParams& kp) {
    constexpr int kPerBlock = WARP ? TPB / 32 : TPB;
    const int stride = t.nblk * kPerBlock;
    const size_t so = (size_t)blockIdx.y * t.S;
    R* V = t.V + (size_t)blockIdx.y * (t.J > 0 ? t.J : 1);
    const int lane = threadIdx.x & 31;
    // schedules are fp64 (host libm pow); the fp32 mode rounds them once
    R w = R(0), pf = R(1), nf = R(1);
    if (KIND == LK_TD_AVG) w = (R)kp.wsched[(size_t)blockIdx.y * kp.cap + *kp.tdev + kp.tofs];
    if (KIND == LK_OBS && kp.post == POST_DCFR) {
        const size_t k = (size_t)blockIdx.y * kp.cap + *kp.tdev + kp.tofs;
        pf = (R)kp.pfsched[k];
        nf = (R)kp.nfsched[k];
    }
    FuseUT<R> fu = t.fu;
    if (KIND == LK_OBS && fu.ip) fu.x += (size_t)blockIdx.y * t.fu_sx;
    const int first = blk * kPerBlock + (WARP ? (int)threadIdx.x / 32 : (int)threadIdx.x);
    if (KIND == LK_TD_AVG && first == 0 && (!WARP || lane == 0) && t.lo == 0 && t.n > 0) {  // the reference axpy also covers the empty sequence (x[0] = 1)
        R* avg = t.avg + so;
        avg[0] = dadd(dmul(w, t.x[so]), avg[0]);
    }
    if (KIND == LK_OBS && fu.ip && first == 0 && lane == 0 && t.lo == 0 && t.n > 0) {  // the empty sequence's row: u[0] (next prediction)
        bool bad = false;
        FuseUT<R> f0 = fu;  // row 0 is outside the level's row shape
        f0.rc = 0;
        fused_u<LdL1>(f0, const_cast<R*>(t.u) + so, 0, bad);
        if (bad) atomicOr(kp.nonfinite, 1);
    }
    if ((KIND == LK_TD_AVG || KIND == LK_TD) && t.top) top_prologue<KIND, R>(t, blk, w);
    for (int item = first; item < t.n; item += stride) {  // warp-uniform in warp mode
        const int j = t.lo + item;
        if constexpr (KIND == LK_TD_AVG || KIND == LK_TD) {
            R xp;  // the top's x is recomputed from the ancestor chain
            if (t.top) xp = top_x(t.top, t.b + so, parent_of<LdL1>(t.T, j));
            const R* xpp = t.top ? &xp : nullptr;
            R* avg = KIND == LK_TD_AVG ? t.avg + so : nullptr;
            if constexpr (WARP) td_dp_warp<LdL1>(t.T, j, t.b + so, t.x + so, avg, w, lane, xpp);
            else td_dp<LdL1>(t.T, j, t.b + so, t.x + so, avg, w, xpp);
        } else if constexpr (KIND == LK_CUR) {
            cur_dp<MAXA, LdL1>(t.T, j, t.r + so, t.x + so);
        } else if constexpr (KIND == LK_OBS) {
            const R* Vc = t.Vc ? t.Vc + so : nullptr;
            if constexpr (WARP)
                obs_dp_warp<LdL1>(t.T, j, t.u ? t.u + so : nullptr, t.r + so, t.b + so, V, kp.post, pf, nf,
                                  kp.do_rm != 0, kp.nonfinite, lane, fu, Vc, t.bw ? t.bw + so : nullptr);
            else
                obs_dp<MAXA, LdL1>(t.T, j, t.u ? t.u + so : nullptr, t.r + so, t.b + so, V, kp.post, pf, nf,
                                   kp.do_rm != 0, kp.nonfinite, fu, Vc, t.skip_v != 0,
                                   t.bw ? t.bw + so : nullptr);
        } else {
            const R* Vc = t.Vc ? t.Vc + so : nullptr;
            if constexpr (WARP)
                pred_dp_warp<LdL1>(t.T, j, t.u ? t.u + so : nullptr, t.r + so, t.b + so, V, kp.plus != 0, lane, Vc);
            else
                pred_dp<MAXA, LdL1>(t.T, j, t.u ? t.u + so : nullptr, t.r + so, t.b + so, V, kp.plus != 0, Vc);
        }
    }
}

// Group mode (kernels.cuh): G = 32/n DPs per warp, lane = (DP, action), on
// big affine levels with n = T.un actions.  The task's warps stride over
// groups of G DPs; the loop bound is warp-uniform so every lane reaches the
// shuffles.  Never used on level 0 (the empty sequence's extra work).
template <int KIND, int N, class R>
__device__ __forceinline__ void level_body_group(const TaskT<R>& t, int blk, const KParams& kp) {
    constexpr int W = TPB / 32;
    const size_t so = (size_t)blockIdx.y * t.S;
    R* V = t.V + (size_t)blockIdx.y * (t.J > 0 ? t.J : 1);
    const int n = N > 0 ? N : t.T.un, G = 32 / n;
    const int lane = threadIdx.x & 31, g = lane / n, a = lane - g * n, gb = g * n;
    R w = R(0), pf = R(1), nf = R(1);
    if (KIND == LK_TD_AVG) w = (R)kp.wsched[(size_t)blockIdx.y * kp.cap + *kp.tdev + kp.tofs];
    if (KIND == LK_OBS && kp.post == POST_DCFR) {
        const size_t k = (size_t)blockIdx.y * kp.cap + *kp.tdev + kp.tofs;
        pf = (R)kp.pfsched[k];
        nf = (R)kp.nfsched[k];
    }
    FuseUT<R> fu = t.fu;
    if (KIND == LK_OBS && fu.ip) fu.x += (size_t)blockIdx.y * t.fu_sx;
    const R* Vc = t.Vc ? t.Vc + so : nullptr;
    if ((KIND == LK_TD_AVG || KIND == LK_TD) && t.top) top_prologue<KIND, R>(t, blk, w);
    if constexpr (KIND == LK_OBS || KIND == LK_PRED) {
        if (t.pair) {  // blocks of pblk parents: their children, then the parents
            FuseUT<R> pfu = t.pfu;
            if (KIND == LK_OBS && pfu.ip) pfu.x += (size_t)blockIdx.y * t.fu_sx;
            const int pn2 = t.PT.un, pG = 32 / pn2, pg = lane / pn2, pa = lane - pg * pn2, pgb = pg * pn2;
            for (int bi = blk * W + (int)(threadIdx.x >> 5); bi * t.pblk < t.pn; bi += t.nblk * W) {
                const int p0 = bi * t.pblk, np = min(t.pblk, t.pn - p0);
                const int c0 = p0 * t.pch, c1 = c0 + np * t.pch;
                for (int base = c0; base < c1; base += G) {
                    const int item = base + g;
                    const bool valid = g < G && item < c1;
                    const int j = t.lo + (valid ? item : c0);
                    if constexpr (KIND == LK_OBS)
                        obs_dp_group<LdL1s, N>(t.T, j, valid, a, gb, n, t.u ? t.u + so : nullptr, t.r + so, t.b + so,
                                               V, kp.post, pf, nf, kp.do_rm != 0, kp.nonfinite, fu, Vc,
                                               t.bw ? t.bw + so : nullptr);
                    else
                        pred_dp_group<LdL1s, N>(t.T, j, valid, a, gb, n, t.u ? t.u + so : nullptr, t.r + so,
                                                t.b + so, V, kp.plus != 0, Vc);
                }
                __syncwarp();  // the children's V (this warp's) before the parents read them
                const bool pv = pg < pG && pg < np;
                const int pj = t.plo + p0 + (pv ? pg : 0);
                if constexpr (KIND == LK_OBS)
                    obs_dp_group<LdL1s>(t.PT, pj, pv, pa, pgb, pn2, t.pu ? t.pu + so : nullptr, t.r + so, t.b + so, V,
                                        kp.post, pf, nf, kp.do_rm != 0, kp.nonfinite, pfu,
                                        static_cast<const R*>(nullptr), t.bw ? t.bw + so : nullptr);
                else
                    pred_dp_group<LdL1s>(t.PT, pj, pv, pa, pgb, pn2, t.pu ? t.pu + so : nullptr, t.r + so, t.b + so,
                                         V, kp.plus != 0, static_cast<const R*>(nullptr));
            }
            return;
        }
    }
    for (int wi = blk * W + (int)(threadIdx.x >> 5); wi * G < t.n; wi += t.nblk * W) {
        const int item = wi * G + g;
        const bool valid = g < G && item < t.n;
        const int j = t.lo + (valid ? item : 0);
        if constexpr (KIND == LK_TD_AVG || KIND == LK_TD) {
            R xp = R(0);  // the top's x, recomputed from the ancestor chain by the group's first lane
            if (t.top) {
                if (valid && a == 0) xp = top_x(t.top, t.b + so, parent_of<LdL1>(t.T, j));
                xp = __shfl_sync(kFullMask, xp, gb);
            }
            td_dp_group<LdL1s>(t.T, j, valid, a, n, t.b + so, t.x + so, KIND == LK_TD_AVG ? t.avg + so : nullptr, w,
                               t.top ? &xp : nullptr);
        } else if constexpr (KIND == LK_CUR) {
            cur_dp_group<LdL1s, N>(t.T, j, valid, a, gb, n, t.r + so, t.x + so);
        } else if constexpr (KIND == LK_OBS) {
            if (t.lfu.ip) {
                FuseUT<R> lfu = t.lfu;
                lfu.x += (size_t)blockIdx.y * t.fu_sx;
                obs_dp_group<LdL1s, N>(t.T, j, valid, a, gb, n, t.u ? t.u + so : nullptr, t.r + so, t.b + so, V,
                                       kp.post, pf, nf, kp.do_rm != 0, kp.nonfinite, fu, Vc,
                                       t.bw ? t.bw + so : nullptr, static_cast<R*>(nullptr), &lfu, t.tu_leaf + so,
                                       t.lshift);
            } else {
                obs_dp_group<LdL1s, N>(t.T, j, valid, a, gb, n, t.u ? t.u + so : nullptr, t.r + so, t.b + so, V,
                                       kp.post, pf, nf, kp.do_rm != 0, kp.nonfinite, fu, Vc,
                                       t.bw ? t.bw + so : nullptr);
            }
        } else {
            pred_dp_group<LdL1s, N>(t.T, j, valid, a, gb, n, t.u ? t.u + so : nullptr, t.r + so, t.b + so, V,
                                kp.plus != 0, Vc);
        }
    }
}

#ifndef SCFR_GROUP_MINB
#define SCFR_GROUP_MINB 8
#endif
#ifndef SCFR_GROUP_MINB_OBS
#define SCFR_GROUP_MINB_OBS SCFR_GROUP_MINB
#endif
template <int KIND, int N, class R>
__global__ void __launch_bounds__(TPB, (KIND == LK_OBS ? SCFR_GROUP_MINB_OBS : SCFR_GROUP_MINB)) k_level_g(const __grid_constant__ TaskT<R> t0,
                                                    const __grid_constant__ TaskT<R> t1,
                                                    const __grid_constant__ KParams kp) {
    pdl_launch_dependents();
    pdl_wait();
    tl_start(kp.tl, kp.tl_idx);
    if ((int)blockIdx.x < t0.nblk) level_body_group<KIND, N, R>(t0, blockIdx.x, kp);
    else level_body_group<KIND, N, R>(t1, blockIdx.x - t0.nblk, kp);
    tl_end(kp.tl, kp.tl_idx);
}

// --- pipelined group mode --------------------------------------------------
// The big affine levels are bound by the loads each warp keeps in flight: a
// group round issues ~4 per lane and waits a full HBM round trip for them
// (Little's law: ~5 MB in flight across the GPU, ~3 TB/s).  Here every warp
// stages the inputs of its next kPipe - 1 rounds into shared memory with
// cp.async (LDGSTS: per-lane addresses, no registers held) while it computes
// the current round from the staged copy.  Slot layout (R values): up passes
// [u | b | r | child values, cn per sequence], top-down [b or r | avg |
// parent x], 32 lanes each.  The per-round arithmetic is the group code.
constexpr int kPipe = 4;

template <class R>
__device__ __forceinline__ void cp_async_val(R* dst, const R* src) {
    if constexpr (sizeof(R) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                     "l"(src)
                     : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                     "l"(src)
                     : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(NPEND) : "memory");
}

template <int KIND, int N, class R>
__device__ __forceinline__ void level_body_gp(const TaskT<R>& t, int blk, const KParams& kp, R* smem) {
    constexpr int W = TPB / 32;
    constexpr bool UP = KIND == LK_OBS || KIND == LK_PRED;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t so = (size_t)blockIdx.y * t.S;
    R* V = t.V + (size_t)blockIdx.y * (t.J > 0 ? t.J : 1);
    constexpr int n = N, G = 32 / N;
    const int g = lane / n, a = lane - g * n, gb = g * n;
    R w = R(0), pf = R(1), nf = R(1);
    if (KIND == LK_TD_AVG) w = (R)kp.wsched[(size_t)blockIdx.y * kp.cap + *kp.tdev + kp.tofs];
    if (KIND == LK_OBS && kp.post == POST_DCFR) {
        const size_t k = (size_t)blockIdx.y * kp.cap + *kp.tdev + kp.tofs;
        pf = (R)kp.pfsched[k];
        nf = (R)kp.nfsched[k];
    }
    FuseUT<R> fu = t.fu;
    if (KIND == LK_OBS && fu.ip) fu.x += (size_t)blockIdx.y * t.fu_sx;
    const DevTree& T = t.T;
    const int cn = UP ? T.cn : 0;
    const int sv = 32 * (3 + cn);  // R values per slot
    R* wsm = smem + (size_t)warp * kPipe * sv;
    const R* Vr = t.Vc ? t.Vc + so : V;
    const R* ug = t.u ? t.u + so : nullptr;
    const bool stage_u = UP && ug && !fu.ip;
    const int ngroups = (t.n + G - 1) / G;
    const int first = blk * W + warp, stride = t.nblk * W;
    auto stage = [&](int wi, int q) {
        if (wi >= ngroups) return;
        const int j0 = t.lo + wi * G;
        const int ns = min(G, t.n - wi * G) * n;
        const int s0 = T.s_lo + (j0 - T.j_lo) * n;
        R* sl = wsm + q * sv;
        if (lane < ns) {
            const int s = s0 + lane;
            if constexpr (UP) {
                if (stage_u) cp_async_val(sl + lane, ug + s);
                cp_async_val(sl + 32 + lane, t.b + so + s);
                cp_async_val(sl + 64 + lane, t.r + so + s);
                const int c0 = T.c_lo + (s - T.s_lo) * cn;
                for (int c = 0; c < cn; ++c) cp_async_val(sl + 96 + lane * cn + c, Vr + c0 + c);
            } else {
                cp_async_val(sl + lane, (KIND == LK_CUR ? t.r : t.b) + so + s);
                if (KIND == LK_TD_AVG) cp_async_val(sl + 32 + lane, t.avg + so + s);
                cp_async_val(sl + 64 + lane, t.x + so + parent_of<LdL1>(T, j0 + lane / n));
            }
        }
    };
#pragma unroll
    for (int i = 0; i < kPipe - 1; ++i) {
        stage(first + i * stride, i);
        cp_async_commit();
    }
    for (int i = 0; first + i * stride < ngroups; ++i) {
        const int wi = first + i * stride;
        stage(first + (i + kPipe - 1) * stride, (i + kPipe - 1) % kPipe);
        cp_async_commit();
        cp_async_wait<kPipe - 1>();  // this lane's copies of round i
        __syncwarp();                // ... and every lane's
        R* sl = wsm + (i % kPipe) * sv;
        const int j0 = t.lo + wi * G;
        const int s0 = T.s_lo + (j0 - T.j_lo) * n;
        const int item = wi * G + g;
        const bool valid = g < G && item < t.n;
        const int j = t.lo + (valid ? item : wi * G);
        if constexpr (UP) {
            const R* u_arg = fu.ip ? ug : stage_u ? sl - s0 : nullptr;
            const R* vc = sl + 96 - (T.c_lo + (s0 - T.s_lo) * cn);
            if constexpr (KIND == LK_OBS)
                obs_dp_group<LdS, N>(T, j, valid, a, gb, n, u_arg, sl + 64 - s0, sl + 32 - s0, V, kp.post, pf, nf,
                                     kp.do_rm != 0, kp.nonfinite, fu, vc, t.bw ? t.bw + so : t.b + so, t.r + so);
            else
                pred_dp_group<LdS, N>(T, j, valid, a, gb, n, u_arg, sl + 64 - s0, sl + 32 - s0, V, kp.plus != 0, vc,
                                      t.b + so);
        } else {
            // td_dp_group / cur_dp_group on the staged copies
            const R xp = sl[64 + lane];
            const int s = s0 + lane;
            if constexpr (KIND == LK_CUR) {
                const R rv = valid ? sl[lane] : R(0);
                const R S = group_seq_sum<N>(rv > R(0) ? rv : R(0), gb, n);
                if (valid) t.x[so + s] = dmul(rm_prob(rv, S, n), xp);
            } else if (valid) {
                const R xa = dmul(sl[lane], xp);
                t.x[so + s] = xa;
                if (KIND == LK_TD_AVG) t.avg[so + s] = dadd(dmul(w, xa), sl[32 + lane]);
            }
        }
        __syncwarp();  // round i's slot is restaged at i + 1
    }
    cp_async_wait<0>();
}

template <int KIND, int N, class R>
__global__ void __launch_bounds__(TPB, 8) k_level_gp(const __grid_constant__ TaskT<R> t0,
                                                     const __grid_constant__ TaskT<R> t1,
                                                     const __grid_constant__ KParams kp) {
    extern __shared__ __align__(16) unsigned char gsm[];
    pdl_launch_dependents();
    pdl_wait();
    tl_start(kp.tl, kp.tl_idx);
    if ((int)blockIdx.x < t0.nblk) level_body_gp<KIND, N, R>(t0, blockIdx.x, kp, reinterpret_cast<R*>(gsm));
    else level_body_gp<KIND, N, R>(t1, blockIdx.x - t0.nblk, kp, reinterpret_cast<R*>(gsm));
    tl_end(kp.tl, kp.tl_idx);
}

// Narrow variants (<= 2 actions in registers: the deep, bandwidth-bound
// levels) are held to 40 registers so 12 CTAs fit per SM (more loads in
// flight); wide / warp variants keep the default budget.  (A batched variant
// with 4 DPs' loads in flight per thread measured no faster: these levels
// already run within ~10% of a bare fp64 stream of the same size on B200,
// scripts/micro/stream_probe.cu.)
template <int KIND, int MAXA, bool WARP, class R>
__global__ void __launch_bounds__(TPB, (MAXA <= 2 && !WARP) ? 12 : WARP ? 4 : 1) k_level(const __grid_constant__ TaskT<R> t0,
                                               const __grid_constant__ TaskT<R> t1,
                                               const __grid_constant__ KParams kp) {
    pdl_launch_dependents();
    pdl_wait();
    tl_start(kp.tl, kp.tl_idx);
    if ((int)blockIdx.x < t0.nblk) level_body<KIND, MAXA, WARP, R>(t0, blockIdx.x, kp);
    else level_body<KIND, MAXA, WARP, R>(t1, blockIdx.x - t0.nblk, kp);
    tl_end(kp.tl, kp.tl_idx);
}

template <class R>
using LevelKernelT = void (*)(TaskT<R>, TaskT<R>, KParams);
using LevelKernel = LevelKernelT<double>;

template <int N, class R>
static LevelKernelT<R> pick_pipe_kernel_n(int kind) {
    switch (kind) {
        case LK_TD_AVG: return k_level_gp<LK_TD_AVG, N, R>;
        case LK_TD: return k_level_gp<LK_TD, N, R>;
        case LK_CUR: return k_level_gp<LK_CUR, N, R>;
        case LK_OBS: return k_level_gp<LK_OBS, N, R>;
        default: return k_level_gp<LK_PRED, N, R>;
    }
}


// Warp-per-DP only pays on small, fat levels: few DPs (parallelism is
// scarce, so per-DP latency is the critical path) with >= 8 child-DP
// references per DP (long serial chains in a single thread).  Measured on
// Goofspiel-5: the 5- and 500-DP top levels drop from 8-16 µs to ~5 µs;
// warp mode on the 24K/432K-DP levels is 2-20x slower than thread mode.
// Wide levels (>= 5 actions somewhere) also go warp-per-DP: the thread path
// walks a wide DP's actions as a serial chain of L2 round trips (Liar's dice:
// 12-way bids, ~15 µs per level launch).
// Small multi-action levels (<= 4096 DPs, at most ~half a wave of warps)
// too: their launch time is one DP's latency chain, and the thread path
// serialises the actions' fused payoff rows (Liar's dice: a 1320-DP level
// with 4 actions took 16 µs as 11 CTAs of threads).
bool warp_level(const scfr_handle* h, const Player& P, int l) {
    return (P.lvl_nj[l] <= h->warp_nj &&
            (P.lvl_nc[l] >= 8.0 * P.lvl_nj[l] || (h->small_warp && P.lvl_maxa[l] >= 2))) ||
           (P.lvl_maxa[l] >= kWideActions && P.lvl_maxa[l] <= 32);
}

// Group kernels specialised on the common widths (2..4 actions: the
// shuffled in-order sums unroll), else the width is read at run time.
template <int N, class R>
static LevelKernelT<R> pick_group_kernel_n(int kind) {
    switch (kind) {
        case LK_TD_AVG: return k_level_g<LK_TD_AVG, N, R>;
        case LK_TD: return k_level_g<LK_TD, N, R>;
        case LK_CUR: return k_level_g<LK_CUR, N, R>;
        case LK_OBS: return k_level_g<LK_OBS, N, R>;
        default: return k_level_g<LK_PRED, N, R>;
    }
}
template <class R>
static LevelKernelT<R> pick_group_kernel(int kind, int un) {
    switch (un) {
        case 2: return pick_group_kernel_n<2, R>(kind);
        case 3: return pick_group_kernel_n<3, R>(kind);
        case 4: return pick_group_kernel_n<4, R>(kind);
        default: return pick_group_kernel_n<0, R>(kind);
    }
}

template <class R>
static LevelKernelT<R> pick_level_kernel(int kind, int maxa, bool warp) {
    const int m = maxa <= 1 ? 0 : maxa <= 2 ? 1 : maxa <= 4 ? 2 : 3;
#define SCFR_PICK(K) \
    (m == 0 ? k_level<K, 1, false, R> : m == 1 ? k_level<K, 2, false, R> : m == 2 ? k_level<K, 4, false, R> : k_level<K, 8, false, R>)
    switch (kind) {
        case LK_TD_AVG: return warp ? k_level<LK_TD_AVG, 1, true, R> : k_level<LK_TD_AVG, 1, false, R>;
        case LK_TD: return warp ? k_level<LK_TD, 1, true, R> : k_level<LK_TD, 1, false, R>;
        case LK_CUR: return SCFR_PICK(LK_CUR);
        case LK_OBS:
            if (warp) return k_level<LK_OBS, 1, true, R>;
            return SCFR_PICK(LK_OBS);
        default:
            if (warp) return k_level<LK_PRED, 1, true, R>;
            return SCFR_PICK(LK_PRED);
    }
#undef SCFR_PICK
}

// avg[0] update for a player without decision points (no TD levels).
template <class R>
__global__ void k_avg0(int S, const R* __restrict__ x, R* __restrict__ avg,
                       const double* __restrict__ wsched, int cap, const long long* __restrict__ tdev) {
    pdl_launch_dependents();
    pdl_wait();
    const size_t o = (size_t)blockIdx.x * S;
    const R w = (R)wsched[(size_t)blockIdx.x * cap + *tdev];
    avg[o] = dadd(dmul(w, x[o]), avg[o]);
}

__global__ void k_br(DevTree T, int lo, int hi, const double* __restrict__ g,
                     double* __restrict__ W) {
    const int j = lo + blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= hi) return;
    br_dp<LdL1>(T, j, g, W);
}

__global__ void k_br_warp(DevTree T, int lo, int hi, const double* __restrict__ g,
                          double* __restrict__ W) {
    const int j = lo + (blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (j >= hi) return;  // warp-uniform
    br_dp_warp<LdL1>(T, j, g, W, threadIdx.x & 31);
}

// br = g[0] + value of the root (the empty sequence's child sum).
__global__ void k_br_root(DevTree T, const double* __restrict__ g, const double* __restrict__ W,
                          double* out) {
    *out = dadd(g[0], child_sum<LdL1>(T.child[0], W));
}

template <class R>
__global__ void k_spmv(int rows, const int* __restrict__ indptr, const int* __restrict__ indices,
                       const R* __restrict__ data, const R* __restrict__ x, int sx,
                       R* __restrict__ out, int so, int negate, int* nonfinite) {
    pdl_launch_dependents();
    pdl_wait();
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= rows) return;
    R acc = spmv_row<LdL1>(indptr, indices, data, x + (size_t)blockIdx.y * sx, row);
    if (negate) acc = dmul(R(-1), acc);
    if (nonfinite && !isfinite(acc)) atomicOr(nonfinite, 1);
    out[(size_t)blockIdx.y * so + row] = acc;
}

__global__ void k_normalize(const double* __restrict__ a, double w, double* __restrict__ out, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = ddiv(a[i], w);
}

__global__ void k_tick(long long* tdev, unsigned long long* tl, int tl_idx) {
    pdl_launch_dependents();
    pdl_wait();
    tl_start(tl, tl_idx);
    *tdev += 1;
    tl_end(tl, tl_idx);
}

// float(t) ** e with the reference's semantics (pkg/solvers.py:82-94, :172):
// both go through libm pow(); an infinite power gives DCFR factor 1.
static double tpow(int64_t t, double e) { return std::pow((double)t, e); }
static double dfactor(int64_t t, double e) {
    const double p = tpow(t, e);
    if (std::isinf(p)) return 1.0;
    return p / (p + 1.0);
}

// Child-DP range of every sequence from dp_parent (child DPs of one sequence
// are contiguous in j, checked on the host): the first DP of each group
// records {first j, count}.
__global__ void k_derive_child(int J, const int* __restrict__ dp_parent, int2* __restrict__ child) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= J) return;
    const int p = dp_parent[j];
    if (j > 0 && dp_parent[j - 1] == p) return;
    int c = 1;
    while (j + c < J && dp_parent[j + c] == p) ++c;
    child[p] = make_int2(j, c);
}

// Uniform behaviour 1.0/n per DP block (pkg/decision_process.py:254-261),
// the RegretState initial b, for every solve of the batch.
template <class R>
__global__ void k_derive_uniform(int J, int S, int B, const int* __restrict__ seq_ptr,
                                 R* __restrict__ b) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= J) return;
    const int s0 = seq_ptr[j], n = seq_ptr[j + 1] - s0;
    const R v = ddiv(R(1), R(n));
    for (int k = 0; k < B; ++k)
        for (int a = 0; a < n; ++a) b[(size_t)k * S + s0 + a] = v;
}

// x[0] = xpost[0] = 1 (the empty sequence's mass) for every solve.
template <class R>
__global__ void k_init_root(int S, int B, R* __restrict__ x, R* __restrict__ xpost) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= B) return;
    x[(size_t)k * S] = R(1);
    xpost[(size_t)k * S] = R(1);
}

// fp32 mode: payoff values rounded to nearest fp32 once, at upload.
__global__ void k_to_f32(int n, const double* __restrict__ d, float* __restrict__ f) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) f[i] = __double2float_rn(d[i]);
}


// SCFR_TRACE=1: create-time breakdown on stderr.
static void trace_stage(const char* what) {
    static const bool on = [] {
        const char* e = std::getenv("SCFR_TRACE");
        return e && e[0] == '1';
    }();
    if (!on) return;
    static thread_local auto prev = std::chrono::steady_clock::now();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[scfr_create]   %-22s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - prev).count());
    prev = now;
}

// Coarsens the reference's levels (DPs grouped by node depth) into the
// fewest contiguous j ranges in which no DP's parent sequence belongs to a DP
// of the same range.  Every pass only needs that order (TD reads the parent
// sequence's x, OBS / PRED / BR the child DPs' V), and each DP's arithmetic is
// unchanged, so the iterates stay bit-identical while a level launch (or a
// persistent phase) covers more DPs: Liar's dice 12 / 11 -> 7 / 6 levels,
// Leduc 5 / 5 -> 4 / 4.  Greedy over the node-depth levels: level l joins the
// current range unless one of its parents is a sequence of that range
// (sequence s belongs to a DP >= start iff s >= seq_ptr[start]).
// SCFR_NO_LEVEL_MERGE=1 keeps the node-depth levels.
// lmax[l]: the largest parent sequence of node-depth level l's DPs (from
// upload_player's validation pass).
static void merge_levels(Player& P, const std::vector<int>& seq_ptr, const std::vector<int>& lmax) {
    const char* e = std::getenv("SCFR_NO_LEVEL_MERGE");  // per create (tests toggle it)
    const bool off = e && e[0] == '1';
    const int L = (int)P.lvl.size() - 1;
    if (off || L < 2) return;
    std::vector<int> merged{0};
    int start = 0;
    for (int l = 1; l < L; ++l) {
        if (lmax[l] >= seq_ptr[start]) {
            start = P.lvl[l];
            merged.push_back(start);
        }
    }
    merged.push_back(P.J);
    P.lvl.swap(merged);
}

// Per-level statistics and exact affine shapes (kernels then compute indices
// instead of loading them), reduced on the device from seq_ptr, dp_parent and
// the derived child ranges: widest / narrowest DP, child-DP references per
// level, whether every DP's parent follows p_lo + (j - j0) / pc, and whether
// every sequence's child range follows c_lo + (s - s0) * cn.  (On the host
// this walk over ~5 M DPs and sequences per player cost 2.5 ms at best and
// up to 70 ms on a busy host.)
struct LevelStat {
    int maxa, mina, par_ok, aff_ok;
    int c0, cfirst0, pc, pmin;  // pmin: smallest parent sequence of the level's DPs
    unsigned long long nc;
};

__device__ __forceinline__ int find_level(const int* __restrict__ starts, int n, int v) {
    int lo = 0, hi = n;  // last i with starts[i] <= v
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (starts[mid] <= v) lo = mid;
        else hi = mid;
    }
    return lo;
}

// Each block walks a contiguous chunk of DPs (threads strided inside it)
// and keeps per-thread partials for the level it is in; a partial reaches
// the level's record (warp-reduced, then one atomic per warp) only when the
// thread's level changes and at the end.  Levels are long j ranges, so the
// atomics per level drop from one per warp of the whole process (~70K on
// Goofspiel-5's last level: 175 us of same-address contention) to a few per
// block.
struct StatAcc {
    int l = -1, mx = 0, mn = INT32_MAX, pm = INT32_MAX, ak = 1;
    int lp = -1;
    unsigned long long nc = 0;
};
__device__ __forceinline__ void stats_flush_dp(StatAcc& a, LevelStat* st) {
    // warp-uniform call: every lane flushes its own level's partial
    const unsigned full = 0xffffffffu;
    const int l0 = __shfl_sync(full, a.l, 0);
    if (__all_sync(full, a.l == l0)) {
        const int mx = (int)__reduce_max_sync(full, (unsigned)a.mx);
        const int mn = (int)__reduce_min_sync(full, (unsigned)a.mn);
        const int pm = (int)__reduce_min_sync(full, (unsigned)a.pm);
        const int ak = (int)__reduce_and_sync(full, (unsigned)a.ak);
        if ((threadIdx.x & 31) == 0 && l0 >= 0) {
            atomicMax(&st[l0].maxa, mx);
            atomicMin(&st[l0].mina, mn);
            atomicMin(&st[l0].pmin, pm);
            if (!ak) atomicAnd(&st[l0].par_ok, 0);
        }
    } else if (a.l >= 0) {
        atomicMax(&st[a.l].maxa, a.mx);
        atomicMin(&st[a.l].mina, a.mn);
        atomicMin(&st[a.l].pmin, a.pm);
        if (!a.ak) atomicAnd(&st[a.l].par_ok, 0);
    }
    a.mx = 0;
    a.mn = INT32_MAX;
    a.pm = INT32_MAX;
    a.ak = 1;
}
__device__ __forceinline__ void stats_flush_nc(StatAcc& a, LevelStat* st) {
    const unsigned full = 0xffffffffu;
    const int l0 = __shfl_sync(full, a.lp, 0);
    if (__all_sync(full, a.lp == l0)) {
        unsigned long long v = a.nc;
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(full, v, o);
        if ((threadIdx.x & 31) == 0 && l0 >= 0 && v) atomicAdd(&st[l0].nc, v);
    } else if (a.lp >= 0 && a.nc) {
        atomicAdd(&st[a.lp].nc, a.nc);
    }
    a.nc = 0;
}

__global__ void k_level_stats_j(int J, int L, const int* __restrict__ lvl, const int* __restrict__ lvl_s0,
                                const int* __restrict__ seq_ptr, const int* __restrict__ dp_parent,
                                const int2* __restrict__ child, LevelStat* __restrict__ st) {
    const int per = (J + gridDim.x - 1) / gridDim.x;
    const int lo = blockIdx.x * per, hi = min(J, lo + per);
    StatAcc a;
    int j0 = 0, l_end = -1, p0 = 0, pc = 1, lp_lo = 0, lp_hi = -1;
    // warp-uniform trip count so the flushes' shuffles see every lane
    for (int base = lo; base < hi; base += blockDim.x) {
        const int j = base + (int)threadIdx.x;
        const bool on = j < hi;
        bool change_dp = false, change_nc = false;
        int l = a.l, lp = a.lp, n = 0, ps = 0;
        if (on) {
            if (j >= l_end) {
                l = find_level(lvl, L, j);
                j0 = lvl[l];
                l_end = l + 1 < L ? lvl[l + 1] : J;
                p0 = dp_parent[j0];
                pc = child[p0].y;
            }
            n = seq_ptr[j + 1] - seq_ptr[j];
            ps = dp_parent[j];
            if (ps != 0 && (ps < lp_lo || ps >= lp_hi)) {
                lp = find_level(lvl_s0, L, ps);
                lp_lo = lvl_s0[lp];
                lp_hi = lp + 1 < L ? lvl_s0[lp + 1] : INT32_MAX;
            }
            change_dp = l != a.l;
            change_nc = ps != 0 && lp != a.lp;
        }
        if (__any_sync(0xffffffffu, change_dp)) stats_flush_dp(a, st);
        if (__any_sync(0xffffffffu, change_nc)) stats_flush_nc(a, st);
        if (on) {
            a.l = l;
            a.mx = max(a.mx, n);
            a.mn = min(a.mn, n);
            a.pm = min(a.pm, ps);
            a.ak &= ps == p0 + (j - j0) / pc;
            if (ps != 0) {
                a.lp = lp;
                ++a.nc;
            }
        }
    }
    stats_flush_dp(a, st);
    stats_flush_nc(a, st);
}

__global__ void k_level_stats_s(int S, int L, const int* __restrict__ lvl_s0, const int2* __restrict__ child,
                                LevelStat* __restrict__ st) {
    const int q = 1 + blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= S) return;
    const int l = find_level(lvl_s0, L, q), s0 = lvl_s0[l];
    const int2 c = child[q], c0 = child[s0];
    if (!(c.y == c0.y && (c0.y == 0 || c.x == c0.x + (q - s0) * c0.y))) atomicAnd(&st[l].aff_ok, 0);
}

__global__ void k_level_stats_fin(int L, const int* __restrict__ lvl, const int* __restrict__ lvl_s0,
                                  const int* __restrict__ dp_parent, const int2* __restrict__ child,
                                  LevelStat* __restrict__ st) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= L) return;
    const int2 c0 = child[lvl_s0[l]];
    st[l].c0 = c0.y;
    st[l].cfirst0 = c0.x;
    st[l].pc = child[dp_parent[lvl[l]]].y;
}

static void level_shapes(Player& P, const std::vector<int>& seq_ptr, const std::vector<int>& dp_parent,
                         cudaStream_t s) {
    const int L = P.levels(), J = P.J, S = P.S;
    P.lvl_maxa.assign(L, 0);
    P.lvl_nc.assign(L, 0.0);
    P.lvl_pmin.assign(L, INT32_MAX);
    P.lvl_shape.assign(L, DevTree{nullptr, nullptr, nullptr});
    if (L == 0) {
        CUDA_OK(cudaStreamSynchronize(s));
        return;
    }
    std::vector<int> meta(2 * L + 1);  // lvl[0..L-1], lvl_s0[0..L-1] (+ pad)
    for (int l = 0; l < L; ++l) {
        meta[l] = P.lvl[l];
        meta[L + l] = P.lvl_s0[l];
    }
    std::vector<LevelStat> st(L, LevelStat{0, INT32_MAX, 1, 1, 0, 0, 1, INT32_MAX, 0ull});
    DevBuf<int> dmeta;
    DevBuf<LevelStat> dst;
    dmeta.alloc(meta.size());
    dst.alloc(L);
    CUDA_OK(copy_async(dmeta.p, meta.data(), meta.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    CUDA_OK(copy_async(dst.p, st.data(), L * sizeof(LevelStat), cudaMemcpyHostToDevice, s));
    if (J > 0)
        k_level_stats_j<<<std::min(grid_for(J), 1184), TPB, 0, s>>>(J, L, dmeta.p, dmeta.p + L, P.seq_ptr.p, P.dp_parent.p,
                                                 P.child.p, dst.p);
    if (S > 1) k_level_stats_s<<<grid_for(S - 1), TPB, 0, s>>>(S, L, dmeta.p + L, P.child.p, dst.p);
    k_level_stats_fin<<<grid_for(L), TPB, 0, s>>>(L, dmeta.p, dmeta.p + L, P.dp_parent.p, P.child.p, dst.p);
    CUDA_OK(cudaGetLastError());
    CUDA_OK(copy_async(st.data(), dst.p, L * sizeof(LevelStat), cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    for (int l = 0; l < L; ++l) {
        const LevelStat& t = st[l];
        P.lvl_maxa[l] = t.maxa;
        P.lvl_nc[l] = (double)t.nc;
        P.lvl_pmin[l] = t.pmin;
        DevTree& sh = P.lvl_shape[l];
        const int j0 = P.lvl[l];
        sh.j_lo = j0;
        sh.s_lo = seq_ptr[j0];
        sh.un = t.mina == t.maxa ? t.maxa : 0;
        sh.cn = t.aff_ok ? t.c0 : -1;
        sh.c_lo = t.aff_ok && t.c0 > 0 ? t.cfirst0 : 0;
        sh.pc = t.par_ok ? t.pc : 0;
        sh.p_lo = dp_parent[j0];
    }
}

// Validates the reference DecisionProcess arrays, builds the int32 device
// structure (seq_ptr, dp_parent on the host: O(J); child ranges and the
// initial behaviour on the device: O(S)) and the per-level bookkeeping.
static void upload_player(const scfr_tfsdp* p, Player& P, int B, cudaStream_t s, int slot, bool f32) {
    if (!p || p->num_seqs < 1 || p->num_decisions < 0 || p->num_nodes < 1)
        fail(SCFR_EINVAL, "bad tfsdp sizes");
    if (p->num_seqs >= (1ll << 31) / 2) fail(SCFR_EINVAL, "tfsdp too large for int32 indexing");
    if (!p->depth || !p->dp_node || !p->dp_first_seq || !p->dp_num_actions || !p->dp_parent_seq)
        fail(SCFR_EINVAL, "tfsdp has a NULL array");
    trace_stage("upload_player begin");
    const int S = (int)p->num_seqs, J = (int)p->num_decisions;
    P.S = S;
    P.J = J;
    P.max_actions = 0;
    constexpr int64_t kGrain = 1 << 16;
    HostScratch& hs = host_scratch();  // create_impl holds the arena lock
    std::vector<int>& seq_ptr = hs.sp[slot];
    std::vector<int>& dp_parent = hs.par[slot];
    resize_pinned(seq_ptr, J + 1);  // page-locked: uploaded below
    resize_pinned(dp_parent, std::max(J, 1));
    // the int32 structure is copied to the device block by block as the pass
    // produces it (the DMA of a block overlaps the conversion of the next)
    P.seq_ptr.alloc(J + 1);
    P.dp_parent.alloc(std::max(J, 1));
    int dev = 0;
    CUDA_OK(cudaGetDevice(&dev));
    constexpr int64_t kDmaBlock = 1 << 18;
    std::atomic<int> dma_err{0};  // (pool threads do not throw: checked after the pass)
    auto dma = [&](int64_t a, int64_t b) {  // [a, b) of both arrays
        if (b <= a) return;
        if (copy_async(P.seq_ptr.p + a, seq_ptr.data() + a, (b - a) * sizeof(int), cudaMemcpyHostToDevice, s) !=
                cudaSuccess ||
            copy_async(P.dp_parent.p + a, dp_parent.data() + a, (b - a) * sizeof(int), cudaMemcpyHostToDevice, s) !=
                cudaSuccess)
            dma_err = 1;
    };
    // One pass (parallel over j): per-DP checks, int32 conversion, the depth
    // order and level starts (a DP's level is its node's depth), and whether
    // dp_parent_seq is non-decreasing.  Each chunk keeps its first offending
    // j; the smallest one is reported.  Reads are sequential: dp_node rises
    // with j in the reference's breadth-first numbering, so the depth reads
    // stream too.
    struct Bad {
        int64_t j = INT64_MAX;
        int code = 0;
    };
    const int T = host_threads();
    std::vector<Bad> bad(T);
    std::vector<int> maxa_c(T, 0), order_bad(T, 0), mono_c(T, 1);
    // per chunk: level starts, and the largest parent of each run of one
    // depth (rmax[c][0]: the run continuing from the previous chunk)
    std::vector<std::vector<int>> starts(T), rmax(T);
    const int64_t N = p->num_nodes;
    parallel_chunks(J, kGrain, [&](int c, int64_t lo, int64_t hi) {
        Bad bd;
        int ma = 0, ob = 0, mono = 1;
        std::vector<int>& st = starts[c];
        std::vector<int>& rm = rmax[c];
        st.clear();
        rm.clear();
        int64_t run_max = -1;
        const int64_t* __restrict__ dfs = p->dp_first_seq;
        const int64_t* __restrict__ dna = p->dp_num_actions;
        const int64_t* __restrict__ dps = p->dp_parent_seq;
        const int64_t* __restrict__ dnd = p->dp_node;
        const int64_t* __restrict__ dep = p->depth;
        int* __restrict__ spo = seq_ptr.data();
        int* __restrict__ pao = dp_parent.data();
        // the previous DP's depth and parent (chunk boundary; its own chunk validates it)
        int64_t pd = -1, pp = INT64_MIN;
        if (lo > 0) {
            const int64_t nd = dnd[lo - 1];
            pd = nd >= 0 && nd < N ? dep[nd] : -1;
            pp = dps[lo - 1];
        }
        cudaSetDevice(dev);  // (pool thread)
        int64_t dma_from = lo, dma_next = std::min(hi, lo + kDmaBlock);
        int64_t j = lo;
        for (;;) {
            // a run of DPs at depth pd (no level start inside: nothing but
            // loads, checks and the int32 stores in the loop)
            int64_t d = pd;
            for (; j < hi; ++j) {
                if (j == dma_next) {
                    dma(dma_from, j);
                    dma_from = j;
                    dma_next = std::min(hi, j + kDmaBlock);
                }
                const int64_t fs = dfs[j];
                const int64_t expect = j == 0 ? 1 : dfs[j - 1] + dna[j - 1];
                const int64_t n = dna[j], ps = dps[j], node = dnd[j];
                const int code = fs != expect ? 1 : n < 1 ? 2 : (ps < 0 || ps >= fs) ? 3
                               : (node < 0 || node >= N) ? 4 : 0;
                if (code) {
                    bd.j = j;
                    bd.code = code;
                    break;
                }
                ma = std::max(ma, (int)n);
                spo[j] = (int)fs;
                pao[j] = (int)ps;
                mono &= ps >= pp;
                pp = ps;
                d = dep[node];
                if (d != pd || j == 0) break;
                run_max = std::max(run_max, ps);
            }
            if (bd.code) break;
            rm.push_back((int)run_max);
            if (j >= hi) break;
            if (j > 0 && d < pd) ob = 1;
            pd = d;
            run_max = pp;
            st.push_back((int)j++);
        }
        if (!bd.code) dma(dma_from, hi);
        bad[c] = bd;
        maxa_c[c] = ma;
        order_bad[c] = ob;
        mono_c[c] = mono;
    });
    {
        Bad first;
        for (const Bad& bd : bad)
            if (bd.j < first.j) first = bd;
        static const char* msg[] = {"", "dp_first_seq is not contiguous in j", "decision point without actions",
                                    "dp_parent_seq out of range or after its decision point",
                                    "dp_node out of range"};
        if (first.code) fail(SCFR_EINVAL, "%s", msg[first.code]);
        for (int m : maxa_c) P.max_actions = std::max(P.max_actions, m);
        const int64_t next = J ? p->dp_first_seq[J - 1] + p->dp_num_actions[J - 1] : 1;
        if (next != S) fail(SCFR_EINVAL, "num_seqs does not match the action counts");
    }
    seq_ptr[J] = S;
    if (dma_err) fail(SCFR_ECUDA, "structure upload failed");
    CUDA_OK(copy_async(P.seq_ptr.p + J, seq_ptr.data() + J, sizeof(int), cudaMemcpyHostToDevice, s));
    // Each parent sequence's child DPs form one contiguous group: implied
    // when dp_parent_seq is non-decreasing (Goofspiel, breadth-first
    // numbering with one DP per observation); otherwise checked with a
    // bitmap of group starts (a group start may not repeat).
    bool mono = true;
    for (int m : mono_c) mono = mono && m;
    if (!mono) {
        const size_t W = ((size_t)S + 63) / 64;
        std::unique_ptr<std::atomic<uint64_t>[]> seen(new std::atomic<uint64_t>[W]());
        std::vector<int> group_bad(T, 0);
        parallel_chunks(J, kGrain, [&](int c, int64_t lo, int64_t hi) {
            for (int64_t j = lo; j < hi; ++j) {
                const int ps = dp_parent[j];
                if (j == 0 || dp_parent[j - 1] != ps) {
                    const uint64_t bit = 1ull << (ps & 63);
                    if (seen[ps >> 6].fetch_or(bit, std::memory_order_relaxed) & bit) group_bad[c] = 1;
                }
            }
        });
        for (int c = 0; c < T; ++c)
            if (group_bad[c]) fail(SCFR_EINVAL, "child decision points of a sequence are not contiguous");
    }
    for (int c = 0; c < T; ++c)
        if (order_bad[c]) fail(SCFR_EINVAL, "decision points are not ordered by depth");
    P.lvl.clear();
    std::vector<int> lmax;
    for (int c = 0; c < T; ++c) {
        const std::vector<int>& st = starts[c];
        const std::vector<int>& rm = rmax[c];
        if (rm.empty()) continue;  // (chunk not run)
        if (!lmax.empty()) lmax.back() = std::max(lmax.back(), rm[0]);
        for (size_t i = 0; i < st.size(); ++i) {
            P.lvl.push_back(st[i]);
            lmax.push_back(rm[i + 1]);
        }
    }
    P.lvl.push_back(J);
    merge_levels(P, seq_ptr, lmax);
    trace_stage("validate+seq_ptr");
    const int L = (int)P.lvl.size() - 1;
    P.lvl_ns.assign(L, 0);
    P.lvl_nj.assign(L, 0);
    P.lvl_nc.assign(L, 0);
    P.lvl_maxa.assign(L, 0);
    P.lvl_s0.assign(L, 0);
    for (int l = 0; l < L; ++l) {
        const int j0 = P.lvl[l], j1 = P.lvl[l + 1];
        P.lvl_s0[l] = seq_ptr[j0];
        P.lvl_ns[l] = seq_ptr[j1] - seq_ptr[j0];
        P.lvl_nj[l] = j1 - j0;
    }
    P.child.alloc(S);
    P.child.zero(s);
    const size_t SB = val_slots((size_t)S * B, f32), JB = val_slots((size_t)std::max(J, 1) * B, f32);
    P.r.alloc(SB);
    P.b.alloc(SB);
    P.x.alloc(SB);
    P.xpost.alloc(SB);
    P.avg.alloc(SB);
    P.u.alloc(SB);
    P.V.alloc(JB);
    P.g.alloc(S);  // best response / evaluation scratch: always fp64
    P.W.alloc(std::max(J, 1));
    P.xbar.alloc(S);
    if (f32) P.wide.alloc(S);
    for (auto* buf : {&P.r, &P.b, &P.x, &P.xpost, &P.avg, &P.u, &P.V}) buf->zero(s);
    trace_stage("copies+allocs");
    if (J) {
        k_derive_child<<<grid_for(J), TPB, 0, s>>>(J, P.dp_parent.p, P.child.p);
        if (f32) k_derive_uniform<float><<<grid_for(J), TPB, 0, s>>>(J, S, B, P.seq_ptr.p, vals<float>(P.b));
        else k_derive_uniform<double><<<grid_for(J), TPB, 0, s>>>(J, S, B, P.seq_ptr.p, P.b.p);
    }
    if (f32) k_init_root<float><<<grid_for(B), TPB, 0, s>>>(S, B, vals<float>(P.x), vals<float>(P.xpost));
    else k_init_root<double><<<grid_for(B), TPB, 0, s>>>(S, B, P.x.p, P.xpost.p);
    CUDA_OK(cudaGetLastError());
    level_shapes(P, seq_ptr, dp_parent, s);
    trace_stage("derive+shapes+sync");
    P.h_seq_ptr = &seq_ptr;  // for the tile planner, during this create only
    P.h_dp_parent = &dp_parent;
}

// Uploads rows [row0, row0 + chunk) of the CSR (all rows unless sharded; the
// last shard may hold fewer), re-based so local row i is global row0 + i.
void derive_transpose(const DevCsr& U, const scfr_csr* UT, DevCsr& T, cudaStream_t s, bool f32);  // transpose.cu

static void upload_csr(const scfr_csr* m, DevCsr& D, cudaStream_t s, bool f32, int world = 1, int rank = 0) {
    if (!m || m->rows < 0 || m->cols < 0 || m->nnz < 0) fail(SCFR_EINVAL, "bad csr");
    if (m->nnz >= (1ll << 31)) fail(SCFR_EINVAL, "csr too large for int32 indexing");
    if (m->indptr[0] != 0 || m->indptr[m->rows] != m->nnz) fail(SCFR_EINVAL, "indptr must start at 0 and end at nnz");
    const int64_t chunk = (m->rows + world - 1) / world;
    const int64_t r0 = std::min<int64_t>(m->rows, chunk * rank);
    const int64_t r1 = std::min<int64_t>(m->rows, r0 + chunk);
    D.full_rows = (int)m->rows;
    D.row0 = (int)r0;
    D.chunk = (int)chunk;
    D.rows = (int)(r1 - r0);
    D.cols = (int)m->cols;
    const int64_t k0 = m->indptr[r0], k1 = m->indptr[r1];
    D.nnz = (int)(k1 - k0);
    trace_stage("upload_csr begin");
    // int32 conversion straight into pinned staging (parallel over rows and
    // nnz), then DMA; pageable host vectors if pinning is unavailable.
    PinnedArena& pa = pinned_arena();  // create_impl holds pa.lock and reset it
    int* ip = static_cast<int*>(pa.take((size_t)(D.rows + 1) * sizeof(int)));
    int* ix = static_cast<int*>(pa.take((size_t)std::max(D.nnz, 1) * sizeof(int)));
    double* dv = static_cast<double*>(pa.take((size_t)std::max(D.nnz, 1) * sizeof(double)));
    std::vector<int> ipv, ixv;
    const bool pinned = ip && ix && dv;
    if (!pinned) {
        ipv.resize(D.rows + 1);
        ixv.resize(std::max(D.nnz, 1));
        ip = ipv.data();
        ix = ixv.data();
        dv = nullptr;
    }
    D.indptr.alloc(D.rows + 1);
    D.indices.alloc(std::max(D.nnz, 1));
    D.data.alloc(std::max(D.nnz, 1));
    // converted block by block; with pinned staging each block's DMA is
    // issued as soon as it is written (it overlaps the next block's
    // conversion).  (restrict-qualified locals: the loops are plain streams)
    int dev = 0;
    CUDA_OK(cudaGetDevice(&dev));
    constexpr int64_t kDmaBlock = 1 << 18;
    std::atomic<int> dma_err{0};  // (pool threads do not throw: checked after the pass)
    parallel_chunks(D.rows + 1, 1 << 16, [&](int, int64_t lo, int64_t hi) {
        if (pinned) cudaSetDevice(dev);  // (pool thread)
        const int64_t* __restrict__ src = m->indptr + r0;
        int* __restrict__ dst = ip;
        for (int64_t b0 = lo; b0 < hi; b0 += kDmaBlock) {
            const int64_t b1 = std::min(hi, b0 + kDmaBlock);
            for (int64_t i = b0; i < b1; ++i) dst[i] = (int)(src[i] - k0);
            if (pinned && copy_async(D.indptr.p + b0, ip + b0, (b1 - b0) * sizeof(int), cudaMemcpyHostToDevice, s) !=
                              cudaSuccess)
                dma_err = 1;
        }
    });
    std::vector<int> badcol(host_threads(), 0);
    parallel_chunks(D.nnz, 1 << 16, [&](int c, int64_t lo, int64_t hi) {
        if (pinned) cudaSetDevice(dev);
        const int64_t* __restrict__ src = m->indices + k0;
        int* __restrict__ dst = ix;
        const int64_t cols = m->cols;
        int bad = 0;
        for (int64_t b0 = lo; b0 < hi; b0 += kDmaBlock) {
            const int64_t b1 = std::min(hi, b0 + kDmaBlock);
            for (int64_t k = b0; k < b1; ++k) {
                const int64_t col = src[k];
                bad |= col < 0 || col >= cols;
                dst[k] = (int)col;
            }
            if (dv) std::memcpy(dv + b0, m->data + k0 + b0, (b1 - b0) * sizeof(double));
            if (pinned && !bad &&  // (a bad block fails the create: nothing reads it)
                (copy_async(D.indices.p + b0, ix + b0, (b1 - b0) * sizeof(int), cudaMemcpyHostToDevice, s) !=
                     cudaSuccess ||
                 copy_async(D.data.p + b0, dv + b0, (b1 - b0) * sizeof(double), cudaMemcpyHostToDevice, s) !=
                     cudaSuccess))
                dma_err = 1;
        }
        badcol[c] = bad;
    });
    for (int b : badcol)
        if (b) fail(SCFR_EINVAL, "column index out of range");
    if (dma_err) fail(SCFR_ECUDA, "payoff upload failed");
    trace_stage("csr convert");
    if (!pinned) {
        CUDA_OK(copy_async(D.indptr.p, ip, (size_t)(D.rows + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
        if (D.nnz) {
            CUDA_OK(copy_async(D.indices.p, ix, (size_t)D.nnz * sizeof(int), cudaMemcpyHostToDevice, s));
            CUDA_OK(copy_async(D.data.p, m->data + k0, (size_t)D.nnz * sizeof(double), cudaMemcpyHostToDevice, s));
        }
    }
    if (f32) {  // the iteration's copy, rounded once (the fp64 one serves best responses)
        D.data32.alloc(std::max(D.nnz, 1));
        if (D.nnz) k_to_f32<<<grid_for(D.nnz), TPB, 0, s>>>(D.nnz, D.data.p, D.data32.p);
        CUDA_OK(cudaGetLastError());
    }
    CUDA_OK(cudaStreamSynchronize(s));
    trace_stage("csr copies+sync");
}

// Per-level bookkeeping of a CSR whose rows are rowP's sequences: indptr at
// the level boundaries (byte accounting, empty-row detection) and, for an
// unsharded matrix, the row length every row of a level shares (FuseUT::rc),
// reduced on the device from the uploaded int32 indptr.
__global__ void k_row_len_stats(int rows, int L, const int* __restrict__ lvl_s0, const int* __restrict__ lvl_end,
                                const int* __restrict__ indptr, int* __restrict__ mn, int* __restrict__ mx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    int l = -1, n = 0;
    if (i < rows && i >= lvl_s0[0]) {
        l = find_level(lvl_s0, L, i);
        if (i >= lvl_end[l]) l = -1;
        else n = indptr[i + 1] - indptr[i];
    }
    const unsigned full = 0xffffffffu;
    const int l0 = __shfl_sync(full, l, 0);
    if (__all_sync(full, l == l0)) {
        if (l0 < 0) return;
        const int a = (int)__reduce_min_sync(full, (unsigned)n), b = (int)__reduce_max_sync(full, (unsigned)n);
        if ((threadIdx.x & 31) == 0) {
            atomicMin(mn + l0, a);
            atomicMax(mx + l0, b);
        }
    } else if (l >= 0) {
        atomicMin(mn + l, n);
        atomicMax(mx + l, n);
    }
}

void device_row_ptrs(const DevCsr& D, const std::vector<int>& rows, std::vector<int64_t>& out,
                     cudaStream_t s);  // transpose.cu

// from_device: D was derived on the device (transpose.cu): its row pointers
// are read from the device copy, not from the caller's arrays.
static void csr_level_info(const scfr_csr* m, DevCsr& D, const Player& rowP, cudaStream_t s, bool unsharded,
                           bool from_device = false) {
    const int L = rowP.levels();
    D.h_rows.clear();  // level boundaries of the row player (global rows)
    D.h_ptr.clear();
    for (int l = 0; l <= L; ++l) {
        const int r = l < L ? rowP.lvl_s0[l] : rowP.S;
        if (r >= 0 && r <= m->rows && (D.h_rows.empty() || D.h_rows.back() < r)) {
            D.h_rows.push_back(r);
            if (!from_device) D.h_ptr.push_back(m->indptr[r]);
        }
    }
    if (from_device) device_row_ptrs(D, D.h_rows, D.h_ptr, s);
    D.lvl_rowc.assign(unsharded ? L : 0, -1);
    if (!unsharded || L == 0 || D.rows == 0) return;
    std::vector<int> meta(4 * L);  // lvl_s0, level ends, min (init), max (init)
    for (int l = 0; l < L; ++l) {
        meta[l] = rowP.lvl_s0[l];
        meta[L + l] = rowP.lvl_s0[l] + (int)rowP.lvl_ns[l];
        meta[2 * L + l] = INT32_MAX;
        meta[3 * L + l] = -1;
    }
    DevBuf<int> dm;
    dm.alloc(meta.size());
    CUDA_OK(copy_async(dm.p, meta.data(), meta.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    k_row_len_stats<<<grid_for(D.rows), TPB, 0, s>>>(D.rows, L, dm.p, dm.p + L, D.indptr.p, dm.p + 2 * L,
                                                    dm.p + 3 * L);
    CUDA_OK(cudaGetLastError());
    CUDA_OK(copy_async(meta.data(), dm.p, meta.size() * sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    for (int l = 0; l < L; ++l) {
        const int mn = meta[2 * L + l], mx = meta[3 * L + l];
        if (mx >= 1 && mn == mx) D.lvl_rowc[l] = mx;
    }
}

// --- NCCL (loaded at run time; only the row-sharded mode needs it) -------

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static const NcclApi& nccl() {
    static NcclApi api;
    static bool loaded = false;
    if (loaded) return api;
    // Prefer the copy already mapped into the process (torch's), else the system one.
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) fail(SCFR_ENCCL, "cannot load libnccl.so.2: %s", dlerror());
    auto sym = [&](const char* name) {
        void* p = dlsym(lib, name);
        if (!p) fail(SCFR_ENCCL, "libnccl lacks %s", name);
        return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.CommSplit = reinterpret_cast<decltype(api.CommSplit)>(sym("ncclCommSplit"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    loaded = true;
    return api;
}

#define NCCL_OK(expr)                                                                     \
    do {                                                                                  \
        ncclResult_t _r = (expr);                                                         \
        if (_r != ncclSuccess) ::scfr::fail(SCFR_ENCCL, "%s failed: %s", #expr,          \
                                            nccl().GetErrorString(_r));                   \
    } while (0)

// In-place all-gather of the per-rank row slices of a vector laid out as
// world x chunk (padded) on the handle's stream.
static void allgather_rows(scfr_handle* h, double* full, int chunk) {
    NCCL_OK(nccl().AllGather(full + (size_t)h->rank * chunk, full, (size_t)chunk, ncclDouble,
                             (ncclComm_t)h->comm, h->stream));
}

// Subtree mode: every rank broadcasts its own range [b[r], b[r+1]) of `buf`
// (elements of `esize` bytes) in place, one NCCL group on `s`.
static void broadcast_ranges(scfr_handle* h, void* buf, size_t esize, const std::vector<int>& b, cudaStream_t s) {
    // the second stream of an overlapped body has its own communicator: each
    // communicator's collectives are issued in one stream order on every rank
    ncclComm_t comm = (ncclComm_t)(s == h->stream2 && h->comm2 ? h->comm2 : h->comm);
    char* base = static_cast<char*>(buf);
    const ncclDataType_t ty = esize == 8 ? ncclDouble : ncclFloat;
    for (int r = 0; r < h->world; ++r) {
        const size_t cnt = (size_t)(b[r + 1] - b[r]);
        if (cnt) {
            void* p = base + (size_t)b[r] * esize;
            NCCL_OK(nccl().Broadcast(p, p, cnt, ty, r, comm, s));
        }
    }
}

// Subtree mode, before a read: the other ranks' subtree state (every state
// vector of every forest level) broadcast by its owners, so that the handle
// holds the one-GPU state.
static void gather_subtrees(scfr_handle* h) {
    if (!h->subtree || !h->sub_stale || h->sub_sim > 1 || h->sub_view >= 0) return;
    NCCL_OK(nccl().GroupStart());
    for (int k = 0; k < 2; ++k) {
        Player& P = h->P[k];
        for (int l = h->sub_ls[k]; l >= 0 && l < P.levels(); ++l) {
            for (DevBuf<double>* v : {&P.r, &P.b, &P.x, &P.xpost, &P.avg, &P.u, &P.bcur})
                if (v->n) broadcast_ranges(h, v->p, sizeof(double), h->sub_sb[k][l], h->stream);
            broadcast_ranges(h, P.V.p, sizeof(double), h->sub_jb[k][l], h->stream);
        }
    }
    NCCL_OK(nccl().GroupEnd());
    h->sub_stale = false;
}

// --- per-iteration launch sequence --------------------------------------

// Algorithmic (compulsory) HBM bytes of one launch, fp64 values / int32
// indices, every array touched once (DESIGN.md §4 has the derivation).
// The player's tree with level l's affine shape attached (SCFR_NO_SHAPE=1:
// always load indices, for A/B measurements).
static DevTree shaped_tree(const Player& P, int l) {
    DevTree t = P.tree();
    static const bool off = [] {
        const char* e = std::getenv("SCFR_NO_SHAPE");
        return e && e[0] == '1';
    }();
    if (!off && l >= 0 && l < P.levels()) {
        const DevTree& sh = P.lvl_shape[l];
        t.j_lo = sh.j_lo;
        t.s_lo = sh.s_lo;
        t.un = sh.un;
        t.cn = sh.cn;
        t.c_lo = sh.c_lo;
        t.pc = sh.pc;
        t.p_lo = sh.p_lo;
    }
    return t;
}

// The deepest level is single-action DPs into end nodes (affine, no child
// DPs) and all its DPs hang under the level above (kernels.cuh leaf_note).
bool leaf_single(const scfr_handle* h, const Player& P) {
    const int L = P.levels();
    if (!h->leaf_skip || L < 2) return false;
    const DevTree& sh = P.lvl_shape[L - 1];
    return sh.un == 1 && sh.cn == 0 && P.lvl_nc[L - 2] == P.lvl_nj[L - 1];
}

// Forced leaf sequences carry copies of their parent sequence's x, xpost
// and avg, bit for bit: x_leaf = 1.0 * x_parent, and avg_leaf accumulates
// w * x_parent from zero exactly as avg_parent does.  With h->leaf_x the
// level engine does not run those top-down launches; the opponent's payoff
// rows read the parent's column instead (DevCsr::iter_indices) and reads
// restore the copies here.  v: one solve's seq-indexed vector.
template <class R>
__global__ void k_expand_leaf(DevTree T, int j_lo, int n, int shift, R* __restrict__ v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int j = j_lo + i;
    v[j + shift] = v[parent_of<LdL1>(T, j)];
}

// The iteration's column indices of M when the column player's deepest level
// is a forced leaf level: leaf columns read the parent sequence instead
// (whose x / xpost equals the leaf's, k_expand_leaf), so that level's
// top-down launches can be skipped.  Built on the device from this rank's
// int32 indices.
__global__ void k_leaf_columns(int nnz, const int* __restrict__ ix, int* __restrict__ out, DevTree T,
                               int s_lo, int n, int shift) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nnz) return;
    const int c = ix[k];
    out[k] = c >= s_lo && c < s_lo + n ? parent_of<LdL1>(T, c - shift) : c;
}

static void build_iter_indices(scfr_handle* h, DevCsr& D, const Player& colP) {
    const int l = colP.levels() - 1;
    const int j0 = colP.lvl[l], n = colP.lvl[l + 1] - j0;
    const int s_lo = colP.lvl_shape[l].s_lo, shift = s_lo - j0;
    D.indices_iter.alloc(std::max(D.nnz, 1));
    if (D.nnz)
        k_leaf_columns<<<grid_for(D.nnz), TPB, 0, h->stream>>>(D.nnz, D.indices.p, D.indices_iter.p,
                                                               shaped_tree(colP, l), s_lo, n, shift);
    CUDA_OK(cudaGetLastError());
}

// Player 2's structurally empty payoff rows hold u = -1.0 * 0.0 = -0.0 after
// the first iteration (the reference's scale(-1, Uᵀx)); with u_empty_skip
// nothing recomputes them, so the first scfr_step writes the constant.
template <class R>
__global__ void k_fill_rows(R* __restrict__ u, int S, int B, int lo, int n, R v) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)n * B) return;
    u[(i / n) * S + lo + i % n] = v;
}

// Structure bytes are counted only where the kernel loads them: an affine
// level (lvl_shape) computes seq_ptr / child / dp_parent arithmetically.
struct LevelBytes {  // v: bytes per value (8 fp64, 4 in the fp32 mode)
    static double seqptr(const Player& P, int l) { return P.lvl_shape[l].un > 0 ? 0.0 : 4.0 * P.lvl_nj[l]; }
    static double child(const Player& P, int l) { return P.lvl_shape[l].cn >= 0 ? 0.0 : 8.0 * P.lvl_ns[l]; }
    static double parent(const Player& P, int l) { return P.lvl_shape[l].pc > 0 ? 0.0 : 4.0 * P.lvl_nj[l]; }
    // single-action levels touch no r / b (kernels.cuh single_action_note)
    static bool single(const Player& P, int l) { return P.lvl_shape[l].un == 1; }
    static double obs(const Player& P, int l, bool rm, double v = 8) {
        const double ns = P.lvl_ns[l], nj = P.lvl_nj[l], nc = P.lvl_nc[l];
        // u, b read; r RMW; [b write]; V write; child V reads; structure
        const double rb = single(P, l) ? 0.0 : (3 + (rm ? 1 : 0)) * v * ns;
        return v * ns + rb + v * nj + v * nc + seqptr(P, l) + child(P, l);
    }
    static double pred(const Player& P, int l, double v = 8) {
        const double ns = P.lvl_ns[l], nj = P.lvl_nj[l], nc = P.lvl_nc[l];
        // m, b, r read; b write; V write; child V reads; structure
        return (single(P, l) ? 1 : 4) * v * ns + v * nj + v * nc + seqptr(P, l) + child(P, l);
    }
    static double td(const Player& P, int l, bool avg, double v = 8) {
        const double ns = P.lvl_ns[l], nj = P.lvl_nj[l];
        // b read, x write, [avg RMW]; parent x; structure
        return ((single(P, l) ? 1 : 2) + (avg ? 2 : 0)) * v * ns + v * nj + seqptr(P, l) + parent(P, l);
    }
    static double cur(const Player& P, int l, double v = 8) {  // r read, x write; parent x; structure
        return (single(P, l) ? 1 : 2) * v * P.lvl_ns[l] + v * P.lvl_nj[l] + seqptr(P, l) + parent(P, l);
    }
    static double spmv(const DevCsr& M, double v = 8) {
        return 4.0 * (M.rows + 1) + (4.0 + v) * M.nnz + v * M.cols + v * M.rows;
    }
};

KParams LaunchBase::kparams(bool do_rm) const {
    return KParams{h->wsched.p, h->pfsched.p, h->nfsched.p, h->cap, h->tdev.p,
                   post_of(h->variant), do_rm ? 1 : 0, h->variant == SCFR_PCFR_PLUS ? 1 : 0,
                   h->nonfinite.p, tl, (int)count, tofs};
}

struct Launcher : LaunchBase {
    explicit Launcher(scfr_handle* hh) : LaunchBase{hh} {}
    bool cur_top_ = false;  // player 1's current-strategy pass: its deeper top (h->top_cur)
    // body_t: player 2's observe levels above its first launch go to obs_side
    // (event ev_lv[l] after level l), and its PRED / TD wait for them
    cudaStream_t obs_side = nullptr;
    bool side_lv[scfr_handle::kSideLevels] = {};
    int side_last = -1;
    bool pred_gate = false;
    // predictive alt mode: player 1's OBS regret-matches into bcur (instead
    // of b, which PRED still needs) and CUR reads it as a plain TD
    void* bcur_ = nullptr;
    // OBS: the forced leaf level of player k is computed inside the group
    // launch of the level above (TaskT::lfu), set per pass by iteration_t
    bool lf_[2] = {false, false};
    bool leaf_fusable(const Player& P) const {
        if (!h->leaf_fuse || !fuse_spmv() || !leaf_single(P) || !h->group) return false;
        const int l = P.levels() - 2;
        if (l < 1) return false;  // (level 0 never runs in group mode)
        const DevTree& sh = P.lvl_shape[l];
        return sh.un >= 2 && sh.un <= 16 && P.lvl_nj[l] > h->group_nj && !warp_level(h, P, l) &&
               !(h->pipe && ((h->pipe_kinds >> LK_OBS) & 1));
    }
    // parent pairs: the level (and pass kind) each player's last pair launch
    // already computed
    int paired_[2] = {-1, -1}, paired_kind_[2] = {-1, -1};
    // Level l can carry its parent level l-1 in one group launch: both
    // uniform group-width levels, and the parents' children are exactly level
    // l, contiguous, the same number per parent (opt-in SCFR_PAIR=1: a warp's
    // block is one serial chain of rounds, 164 vs 145 us on Goofspiel-5).
    bool pair_ok(const Player& P, int l) const {
        if (!h->pair || l < 1 || l >= P.levels()) return false;
        const DevTree& c = P.lvl_shape[l];
        const DevTree& p = P.lvl_shape[l - 1];
        if (c.un < 2 || c.un > 16 || p.un < 2 || p.un > 16 || p.cn < 1) return false;
        if (p.c_lo != P.lvl[l] || (double)p.un * p.cn * P.lvl_nj[l - 1] != P.lvl_nj[l]) return false;
        return true;
    }
    // first level of player P that top-down passes launch (the top's are not)
    int first_level(const Player& P) const {
        const int k = &P == &h->P[0] ? 0 : 1;
        return h->top[k].on ? h->top[k].ls : 0;
    }


    // Task for level l of player P (l outside [0, L) -> empty task).
    template <class R>
    static TaskT<R> task(Player& P, int l, const R* u, R* x) {
        TaskT<R> t{};
        t.T = shaped_tree(P, l);
        t.S = P.S;
        t.J = P.J;
        t.u = u;
        t.r = vals<R>(P.r);
        t.b = vals<R>(P.b);
        t.x = x;
        t.avg = vals<R>(P.avg);
        t.V = vals<R>(P.V);
        if (l >= 0 && l < P.levels()) {
            t.lo = P.lvl[l];
            t.n = P.lvl[l + 1] - P.lvl[l];
        }
        return t;
    }
    // Resident CTAs of a level kernel on the whole GPU (cached per handle),
    // or num_sms * SCFR_WAVE_CTAS when that is set.
    template <class K>
    int resident_ctas(K kern) const {
        if (h->wave_ctas_env) return h->num_sms * h->wave_ctas;
        const void* key = reinterpret_cast<const void*>(kern);
        for (const auto& e : h->tile_occ)
            if (e.first == key) return e.second * h->num_sms;
        int occ = 0;
        CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, TPB, 0));
        occ = std::max(occ, 1);
        h->tile_occ.emplace_back(key, occ);
        return occ * h->num_sms;
    }

    // The deepest level is single-action DPs into end nodes (affine, no child
    // DPs) and all its DPs hang under the level above (kernels.cuh leaf_note).
    bool leaf_single(const Player& P) const { return scfr::leaf_single(h, P); }
    // All payoff rows of level l's sequences are empty (level 0: with row 0).
    static bool rows_empty(const Player& P, int l, const DevCsr& M) {
        if (l < 0 || l >= P.levels()) return false;
        const int s0 = l == 0 ? 0 : P.lvl_s0[l], s1 = P.lvl_s0[l] + (int)P.lvl_ns[l];
        return M.ptr_at(s1) - M.ptr_at(s0) == 0 && M.ptr_at(s1) >= 0;
    }

    // SpMV fused into OBS unless a player has no decision points (then no
    // OBS level would produce its u) or SCFR_NO_FUSE=1.
    bool fuse_spmv() const { return h->fuse && h->P[0].J > 0 && h->P[1].J > 0; }

    // Top-down passes go warp-per-DP on levels with >= kWideActions actions.
    static bool wide(const Player& P, int l) {
        return l >= 0 && l < P.levels() && P.lvl_maxa[l] >= kWideActions;
    }
    bool fat(const Player& P, int l) const {
        return l >= 0 && l < P.levels() && warp_level(h, P, l);
    }

    // Rows of level l all of one length: index them without indptr.
    template <class R>
    static void set_row_shape(FuseUT<R>& f, const DevCsr& M, const Player* P, int l) {
        if (!P || l < 0 || l >= P->levels() || l >= (int)M.lvl_rowc.size() || M.lvl_rowc[l] < 1) return;
        f.rc = M.lvl_rowc[l];
        f.rs0 = P->lvl_s0[l];
        f.rk0 = (int)M.ptr_at(P->lvl_s0[l]);
    }

    // Payoff values in the handle's arithmetic (fp32 copy in the fp32 mode).
    template <class R>
    const R* payoff_data(const DevCsr& M) const {
        if constexpr (sizeof(R) == 4) return M.data32.p;
        else return M.data.p;
    }

    // One launch over level la of A and level lb of Bp (either may be absent);
    // subtree mode: a bottom-up launch of a split level is followed by the
    // exchange of the roots' V (also on a rank whose own range is empty).
    template <class R>
    void level(int lk, int kk, Player* A, int la, Player* Bp, int lb, const R* ua, const R* ub,
               R* xa, R* xb, bool do_rm, const R* vca = nullptr, const R* vcb = nullptr, int skipa = 0,
               int skipb = 0) {
        // SCFR_SUBTREE_SIM=W at world 1: a forest level runs as W launches, one
        // per rank range of a W-rank plan (tests the range restriction on one GPU)
        const bool forest = h->subtree && ((A && la >= 0 && la >= h->sub_ls[0]) || (Bp && lb >= 0 && lb >= h->sub_ls[1]));
        const int parts = forest && h->sub_sim > 1 ? h->sub_sim : 1;
        for (int part = 0; part < parts; ++part)
            level_launch<R>(lk, kk, A, la, Bp, lb, ua, ub, xa, xb, do_rm, vca, vcb, skipa, skipb, part);
        if (!h->subtree || h->sub_sim > 1 || h->sub_view >= 0 || (lk != LK_OBS && lk != LK_PRED)) return;
        const bool ea = A && la >= 0 && la == h->sub_ls[0];
        const bool eb = Bp && lb >= 0 && lb == h->sub_ls[1];
        if (!ea && !eb) return;
        cudaStream_t s = st ? st : h->stream;
        NCCL_OK(nccl().GroupStart());
        auto vbuf = [&](Player* P) { return lk == LK_PRED && P->PV.n ? P->PV.p : P->V.p; };
        if (ea) broadcast_ranges(h, vbuf(A), sizeof(R), h->sub_jb[0][la], s);
        if (eb) broadcast_ranges(h, vbuf(Bp), sizeof(R), h->sub_jb[1][lb], s);
        NCCL_OK(nccl().GroupEnd());
    }

    template <class R>
    void level_launch(int lk, int kk, Player* A, int la, Player* Bp, int lb, const R* ua, const R* ub,
                      R* xa, R* xb, bool do_rm, const R* vca, const R* vcb, int skipa, int skipb, int part) {
        // a level already computed by its child level's pair launch
        if (A && la >= 0 && la == paired_[0] && lk == paired_kind_[0]) la = -1;
        if (Bp && lb >= 0 && lb == paired_[1] && lk == paired_kind_[1]) lb = -1;
        TaskT<R> t0 = A ? task<R>(*A, la, ua, xa) : TaskT<R>{};
        TaskT<R> t1 = Bp ? task<R>(*Bp, lb, ub, xb) : TaskT<R>{};
        t0.Vc = vca;
        t1.Vc = vcb;
        if (lk == LK_PRED) {  // PRED's values in their own buffer (PV) when there is one
            if (A && A->PV.n) t0.V = vals<R>(A->PV);
            if (Bp && Bp->PV.n) t1.V = vals<R>(Bp->PV);
        }
        if (bcur_ && A == &h->P[0]) {
            if (lk == LK_OBS) t0.bw = static_cast<R*>(bcur_);
            else if (lk == LK_TD) t0.b = static_cast<R*>(bcur_);
        }
        t0.skip_v = skipa;
        t1.skip_v = skipb;
        // the top-down launch of level ls of a player with a top recomputes the top
        auto attach_top = [&](TaskT<R>& t, Player* P, int l) {
            if (!P || (lk != LK_TD_AVG && lk != LK_TD)) return;
            const TopPlayer& tp = cur_top_ && P == &h->P[0] ? h->top_cur : h->top[P == &h->P[0] ? 0 : 1];
            if (tp.on && l == tp.ls) t.top = tp.info.p;
        };
        attach_top(t0, A, la);
        attach_top(t1, Bp, lb);
        if (h->subtree) {  // this rank's DPs of a forest level
            const int rk = h->sub_sim > 1 ? part : h->sub_view >= 0 ? h->sub_view : h->rank;
            auto own = [&](TaskT<R>& t, Player* P, int l) {
                const int k = P == &h->P[0] ? 0 : 1;
                if (part > 0) t.top = nullptr;  // (simulated ranks: the first part wrote the top)
                if (!P || l < 0 || l >= P->levels()) return;
                if (l < h->sub_ls[k]) {
                    if (part > 0) t.n = 0;  // the trunk runs once
                    return;
                }
                const std::vector<int>& jb = h->sub_jb[k][l];
                t.lo = jb[rk];
                t.n = jb[rk + 1] - t.lo;
            };
            own(t0, A, la);
            own(t1, Bp, lb);
        }
        const bool fused_here = lk == LK_OBS && fuse_spmv();
        if (t0.n == 0 && t1.n == 0) return;
        const bool fused = fused_here;
        if (fused) {  // u1 = U x2 and u2 = -Uᵀ x1 (x1' in alt mode) computed inside OBS
            Player& P1 = h->P[0];
            Player& P2 = h->P[1];
            t0.fu = FuseUT<R>{h->U.indptr.p, h->U.iter_indices(), payoff_data<R>(h->U), vals<R>(P2.x), 0};
            t0.fu_sx = P2.S;
            t1.fu = FuseUT<R>{h->UT.indptr.p, h->UT.iter_indices(), payoff_data<R>(h->UT),
                              h->mode == SCFR_MODE_ALT ? vals<R>(P1.xpost) : vals<R>(P1.x), 1};
            t1.fu_sx = P1.S;
            if (h->affine_rows) {
                set_row_shape(t0.fu, h->U, A, la);
                set_row_shape(t1.fu, h->UT, Bp, lb);
            }
        }
        // a forced leaf level computed inside this launch (leaf_fusable)
        double leaf_bytes = 0.0;
        if (lk == LK_OBS && fused) {
            auto attach_leaf = [&](TaskT<R>& t, Player* P, int l) {
                const int k = P == &h->P[0] ? 0 : 1;
                if (!P || !lf_[k] || l != P->levels() - 2) return;
                const DevCsr& M = k == 0 ? h->U : h->UT;
                const int ll = P->levels() - 1;
                t.lfu = FuseUT<R>{M.indptr.p, M.iter_indices(), payoff_data<R>(M),
                                  k == 0 ? vals<R>(h->P[1].x)
                                         : (h->mode == SCFR_MODE_ALT ? vals<R>(h->P[0].xpost) : vals<R>(h->P[0].x)),
                                  k};
                if (h->affine_rows) set_row_shape(t.lfu, M, P, ll);
                t.lshift = P->lvl_shape[ll].s_lo - P->lvl_shape[ll].j_lo;
                t.tu_leaf = vals<R>(P->u);
                t.fu_sx = h->P[1 - k].S;
                t.Vc = nullptr;
                const double ns = P->lvl_ns[ll];
                const double nnz = (double)(M.ptr_at(P->lvl_s0[ll] + (int)ns) - M.ptr_at(P->lvl_s0[ll]));
                const bool shaped = h->affine_rows && ll < (int)M.lvl_rowc.size() && M.lvl_rowc[ll] >= 1;
                // the leaf's rows (indptr, indices + data, x gathers) and its u writes
                // replace the launch's reads of the leaf utilities
                leaf_bytes += (shaped ? 0.0 : 4.0 * (ns + 1)) + (4.0 + sizeof(R)) * nnz + sizeof(R) * nnz;
            };
            attach_leaf(t0, A, la);
            attach_leaf(t1, Bp, lb);
        }
        // levels whose payoff rows are all empty: u is a constant ±0.0
        // (kernels.cuh ld_u), neither computed nor read
        bool empty[2] = {false, false};
        if ((lk == LK_OBS || lk == LK_PRED) && h->u_empty_skip) {
            empty[0] = A && rows_empty(*A, la, h->U);
            empty[1] = Bp && rows_empty(*Bp, lb, h->UT);
            if (empty[0]) {
                t0.u = nullptr;
                t0.fu = FuseUT<R>{};
            }
            if (empty[1]) {
                t1.u = nullptr;
                t1.fu = FuseUT<R>{};
            }
        }
        const bool warp = (lk == LK_OBS || lk == LK_PRED) ? (A && fat(*A, la)) || (Bp && fat(*Bp, lb))
                          : (lk == LK_TD_AVG || lk == LK_TD) && h->td_warp &&
                                ((A && wide(*A, la)) || (Bp && wide(*Bp, lb)));
        // group mode: big affine levels of 2..16 actions (both tasks, if two)
        auto groupable = [&](const Player* P, int l) {
            return !P || l < 0 || l >= P->levels() ||
                   (l > 0 && P->lvl_shape[l].un >= 2 && P->lvl_shape[l].un <= 16 && P->lvl_nj[l] > h->group_nj);
        };
        const bool group = h->group && !warp && (A || Bp) && groupable(A, la) && groupable(Bp, lb) &&
                           !(A && la == 0) && !(Bp && lb == 0);
        auto group_per = [&](const Player* P, int l) {
            return P && l >= 0 && l < P->levels() ? (TPB / 32) * (32 / P->lvl_shape[l].un) : TPB;
        };
        const int per = warp ? TPB / 32 : TPB;
        // about one resident wave per task; the blocks grid-stride over the DPs
        const int cap = h->num_sms * h->wave_ctas;
        const int per0 = group ? group_per(A, la) : per, per1 = group ? group_per(Bp, lb) : per;
        t0.nblk = std::min((t0.n + per0 - 1) / per0, cap);
        t1.nblk = std::min((t1.n + per1 - 1) / per1, cap);
        int maxa = 1;
        double bytes = 0.0;
        const double v = sizeof(R);
        for (int k = 0; k < 2; ++k) {
            Player* P = k == 0 ? A : Bp;
            const int l = k == 0 ? la : lb;
            if (!P || l < 0 || l >= P->levels()) continue;
            maxa = std::max(maxa, P->lvl_maxa[l]);
            switch (lk) {
                case LK_TD_AVG: bytes += LevelBytes::td(*P, l, true, v); break;
                case LK_TD: bytes += LevelBytes::td(*P, l, false, v); break;
                case LK_CUR: bytes += LevelBytes::cur(*P, l, v); break;
                case LK_OBS: bytes += LevelBytes::obs(*P, l, do_rm, v) - ((k == 0 ? skipa : skipb) ? v * P->lvl_nj[l] : 0.0); break;
                default: bytes += LevelBytes::pred(*P, l, v); break;
            }
            if (empty[k]) {  // no u read / write, no row pointers
                bytes -= v * P->lvl_ns[l];
                continue;
            }
            if (fused) {  // this level's payoff rows; u is written instead of read
                const DevCsr& M = k == 0 ? h->U : h->UT;
                const int s0 = P->lvl_s0[l], s1 = s0 + (int)P->lvl_ns[l];
                const double nnz = (double)(M.ptr_at(s1) - M.ptr_at(s0));
                const bool shaped = h->affine_rows && l < (int)M.lvl_rowc.size() && M.lvl_rowc[l] >= 1;
                bytes += (shaped ? 0.0 : 4.0 * (s1 - s0 + 1)) + (4.0 + v) * nnz + v * nnz;
            }
        }
        // both tasks of a group launch share one width, or the kernel reads it
        int gun = 0;
        if (group) {
            const int ua = A && la >= 0 && la < A->levels() ? A->lvl_shape[la].un : -1;
            const int ub = Bp && lb >= 0 && lb < Bp->levels() ? Bp->lvl_shape[lb].un : -1;
            gun = ua < 0 ? ub : ub < 0 ? ua : ua == ub ? ua : 0;
        }
        bytes += leaf_bytes;
        const LevelKernelT<R> kern = group ? pick_group_kernel<R>(lk, gun) : pick_level_kernel<R>(lk, maxa, warp);
        // parent pairs: a bottom-up group launch also computes the parent level
        if (group && (lk == LK_OBS || lk == LK_PRED)) {
            auto pair = [&](TaskT<R>& t, Player* P, int l, int skip_v, const R* u) {
                if (!P || !pair_ok(*P, l) || skip_v) return;
                const DevTree& ps = P->lvl_shape[l - 1];
                const int G = 32 / P->lvl_shape[l].un, pG = 32 / ps.un, C = ps.un * ps.cn;
                int pb = pG;
                for (int q = pG; q >= 1; --q)
                    if ((q * C) % G == 0) {
                        pb = q;
                        break;
                    }
                t.pair = 1;
                t.plo = P->lvl[l - 1];
                t.pn = P->lvl[l] - P->lvl[l - 1];
                t.pblk = pb;
                t.pch = C;
                t.PT = shaped_tree(*P, l - 1);
                t.pu = u;
                t.pfu = FuseUT<R>{};
                const DevCsr& M = P == &h->P[0] ? h->U : h->UT;  // the player's payoff rows
                const bool empty = h->u_empty_skip && rows_empty(*P, l - 1, M);
                if (empty) t.pu = nullptr;
                if (lk == LK_OBS && fused && !empty) {
                    t.pfu = t.fu.ip ? t.fu : FuseUT<R>{M.indptr.p, M.iter_indices(), payoff_data<R>(M),
                                                        P == &h->P[0] ? vals<R>(h->P[1].x)
                                                                      : (h->mode == SCFR_MODE_ALT ? vals<R>(h->P[0].xpost)
                                                                                                  : vals<R>(h->P[0].x)),
                                                        P == &h->P[0] ? 0 : 1};
                    t.pfu.rc = 0;
                    if (h->affine_rows) set_row_shape(t.pfu, M, P, l - 1);
                    if (!t.fu.ip) t.fu_sx = P == &h->P[0] ? h->P[1].S : h->P[0].S;
                }
                const int k = P == &h->P[0] ? 0 : 1;
                paired_[k] = l - 1;
                paired_kind_[k] = lk;
                bytes += lk == LK_OBS ? LevelBytes::obs(*P, l - 1, do_rm, sizeof(R)) : LevelBytes::pred(*P, l - 1, sizeof(R));
                // the parents of a block are processed by the warp of their children
                t.nblk = std::min(t.nblk, std::max(1, (t.pn + t.pblk * (TPB / 32) - 1) / (t.pblk * (TPB / 32))));
            };
            pair(t0, A, la, skipa, ua);
            pair(t1, Bp, lb, skipb, ub);
        }
        // big affine group levels: the cp.async-pipelined variant (one width,
        // affine children / parents, no top, no pair)
        size_t psmem = 0;
        LevelKernelT<R> pkern = nullptr;
        if (group && h->pipe && gun >= 2 && gun <= 4 && ((h->pipe_kinds >> lk) & 1)) {
            auto pipeable = [&](const TaskT<R>& t, Player* P, int l) {
                if (!P || l < 0 || l >= P->levels()) return true;  // absent task
                const DevTree& sh = P->lvl_shape[l];
                if (P->lvl_nj[l] < h->pipe_nj || t.top || t.pair || t.skip_v) return false;
                if (lk == LK_OBS || lk == LK_PRED) return sh.cn >= 0 && sh.cn <= 8;
                return sh.pc > 0;
            };
            if (pipeable(t0, A, la) && pipeable(t1, Bp, lb) && (t0.n > 0 || t1.n > 0)) {
                int cn = 0;
                if (lk == LK_OBS || lk == LK_PRED)
                    for (int k = 0; k < 2; ++k) {
                        Player* P = k == 0 ? A : Bp;
                        const int l = k == 0 ? la : lb;
                        if (P && l >= 0 && l < P->levels()) cn = std::max(cn, P->lvl_shape[l].cn);
                    }
                // both tasks index their slots with the widest child count
                if (lk == LK_OBS || lk == LK_PRED) {
                    const int ca = A && la >= 0 && la < A->levels() ? A->lvl_shape[la].cn : cn;
                    const int cb = Bp && lb >= 0 && lb < Bp->levels() ? Bp->lvl_shape[lb].cn : cn;
                    if (ca != cb) cn = -1;
                }
                if (cn >= 0) {
                    psmem = (size_t)(TPB / 32) * kPipe * 32 * (3 + cn) * sizeof(R);
                    switch (gun) {
                        case 2: pkern = pick_pipe_kernel_n<2, R>(lk); break;
                        case 3: pkern = pick_pipe_kernel_n<3, R>(lk); break;
                        default: pkern = pick_pipe_kernel_n<4, R>(lk); break;
                    }
                }
            }
        }
        // overlapped body: only stream B's small (latency-bound) launches jump
        // the queue; its big ones share the SMs with NEXT1's (SCFR_PRIO_NJ)
        struct PrioGuard {
            int& p;
            int saved;
            ~PrioGuard() { p = saved; }
        } pg{prio, prio};
        if (prio && (int64_t)t0.n + t1.n > h->prio_nj) prio = 0;
        if (pkern) {
            int occ = 0;
            CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pkern, TPB, psmem));
            const int wave = std::max(1, occ) * h->num_sms;
            t0.nblk = std::min(t0.nblk, wave);
            t1.nblk = std::min(t1.nblk, wave);
            const KParams kp = kparams(do_rm);
            launch(kk, bytes, [&] { run_ex(pkern, dim3(t0.nblk + t1.nblk, h->B), TPB, psmem, t0, t1, kp); });
            return;
        }
        // grid-stride tasks: cap each at one resident wave of this kernel
        const int wave = resident_ctas(kern);
        t0.nblk = std::min(t0.nblk, wave);
        t1.nblk = std::min(t1.nblk, wave);
        const KParams kp = kparams(do_rm);
        launch(kk, bytes, [&] {
            run(kern, dim3(t0.nblk + t1.nblk, h->B), t0, t1, kp);
        });
    }

    // out[row0 + i] = (±) row i of M applied to x (this rank's rows), then in
    // the row-sharded mode the slices are all-gathered into the full vector.
    template <class R>
    void spmv(const DevCsr& M, const R* x, int sx, R* out, int so, bool neg) {
        launch(KK_SPMV, LevelBytes::spmv(M, sizeof(R)), [&] {
            dim3 grid(grid_for(M.rows), h->B);
            run(k_spmv<R>, grid, M.rows, (const int*)M.indptr.p, (const int*)M.iter_indices(),
                payoff_data<R>(M), x, sx, out + M.row0, so, neg ? 1 : 0, h->nonfinite.p);
        });
        if constexpr (sizeof(R) == 8)
            if (h->rowshard()) allgather_rows(h, out, M.chunk);
    }

    void iteration() {
        if (h->engine == SCFR_ENGINE_TILED) {
            tiled_iteration(*this);
            return;
        }
        if (h->f32) iteration_t<float>();
        else iteration_t<double>();
    }

    template <class R>
    void iteration_t() {
        next_part<R>(true, true);
        observe_part<R>(true, true);
        tick();
    }

    void tick() { launch(KK_TICK, 0.0, [&] { run1(k_tick, dim3(1), h->tdev.p, tl, (int)count); }); }

    // next_strategy of the chosen players (independent): PRED deep -> shallow,
    // then TD + average shallow -> deep, two players sharing launches.
    template <class R>
    void next_part(bool p1, bool p2) {
        Player& A = h->P[0];
        Player& Bp = h->P[1];
        Player* pa = p1 ? &A : nullptr;
        Player* pb = p2 ? &Bp : nullptr;
        R *Au = vals<R>(A.u), *Bu = vals<R>(Bp.u), *Ax = vals<R>(A.x), *Bx = vals<R>(Bp.x);
        const bool pr = predictive(h->variant);
        const int LA = A.levels(), LB = Bp.levels(), L = std::max(LA, LB);
        const int fa = first_level(A), fb = first_level(Bp);  // the top's levels are not launched
        auto skip = [](int l, int f) { return l < f ? -1 : l; };
        if (pr) {
            // a deepest level of forced moves into end nodes needs no PRED
            // launch: its parent level reads the prediction itself (leaf_note)
            const bool sa = leaf_single(A), sb = leaf_single(Bp);
            auto vc = [](const Player& P, const R* u) {  // u shifted to index by the leaf level's DP id
                const DevTree& sh = P.lvl_shape[P.levels() - 1];
                return u + (sh.s_lo - sh.j_lo);
            };
            for (int k = 0; k < L; ++k) {
                const int la = LA - 1 - k, lb = LB - 1 - k;
                // body_t: PRED of player 2's level waits for its observe there
                if (pred_gate && pb && lb >= 0 && lb < scfr_handle::kSideLevels && side_lv[lb])
                    CUDA_OK(cudaStreamWaitEvent(st ? st : h->stream, h->ev_lv[lb], 0));
                level<R>(LK_PRED, KK_PRED, pa, sa && la == LA - 1 ? -1 : la, pb, sb && lb == LB - 1 ? -1 : lb,
                         Au, Bu, Ax, Bx, false, sa && la == LA - 2 ? vc(A, Au) : nullptr,
                         sb && lb == LB - 2 ? vc(Bp, Bu) : nullptr);
            }
        }
        for (Player* P : {pa, pb})
            if (P && P->J == 0)
                launch(KK_TD_AVG, 2.0 * sizeof(R), [&] {
                    run1(k_avg0<R>, dim3(h->B), P->S, (const R*)vals<R>(P->x), vals<R>(P->avg),
                         (const double*)h->wsched.p, h->cap, (const long long*)h->tdev.p);
                });
        // body_t: the top-down pass follows all of player 2's observe (the join)
        if (pred_gate && side_last >= 0) CUDA_OK(cudaStreamWaitEvent(st ? st : h->stream, h->ev_lv[side_last], 0));
        // forced leaf levels: their x / avg are the parents' (k_expand_leaf)
        const bool xa = h->leaf_x && leaf_single(A), xb = h->leaf_x && leaf_single(Bp);
        for (int k = 0; k < L; ++k)
            level<R>(LK_TD_AVG, KK_TD_AVG, pa, xa && k == LA - 1 ? -1 : skip(k, fa), pb,
                     xb && k == LB - 1 ? -1 : skip(k, fb), nullptr, nullptr, Ax, Bx, false);
    }

    // observe (and, alt mode, player 1's current strategy): part1 = OBS of
    // player 1 + CUR (alt) or OBS of both (sim); part2 = OBS of player 2 (alt)
    template <class R>
    void observe_part(bool part1, bool part2) {
        Player& A = h->P[0];
        Player& Bp = h->P[1];
        R *Au = vals<R>(A.u), *Bu = vals<R>(Bp.u), *Ax = vals<R>(A.x), *Bx = vals<R>(Bp.x);
        R* Axp = vals<R>(A.xpost);
        const bool pr = predictive(h->variant);
        const int LA = A.levels(), LB = Bp.levels(), L = std::max(LA, LB);
        const int fa = first_level(A);
        auto skip = [](int l, int f) { return l < f ? -1 : l; };
        const bool xa = h->leaf_x && leaf_single(A);
        const bool fused = fuse_spmv();
        // OBS on a forced leaf level: its V equals u (leaf_note), so the
        // parent level reads u and the leaf launch skips writing V
        const bool oa = leaf_single(A), ob = leaf_single(Bp);
        auto leaf_u = [](const Player& P, const R* u) {
            const DevTree& sh = P.lvl_shape[P.levels() - 1];
            return u + (sh.s_lo - sh.j_lo);
        };
        if (h->mode == SCFR_MODE_SIM) {
            if (!part1) return;
            if (!fused) spmv<R>(h->U, Bx, Bp.S, Au, A.S, false);   // u1 = U x2
            if (!fused) spmv<R>(h->UT, Ax, A.S, Bu, Bp.S, true);  // u2 = -Uᵀ x1
            lf_[0] = lf_[1] = leaf_fusable(A) && leaf_fusable(Bp) && LA == LB;  // (one launch: both or none)
            for (int k = 0; k < L; ++k)
                level<R>(LK_OBS, pr ? KK_OBS : KK_OBS_RM, &A, lf_[0] && k == 0 ? -1 : LA - 1 - k, &Bp,
                         lf_[1] && k == 0 ? -1 : LB - 1 - k, Au, Bu, Ax, Bx, !pr,
                         oa && k == 1 ? leaf_u(A, Au) : nullptr, ob && k == 1 ? leaf_u(Bp, Bu) : nullptr,
                         oa && k == 0, ob && k == 0);
            lf_[0] = lf_[1] = false;
            return;
        }
        if (part1) {
            if (!fused) spmv<R>(h->U, Bx, Bp.S, Au, A.S, false);  // u1 = U x2
            const bool bc = pr && h->bcur_on;
            if (bc) bcur_ = vals<R>(A.bcur);
            lf_[0] = leaf_fusable(A);
            for (int k = 0; k < LA; ++k)
                level<R>(LK_OBS, pr ? KK_OBS : KK_OBS_RM, &A, lf_[0] && k == 0 ? -1 : LA - 1 - k, nullptr, -1, Au,
                         nullptr, Ax, nullptr, !pr || bc, oa && k == 1 ? leaf_u(A, Au) : nullptr, nullptr,
                         oa && k == 0, 0);
            lf_[0] = false;
            // current_strategy of player 1 into xpost: TD of the b that OBS
            // already regret-matched (into b, or into bcur for the predictive
            // variants), or RM on the fly (SCFR_NO_BCUR=1)
            const int fc = h->top_cur.on ? h->top_cur.ls : fa;  // (prepare_cur_top)
            cur_top_ = h->top_cur.on;
            for (int k = 0; k < LA; ++k)
                level<R>(pr && !bc ? LK_CUR : LK_TD, pr ? KK_CUR : KK_TD, &A, xa && k == LA - 1 ? -1 : skip(k, fc),
                         nullptr, -1, nullptr, nullptr, Axp, nullptr, false);
            cur_top_ = false;
            bcur_ = nullptr;
        }
        if (part2) {
            if (!fused) spmv<R>(h->UT, Axp, A.S, Bu, Bp.S, true);  // u2 = -Uᵀ x1'
            lf_[1] = leaf_fusable(Bp);
            int launched = 0;
            for (int k = 0; k < LB; ++k) {
                const int lb = lf_[1] && k == 0 ? -1 : LB - 1 - k;
                const bool side = obs_side && lb >= 0 && launched > 0 && lb < scfr_handle::kSideLevels;
                cudaStream_t keep = st;
                if (side) {
                    if (side_last < 0) {  // fork after the deepest launch
                        CUDA_OK(cudaEventRecord(h->ev_side, st));
                        CUDA_OK(cudaStreamWaitEvent(obs_side, h->ev_side, 0));
                    }
                    st = obs_side;
                }
                level<R>(LK_OBS, pr ? KK_OBS : KK_OBS_RM, nullptr, -1, &Bp, lb, nullptr, Bu, nullptr, Bx, !pr,
                         nullptr, ob && k == 1 ? leaf_u(Bp, Bu) : nullptr, 0, ob && k == 0);
                if (side) {
                    CUDA_OK(cudaEventRecord(h->ev_lv[lb], obs_side));
                    side_lv[lb] = true;
                    side_last = lb;
                }
                st = keep;
                if (lb >= 0) ++launched;
            }
            lf_[1] = false;
        }
    }

    // Overlapped alt iteration body: iteration t's observe with iteration
    // t+1's next, on two streams (captured as a fork / join):
    //   stream A: OBS1(t), CUR1(t) -> ev_a; NEXT1(t+1); wait ev_b; tick
    //   stream B: wait ev_a; OBS2(t); NEXT2(t+1) -> ev_b
    // NEXT1(t+1) reads only what OBS1(t) wrote and writes player 1's x / avg /
    // b / V, which OBS2(t) does not touch (it reads x1' = xpost); NEXT2(t+1)
    // follows OBS2(t) in stream order.  Schedules of t+1 via tofs = 1.
    template <class R>
    void body_t() {
        cudaStream_t A = h->stream, B = h->stream2;
        CUDA_OK(cudaEventRecord(h->ev_fork, A));
        CUDA_OK(cudaStreamWaitEvent(B, h->ev_fork, 0));
        st = A;
        observe_part<R>(true, false);
        CUDA_OK(cudaEventRecord(h->ev_a, A));
        CUDA_OK(cudaStreamWaitEvent(B, h->ev_a, 0));
        // stream B carries the critical chain from here on: its blocks are
        // scheduled ahead of NEXT1's when both are pending
        st = B;
        prio = h->prio_hi;
        obs_side = h->stream3;
        side_last = -1;
        for (bool& b : side_lv) b = false;
        observe_part<R>(false, true);
        obs_side = nullptr;
        tofs = 1;
        pred_gate = h->stream3 != nullptr;
        next_part<R>(false, true);
        pred_gate = false;
        CUDA_OK(cudaEventRecord(h->ev_b, B));
        prio = 0;
        st = A;
        next_part<R>(true, false);
        tofs = 0;
        CUDA_OK(cudaStreamWaitEvent(A, h->ev_b, 0));
        tick();
        st = nullptr;
    }
    void body() {
        if (h->f32) body_t<float>();
        else body_t<double>();
    }
    void prologue() {  // next of both players (iteration t)
        if (h->f32) next_part<float>(true, true);
        else next_part<double>(true, true);
    }
    void epilogue() {  // observe of the last iteration, then the tick
        if (h->f32) observe_part<float>(true, true);
        else observe_part<double>(true, true);
        tick();
    }
};

// Raise the device pool's release threshold once so freed solver buffers stay
// in the pool for the next solver (cudaMallocAsync path of DevBuf).
static void keep_pool_resident(int device) {
    static std::vector<char> done(64, 0);
    if (device < 0 || device >= 64 || done[device]) return;
    cudaMemPool_t pool;
    CUDA_OK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t threshold = UINT64_MAX;
    CUDA_OK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    done[device] = 1;
}

// Per-iteration scalars of every solve, [B][cap] on the host and the device:
// the averaging weight t^gamma and the DCFR factors, from libm pow like the
// reference (or the caller's values, scfr_set_schedule).  Growing the
// capacity keeps the entries already there.
static void upload_schedule(scfr_handle* h) {
    CUDA_OK(cudaStreamSynchronize(h->stream));
    CUDA_OK(copy_sync(h->wsched.p, h->w_host.data(), h->w_host.size() * sizeof(double), cudaMemcpyHostToDevice));
    CUDA_OK(copy_sync(h->pfsched.p, h->pf_host.data(), h->pf_host.size() * sizeof(double), cudaMemcpyHostToDevice));
    CUDA_OK(copy_sync(h->nfsched.p, h->nf_host.data(), h->nf_host.size() * sizeof(double), cudaMemcpyHostToDevice));
}

static void ensure_schedule(scfr_handle* h, int64_t upto) {
    if (upto <= h->cap) return;
    AllocStream alloc_on(h->stream);
    int64_t cap = std::max<int64_t>(4096, h->cap);
    while (cap < upto) cap *= 2;
    if (cap >= (1ll << 31)) fail(SCFR_EINVAL, "iteration count too large");
    const int B = h->B;
    const int64_t old = h->cap;
    std::vector<double> w((size_t)B * cap), pf((size_t)B * cap), nf((size_t)B * cap);
    for (int k = 0; k < B; ++k)
        for (int64_t i = 0; i < cap; ++i) {
            const size_t q = (size_t)k * cap + i;
            if (i < old) {  // (keeps caller-set entries)
                const size_t o = (size_t)k * old + i;
                w[q] = h->w_host[o];
                pf[q] = h->pf_host[o];
                nf[q] = h->nf_host[o];
                continue;
            }
            const int64_t t = i + 1;  // reference RegretState.t during iteration i+1
            w[q] = tpow(t, h->gamma[k]);
            pf[q] = dfactor(t, h->alpha[k]);
            nf[q] = dfactor(t, h->beta[k]);
        }
    CUDA_OK(cudaStreamSynchronize(h->stream));
    h->wsched.alloc(w.size());
    h->pfsched.alloc(pf.size());
    h->nfsched.alloc(nf.size());
    h->w_host.swap(w);
    h->pf_host.swap(pf);
    h->nf_host.swap(nf);
    h->cap = (int)cap;
    upload_schedule(h);
    for (cudaGraphExec_t* e : {&h->exec, &h->exec_pro, &h->exec_body, &h->exec_epi})
        if (*e) {
            cudaGraphExecDestroy(*e);
            *e = nullptr;
        }
}

template <class F>
static cudaGraphExec_t capture(scfr_handle* h, int64_t& nodes, F&& body) {
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    Launcher L(h);
    CUDA_OK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    body(L);
    CUDA_OK(cudaStreamEndCapture(h->stream, &graph));
    CUDA_OK(cudaGraphInstantiate(&exec, graph, cudaGraphInstantiateFlagUseNodePriority));
    cudaGraphDestroy(graph);
    nodes = L.count;
    return exec;
}

static void build_graph(scfr_handle* h) {
    h->exec = capture(h, h->nodes_per_iter, [](Launcher& L) { L.iteration(); });
}

static void build_overlap_graphs(scfr_handle* h) {
    h->exec_pro = capture(h, h->nodes_pro, [](Launcher& L) { L.prologue(); });
    h->exec_body = capture(h, h->nodes_body, [](Launcher& L) { L.body(); });
    h->exec_epi = capture(h, h->nodes_epi, [](Launcher& L) { L.epilogue(); });
}

static void set_device(const scfr_handle* h) { CUDA_OK(cudaSetDevice(h->device)); }

// Before the first iteration: player 2's structurally empty rows get the
// -0.0 that iteration would leave in u (k_fill_rows).
static void preset_constant_rows(scfr_handle* h) {
    if (h->t != 0) return;
    for (const auto& rg : h->neg_zero_rows) {
        const size_t cnt = (size_t)rg.second * h->B;
        const unsigned grid = (unsigned)((cnt + TPB - 1) / TPB);
        if (h->f32)
            k_fill_rows<float><<<grid, TPB, 0, h->stream>>>(vals<float>(h->P[1].u), h->P[1].S, h->B, rg.first,
                                                            rg.second, -0.0f);
        else
            k_fill_rows<double><<<grid, TPB, 0, h->stream>>>(h->P[1].u.p, h->P[1].S, h->B, rg.first, rg.second,
                                                             -0.0);
        CUDA_OK(cudaGetLastError());
    }
}

// Device -> caller memory for large state reads: DMA into the pinned arena,
// then a parallel copy out (pageable DMA of a Goofspiel-5 vector is ~3 ms).
// Several vectors (segments) share one pipeline: the copy out of a chunk
// overlaps the DMA of every chunk after it, across segments.
struct ReadSeg {
    double* host_out;
    const double* dev;
    size_t count;
};
static void read_to_host_multi(scfr_handle* h, const ReadSeg* seg, int nseg) {
    size_t total = 0;
    for (int k = 0; k < nseg; ++k) total += seg[k].count;
    if (!total) return;
    const size_t bytes = total * sizeof(double);
    PinnedArena& pa = pinned_arena();
    std::lock_guard<std::mutex> guard(pa.lock);
    pa.reset();
    double* stage = bytes >= (1u << 20) && pa.reserve(std::max(bytes, pa.cap)) ? static_cast<double*>(pa.take(bytes))
                                                                               : nullptr;
    if (!stage) {
        for (int k = 0; k < nseg; ++k)
            if (seg[k].count)
                CUDA_OK(copy_async(seg[k].host_out, seg[k].dev, seg[k].count * sizeof(double), cudaMemcpyDeviceToHost,
                                   h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));
        return;
    }
    constexpr int kParts = scfr_handle::kReadParts;  // chunks per segment
    cudaEvent_t* ev = h->rd_ev;                      // (the handle's device)
    if (!ev[0])
        for (int i = 0; i < scfr_handle::kReadEvents; ++i)
            CUDA_OK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    size_t base = 0;
    for (int k = 0; k < nseg; ++k) {
        const size_t count = seg[k].count, per = (count + kParts - 1) / kParts;
        for (int i = 0; i < kParts; ++i) {
            const size_t lo = std::min(count, i * per), n = std::min(count, lo + per) - lo;
            if (n)
                CUDA_OK(copy_async(stage + base + lo, seg[k].dev + lo, n * sizeof(double), cudaMemcpyDeviceToHost,
                                   h->stream));
            CUDA_OK(cudaEventRecord(ev[k * kParts + i], h->stream));
        }
        base += count;
    }
    base = 0;
    for (int k = 0; k < nseg; ++k) {
        const size_t count = seg[k].count, per = (count + kParts - 1) / kParts;
        double* out = seg[k].host_out;
        for (int i = 0; i < kParts; ++i) {
            const size_t lo = std::min(count, i * per), n = std::min(count, lo + per) - lo;
            CUDA_OK(cudaEventSynchronize(ev[k * kParts + i]));
            if (!n) continue;
            const double* src = stage + base + lo;
            parallel_chunks((int64_t)n, 1 << 16, [&](int, int64_t a, int64_t b) {
                std::memcpy(out + lo + a, src + a, (b - a) * sizeof(double));
            });
        }
        base += count;
    }
}
static void read_to_host(scfr_handle* h, double* host_out, const double* dev, size_t count) {
    const ReadSeg seg{host_out, dev, count};
    read_to_host_multi(h, &seg, 1);
}

static void check_player(const scfr_handle* h, int player, int solve) {
    if (!h) fail(SCFR_EINVAL, "handle is NULL");
    if (player != 1 && player != 2) fail(SCFR_EINVAL, "player must be 1 or 2");
    if (solve < 0 || solve >= h->B) fail(SCFR_EINVAL, "solve index out of range");
}

static void add_weights(scfr_handle* h, int64_t n) {
    ensure_schedule(h, h->t + n);
    // float(t)**gamma must be finite for every iteration about to run: the
    // reference's Python float power raises OverflowError there (and an
    // infinite weight would turn the average into NaN)
    for (int k = 0; k < h->B; ++k)
        for (int64_t i = 0; i < n; ++i)
            if (!std::isfinite(h->w_host[(size_t)k * h->cap + h->t + i]))
                fail(SCFR_EOVERFLOW, "t**gamma overflows at iteration %lld (solve %d, gamma %g)",
                     (long long)(h->t + i + 1), k, h->gamma[k]);
    for (int k = 0; k < h->B; ++k)
        for (int64_t i = 0; i < n; ++i) h->avg_weight[k] += h->w_host[(size_t)k * h->cap + h->t + i];
}

// Best response of `player` against the opponent's strategy x_opp (one solve).
// out = (±) M x for one solve outside the iteration graph (best response,
// expected value): this rank's rows, all-gathered when sharded.
static void solve_spmv(scfr_handle* h, const DevCsr& M, const double* x, double* out, bool neg) {
    k_spmv<<<dim3(grid_for(M.rows), 1), TPB, 0, h->stream>>>(M.rows, M.indptr.p, M.indices.p,
                                                            M.data.p, x, 0, out + M.row0, 0,
                                                            neg ? 1 : 0, nullptr);
    CUDA_OK(cudaGetLastError());
    if (h->rowshard()) allgather_rows(h, out, M.chunk);
}

static double best_response(scfr_handle* h, int player, const double* x_opp) {
    Player& P = h->P[player - 1];
    solve_spmv(h, player == 1 ? h->U : h->UT, x_opp, P.g.p, player == 2);
    for (int l = P.levels() - 1; l >= 0; --l) {
        const int lo = P.lvl[l], hi = P.lvl[l + 1];
        if (warp_level(h, P, l))
            k_br_warp<<<(hi - lo + TPB / 32 - 1) / (TPB / 32), TPB, 0, h->stream>>>(shaped_tree(P, l), lo, hi, P.g.p, P.W.p);
        else
            k_br<<<grid_for(hi - lo), TPB, 0, h->stream>>>(shaped_tree(P, l), lo, hi, P.g.p, P.W.p);
    }
    k_br_root<<<1, 1, 0, h->stream>>>(P.tree(), P.g.p, P.W.p, h->brout.p + (player - 1));
    CUDA_OK(cudaGetLastError());
    double v = 0.0;
    CUDA_OK(copy_async(&v, h->brout.p + (player - 1), sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CUDA_OK(cudaStreamSynchronize(h->stream));
    return v;
}

// Device pointer to the solve's profile component: normalised average
// (written into xbar) or the last emitted strategy.
// Restores the forced leaf copies (k_expand_leaf) of x / xpost / avg of
// one solve before it is read.
static void expand_leaves(scfr_handle* h, int player, DevBuf<double>& buf, int solve) {
    Player& P = h->P[player - 1];
    if (!h->leaf_x || !leaf_single(h, P)) return;
    const int l = P.levels() - 1;
    const DevTree T = shaped_tree(P, l);
    const int j0 = P.lvl[l], n = P.lvl[l + 1] - j0, shift = P.lvl_shape[l].s_lo - j0;
    if (h->f32)
        k_expand_leaf<float><<<grid_for(n), TPB, 0, h->stream>>>(T, j0, n, shift, vals<float>(buf) + (size_t)solve * P.S);
    else
        k_expand_leaf<double><<<grid_for(n), TPB, 0, h->stream>>>(T, j0, n, shift, buf.p + (size_t)solve * P.S);
    CUDA_OK(cudaGetLastError());
}

static const double* profile(scfr_handle* h, int player, int solve, int which) {
    Player& P = h->P[player - 1];
    if (which == 1) {
        expand_leaves(h, player, P.x, solve);
        return orig_order(h, player, P.x.p, solve);
    }
    expand_leaves(h, player, P.avg, solve);
    if (h->avg_weight[solve] == 0.0) fail(SCFR_EINVAL, "no strategies accumulated yet");
    const double* avg = orig_order(h, player, P.avg.p, solve);
    k_normalize<<<grid_for(P.S), TPB, 0, h->stream>>>(avg, h->avg_weight[solve], P.xbar.p, P.S);
    CUDA_OK(cudaGetLastError());
    return P.xbar.p;
}

}  // namespace scfr

using namespace scfr;

extern "C" {

// Shared body of scfr_create / scfr_create_sharded (nccl_id == nullptr: one GPU).
// The top of player k (TopInfo): the largest split ls whose levels [0, ls)
// hold at most kTopDPs decision points and under whose sequences hang only
// level-ls DPs.  Top-down passes (TD + average, TD into xpost) then do not
// launch those levels: the level-ls launch recomputes each DP's parent x from
// its ancestor chain, x = b_a·(…·(b_0·1.0)), the same products in the same
// order, and writes the top's x (and average) once.  Bottom-up passes keep
// launching every level (completing the top in-kernel by last arrival
// measured slower than the launches it saved: DESIGN.md §4).
static void build_top(scfr_handle* h, int k, int ls, int pro, TopPlayer& tp);

__global__ void k_min_index(int n, const int* __restrict__ ix, int* __restrict__ out) {
    int m = INT32_MAX;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) m = min(m, ix[i]);
    m = __reduce_min_sync(0xffffffffu, (unsigned)m);
    if ((threadIdx.x & 31) == 0) atomicMin(out, m);
}

// Alternating mode: player 1's x' (xpost) is read only through player 2's
// fused payoff rows.  When every such row reads sequences of the level just
// below player 1's top (Goofspiel-5: level 3 after the leaf mapping), the
// current-strategy pass skips that level too: its one launch recomputes each
// DP's parent x' from a one-level-longer ancestor chain, and x' above it is
// never written (TopInfo::pro = 0).  One launch fewer on the alternating
// critical path, but opt-in (SCFR_CUR_TOP=1): the longer chains cost more
// than the launch (Goofspiel-5 124.4 vs 122.1 us, bit-exact either way).
static void prepare_cur_top(scfr_handle* h) {
    const char* on = std::getenv("SCFR_CUR_TOP");
    if (!(on && on[0] == '1')) return;
    if (h->mode != SCFR_MODE_ALT || !h->fuse || h->P[0].J == 0 || h->P[1].J == 0 || !h->top[0].on) return;
    if (predictive(h->variant) && !h->bcur_on) return;  // (CUR regret-matches on the fly: no chain source)
    Player& P = h->P[0];
    const int L = P.levels(), lc = h->top[0].ls + 1;
    const bool xa = h->leaf_x && leaf_single(h, P);
    if (lc > kTopMax || lc > (xa ? L - 2 : L - 1)) return;
    const std::vector<int>& sp = *P.h_seq_ptr;
    const int Stop = sp[P.lvl[lc]];
    for (int m = lc + 1; m < L; ++m)  // DPs below hang under level->=lc sequences only
        if (P.lvl_pmin[m] < Stop) return;
    // every column of player 2's rows (after the leaf mapping) at or below level lc
    const DevCsr& M = h->UT;
    if (M.nnz > 0) {
        DevBuf<int> mn;
        mn.alloc(1);
        const int init = INT32_MAX;
        CUDA_OK(copy_async(mn.p, &init, sizeof init, cudaMemcpyHostToDevice, h->stream));
        k_min_index<<<std::min(grid_for(M.nnz), 4 * h->num_sms), TPB, 0, h->stream>>>(M.nnz, M.iter_indices(), mn.p);
        CUDA_OK(cudaGetLastError());
        int v = 0;
        CUDA_OK(copy_async(&v, mn.p, sizeof v, cudaMemcpyDeviceToHost, h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));
        if (v < Stop) return;
    }
    build_top(h, 0, lc, 0, h->top_cur);
}

static void prepare_top(scfr_handle* h, int k) {
    int kTopDPs = 4096;  // SCFR_TOP_DPS: the cap (A/B: Goofspiel-5 137.4 us at 505 top DPs vs 142.1 us at 24505)
    if (const char* e = std::getenv("SCFR_TOP_DPS")) kTopDPs = std::atoi(e);
    const char* off = std::getenv("SCFR_NO_TOP");
    if (off && off[0] == '1') return;
    Player& P = h->P[k];
    const int L = P.levels();
    if (L < 2 || !P.h_seq_ptr || !P.h_dp_parent) return;
    // player 1's current strategy regret-matches on the fly (SCFR_NO_BCUR=1):
    // its chain would need the sums, so keep its top launched
    if (k == 0 && predictive(h->variant) && h->mode == SCFR_MODE_ALT && !h->bcur_on) return;
    const std::vector<int>& sp = *P.h_seq_ptr;
    const std::vector<int>& par = *P.h_dp_parent;
    // the level-ls launch must run: not a forced leaf level whose top-down
    // launches are skipped (leaf_x)
    const int lmax = std::min(h->leaf_x && leaf_single(h, P) ? L - 2 : L - 1, kTopMax);
    int ls = 0;
    for (int l = lmax; l >= 1; --l) {
        if (P.lvl[l] > kTopDPs) continue;
        const int Stop = sp[P.lvl[l]];
        bool ok = true;  // DPs below level l hang under forest sequences only (per-level minima)
        for (int m = l + 1; m < L && ok; ++m) ok = P.lvl_pmin[m] >= Stop;
        if (ok) {
            ls = l;
            break;
        }
    }
    if (ls == 0) return;
    build_top(h, k, ls, 1, h->top[k]);
}

// The ancestor chains of every sequence above level ls of player k (TopInfo).
static void build_top(scfr_handle* h, int k, int ls, int pro, TopPlayer& tp) {
    Player& P = h->P[k];
    const std::vector<int>& sp = *P.h_seq_ptr;
    const std::vector<int>& par = *P.h_dp_parent;
    const int Jtop = P.lvl[ls], Stop = sp[Jtop];
    std::vector<int> sdp(std::max(Stop, 1), -1), lvl_of(Jtop, 0);
    for (int q = 0; q < Jtop; ++q)
        for (int s = sp[q]; s < sp[q + 1]; ++s) sdp[s] = q;
    for (int l = 0; l < ls; ++l)
        for (int q = P.lvl[l]; q < P.lvl[l + 1]; ++q) lvl_of[q] = l;
    std::vector<int> anc((size_t)std::max(Stop, 1) * ls, -1);
    for (int s = 1; s < Stop; ++s) {
        int chain[kTopMax + 1], n = 0;
        for (int a = s; a != 0 && n <= kTopMax; a = par[sdp[a]]) chain[n++] = a;
        if (n > ls) return;  // (cannot happen: one ancestor per top level)
        for (int i = 0; i < n; ++i) {
            const int a = chain[n - 1 - i];
            anc[(size_t)s * ls + i] = a | (P.lvl_shape[lvl_of[sdp[a]]].un == 1 ? 1 << 30 : 0);
        }
    }
    TopInfo info{};
    info.ls = ls;
    info.Stop = Stop;
    info.pro = pro;
    tp.anc.alloc(anc.size());
    CUDA_OK(copy_async(tp.anc.p, anc.data(), anc.size() * sizeof(int), cudaMemcpyHostToDevice, h->stream));
    info.anc = tp.anc.p;
    tp.info.alloc(1);
    CUDA_OK(copy_async(tp.info.p, &info, sizeof info, cudaMemcpyHostToDevice, h->stream));
    CUDA_OK(cudaStreamSynchronize(h->stream));  // the host vectors die here
    tp.ls = ls;
    tp.on = true;
}

// Subtree mode: the partition (subtree.h) on the structure this create
// converted; every rank must launch the level that recomputes a player's top
// (its top_prologue writes the whole top's x).
static void plan_subtree_mode(scfr_handle* h, const scfr_csr* U) {
    HostProcess H[2];
    for (int k = 0; k < 2; ++k) {
        const Player& P = h->P[k];
        if (!P.h_seq_ptr || !P.h_dp_parent || P.J == 0)
            fail(SCFR_EINVAL, "the subtree-sharded mode needs decision points for both players");
        H[k] = HostProcess{P.h_seq_ptr->data(), P.h_dp_parent->data(), &P.lvl, P.J, P.S};
    }
    SubtreePlan plan;
    const char* sim = std::getenv("SCFR_SUBTREE_SIM");
    h->sub_sim = h->world == 1 && sim ? std::max(1, std::atoi(sim)) : 1;
    // SCFR_SUBTREE_VIEW="W,r" (world 1, timing only): launch exactly rank r's
    // ranges of a W-rank plan, no exchange: one rank's per-iteration kernel
    // time at N = W (the values are not a solve: other ranks' roots are stale)
    int vw = 1;
    if (const char* v = std::getenv("SCFR_SUBTREE_VIEW"))
        if (h->world == 1 && std::sscanf(v, "%d,%d", &vw, &h->sub_view) == 2 && vw >= 1 && h->sub_view >= 0 &&
            h->sub_view < vw) {
            h->sub_sim = 1;
        } else {
            vw = 1;
            h->sub_view = -1;
        }
    plan_subtrees(H, U, h->world * h->sub_sim * vw, plan);
    for (int k = 0; k < 2; ++k) {
        h->sub_ls[k] = plan.ls[k];
        h->sub_jb[k] = std::move(plan.jb[k]);
        h->sub_sb[k] = std::move(plan.sb[k]);
        const TopPlayer& tp = h->top[k];
        if (tp.on && tp.ls >= h->sub_ls[k]) {
            const std::vector<int>& jb = h->sub_jb[k][tp.ls];
            for (int r = 0; r < h->world * h->sub_sim * vw; ++r)
                if (jb[r + 1] == jb[r])
                    fail(SCFR_EINVAL, "rank %d holds no level-%d decision point of player %d", r, tp.ls, k + 1);
        }
    }
}

static void create_impl(const scfr_tfsdp* p1, const scfr_tfsdp* p2, const scfr_csr* U,
                        const scfr_csr* UT, const scfr_config* cfg, int device,
                        const char* nccl_id, int rank, int world, scfr_handle** out, bool subtree = false) {
    NvtxRange nvtx("scfr_create");
    {
        if (!out || !cfg || !p1 || !p2 || !U || !UT) fail(SCFR_EINVAL, "NULL argument");
        const char* mname = subtree ? "subtree-sharded" : "row-sharded";
        if (nccl_id) {
            if (world < 1 || rank < 0 || rank >= world) fail(SCFR_EINVAL, "bad rank / world size");
            if (cfg->batch != 1) fail(SCFR_EINVAL, "the %s mode runs a single solve (batch 1)", mname);
            if (cfg->engine != SCFR_ENGINE_AUTO && cfg->engine != SCFR_ENGINE_LEVELS)
                fail(SCFR_EINVAL, "the %s mode runs on the level engine", mname);
        }
        if (cfg->variant < SCFR_CFR || cfg->variant > SCFR_PCFR_PLUS) fail(SCFR_EINVAL, "unknown variant");
        if (cfg->dtype != SCFR_DTYPE_F64 && cfg->dtype != SCFR_DTYPE_F32) fail(SCFR_EINVAL, "unknown dtype");
        if (cfg->dtype == SCFR_DTYPE_F32) {
            if (nccl_id) fail(SCFR_EINVAL, "the fp32 mode does not run the %s mode", mname);
            if (cfg->engine != SCFR_ENGINE_AUTO && cfg->engine != SCFR_ENGINE_LEVELS)
                fail(SCFR_EINVAL, "the fp32 mode runs on the level engine");
        }
        if (cfg->mode != SCFR_MODE_SIM && cfg->mode != SCFR_MODE_ALT) fail(SCFR_EINVAL, "mode must be sim or alt");
        if (cfg->batch < 1) fail(SCFR_EINVAL, "batch must be >= 1");
        if (cfg->engine < SCFR_ENGINE_AUTO || cfg->engine > SCFR_ENGINE_PERSISTENT_CLUSTER)
            fail(SCFR_EINVAL, "unknown engine");
        if (cfg->engine == SCFR_ENGINE_PERSISTENT_GRID && cfg->batch != 1)
            fail(SCFR_EINVAL, "the grid-persistent engine runs a single solve (batch 1)");
        int ndev = 0;
        cudaError_t e = cudaGetDeviceCount(&ndev);
        if (e != cudaSuccess || ndev == 0) fail(SCFR_ECUDA, "no CUDA device available: %s", cudaGetErrorString(e));
        if (device < 0 || device >= ndev) fail(SCFR_EINVAL, "device index out of range");
        CUDA_OK(cudaSetDevice(device));
        int major = 0, nsm = 0;  // (cudaGetDeviceProperties costs milliseconds)
        CUDA_OK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
        CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
        if (major < 10) {
            int minor = 0;
            cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
            fail(SCFR_ECUDA, "device %d is sm_%d%d; this build targets sm_100a", device, major, minor);
        }
        std::unique_ptr<scfr_handle> h(new scfr_handle());
        h->device = device;
        h->num_sms = nsm;
        h->B = cfg->batch;
        h->f32 = cfg->dtype == SCFR_DTYPE_F32;
        h->variant = cfg->variant;
        h->mode = cfg->mode;
        h->engine = cfg->engine;
        h->alpha.resize(h->B);
        h->beta.resize(h->B);
        h->gamma.resize(h->B);
        for (int k = 0; k < h->B; ++k) {
            h->alpha[k] = cfg->batch_alpha ? cfg->batch_alpha[k] : cfg->alpha;
            h->beta[k] = cfg->batch_beta ? cfg->batch_beta[k] : cfg->beta;
            h->gamma[k] = cfg->batch_gamma ? cfg->batch_gamma[k] : cfg->gamma;
            if (!std::isfinite(h->alpha[k]) || !std::isfinite(h->beta[k])) fail(SCFR_EINVAL, "alpha and beta must be finite");
            if (!(h->gamma[k] >= 0)) fail(SCFR_EINVAL, "gamma must be >= 0");
        }
        if (p1->num_seqs != U->rows || p2->num_seqs != U->cols || UT->rows != U->cols ||
            UT->cols != U->rows || UT->nnz != U->nnz)
            fail(SCFR_EINVAL, "dimension mismatch between the payoff matrix and the decision processes");
        const char* trace = std::getenv("SCFR_TRACE");
        auto t_prev = std::chrono::steady_clock::now();
        auto stage = [&](const char* what) {  // SCFR_TRACE=1: create-time breakdown on stderr
            nvtxMarkA(what);
            if (!(trace && trace[0] == '1')) return;
            const auto now = std::chrono::steady_clock::now();
            std::fprintf(stderr, "[scfr_create] %-12s %8.2f ms\n", what,
                         std::chrono::duration<double, std::milli>(now - t_prev).count());
            t_prev = now;
        };
        CUDA_OK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        keep_pool_resident(device);
        AllocStream alloc_on(h->stream);
        CUDA_OK(cudaEventCreate(&h->ev0));
        CUDA_OK(cudaEventCreate(&h->ev1));
        stage("stream");
        PinnedArena& pa = pinned_arena();
        std::lock_guard<std::mutex> pin_guard(pa.lock);
        pa.reserve((size_t)(U->rows + UT->rows) * 4 + (size_t)std::max<int64_t>(U->nnz, 1) * 24 + 8192);
        pa.reset();
        const int w = nccl_id ? world : 1, rk = nccl_id ? rank : 0;
        const int wc = subtree ? 1 : w, rc = subtree ? 0 : rk;  // payoff rows held: all in the subtree mode
        {
            // four concurrent tasks (player 1, player 2, U, Uᵀ), a quarter of
            // the host threads each (2/3 for the players' validation measured
            // no better: the host is memory-bound across the four)
            // (+ a fifth: the first 4096 iterations' schedules, host libm pow,
            // which the first scfr_step would otherwise compute).  Unsharded,
            // Uᵀ is derived from U on the device afterwards (transpose.cu), so
            // three uploads share the threads.
            const char* hut = std::getenv("SCFR_HOST_UT");
            const bool dev_ut = wc == 1 && !(hut && hut[0] == '1');
            const int quarter = std::max(1, host_threads() / (dev_ut ? 3 : 4));
            std::exception_ptr err[5];
            auto task = [&](int k) {
                try {
                    CUDA_OK(cudaSetDevice(h->device));  // (per-thread current device)
                    tl_host_threads = quarter;
                    cudaStream_t sk = h->stream;  // (own streams per upload measured no faster: PCIe-bound)
                    AllocStream alloc_k(sk);
                    switch (k) {
                        case 0: upload_player(p1, h->P[0], h->B, sk, 0, h->f32); break;
                        case 1: upload_player(p2, h->P[1], h->B, sk, 1, h->f32); break;
                        case 2: upload_csr(U, h->U, sk, h->f32, wc, rc); break;
                        case 3: upload_csr(UT, h->UT, sk, h->f32, wc, rc); break;
                        default: ensure_schedule(h.get(), 1); break;
                    }
                } catch (...) {
                    err[k] = std::current_exception();
                }
            };
            std::thread t1(task, 1), t2(task, 2), t4(task, 4);
            std::thread t3;
            if (!dev_ut) t3 = std::thread(task, 3);
            const int saved = tl_host_threads;
            task(0);
            tl_host_threads = saved;
            t1.join();
            t2.join();
            if (t3.joinable()) t3.join();
            t4.join();
            for (auto& e : err)
                if (e) std::rethrow_exception(e);
            if (dev_ut) {
                AllocStream alloc_t(h->stream);
                derive_transpose(h->U, UT, h->UT, h->stream, h->f32);
            }
            csr_level_info(U, h->U, h->P[0], h->stream, wc == 1);  // U's rows: player 1's sequences
            csr_level_info(UT, h->UT, h->P[1], h->stream, wc == 1, dev_ut);
            CUDA_OK(cudaStreamSynchronize(h->stream));
        }
        stage("players+payoff");
        if (nccl_id) {
            // u and the BR gradient are gathered as world x chunk (padded) vectors
            for (int k = 0; k < 2 && !subtree; ++k) {
                Player& P = h->P[k];
                const size_t pad = (size_t)w * (k == 0 ? h->U.chunk : h->UT.chunk);
                if (pad > (size_t)P.S) {
                    P.u.alloc(pad);
                    P.u.zero(h->stream);
                    P.g.alloc(pad);
                }
            }
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof id);
            ncclComm_t comm;
            NCCL_OK(nccl().CommInitRank(&comm, w, id, rk));
            h->comm = comm;
            h->comm_destroy = [](void* c) { nccl().CommDestroy((ncclComm_t)c); };
            h->world = w;
            h->rank = rk;
            h->subtree = subtree;
        }
        stage("payoff");
        h->tdev.alloc(1);
        h->tdev.zero(h->stream);
        h->nonfinite.alloc(1);
        h->nonfinite.zero(h->stream);
        h->brout.alloc(2);
        h->avg_weight.assign(h->B, 0.0);
        const char* ng = std::getenv("SCFR_NO_GRAPH");
        h->use_graph = !(ng && ng[0] == '1');
        const char* np = std::getenv("SCFR_NO_PDL");
        h->pdl = !(np && np[0] == '1');
        const char* nls = std::getenv("SCFR_NO_LEAF_SKIP");
        h->leaf_skip = !(nls && nls[0] == '1');
        const char* ngr = std::getenv("SCFR_NO_GROUP");
        h->group = !(ngr && ngr[0] == '1');
        const char* nlf = std::getenv("SCFR_NO_LEAF_FUSE");
        h->leaf_fuse = !(nlf && nlf[0] == '1');
        const char* npp = std::getenv("SCFR_NO_PIPE");
        h->pipe = !(npp && npp[0] == '1');
        if (const char* pnj = std::getenv("SCFR_PIPE_NJ")) h->pipe_nj = std::atoll(pnj);
        if (const char* pk = std::getenv("SCFR_PIPE_KINDS")) h->pipe_kinds = std::atoi(pk);
        const char* npr = std::getenv("SCFR_PAIR");  // opt-in: measured slower
        h->pair = npr && npr[0] == '1' && !subtree;
        if (const char* gnj = std::getenv("SCFR_GROUP_NJ")) h->group_nj = std::atoll(gnj);
        const char* nsw = std::getenv("SCFR_NO_SMALL_WARP");
        h->small_warp = !(nsw && nsw[0] == '1');
        if (const char* wnj = std::getenv("SCFR_WARP_NJ")) h->warp_nj = std::atoll(wnj);
        const char* nar = std::getenv("SCFR_NO_ROW_SHAPE");
        h->affine_rows = !(nar && nar[0] == '1');
        const char* ntw = std::getenv("SCFR_NO_TD_WARP");
        h->td_warp = !(ntw && ntw[0] == '1');
        const char* nfz = std::getenv("SCFR_NO_FUSE");
        h->fuse = !(nfz && nfz[0] == '1') && !h->rowshard();  // row-sharded: SpMV + all-gather instead
        if (subtree && !h->fuse) fail(SCFR_EINVAL, "the subtree-sharded mode runs the fused level engine");
        if (const char* wc = std::getenv("SCFR_WAVE_CTAS")) {
            h->wave_ctas = std::max(1, std::atoi(wc));
            h->wave_ctas_env = true;
        }
        const char* eng = std::getenv("SCFR_ENGINE");  // override for experiments / tests
        if (eng && h->engine == SCFR_ENGINE_AUTO && !h->comm) h->engine = std::atoi(eng);
        if (h->f32) h->engine = SCFR_ENGINE_LEVELS;  // (validated above)
        if (h->engine == SCFR_ENGINE_AUTO) {
            // the tile engine is opt-in: bit-exact, but not yet faster than
            // PDL-chained level kernels on the config games
            h->engine = h->comm ? SCFR_ENGINE_LEVELS : choose_engine(h.get());
        } else if (h->engine == SCFR_ENGINE_TILED) {
            prepare_tiled(h.get(), U, UT, true);
        }
        if (h->engine == SCFR_ENGINE_PERSISTENT || h->engine == SCFR_ENGINE_PERSISTENT_GRID ||
            h->engine == SCFR_ENGINE_PERSISTENT_CLUSTER)
            prepare_persistent(h.get());
        if (h->engine == SCFR_ENGINE_LEVELS && !h->rowshard() && h->fuse && h->P[0].J > 0 && h->P[1].J > 0) {
            // structurally empty payoff rows: u is a constant ±0.0 (kernels.cuh ld_u)
            const char* nue = std::getenv("SCFR_NO_EMPTY_ROWS");
            h->u_empty_skip = !(nue && nue[0] == '1');
            const Player& P2 = h->P[1];
            for (int l = 0; h->u_empty_skip && l < P2.levels(); ++l)
                if (Launcher::rows_empty(P2, l, h->UT)) {
                    const int s0 = l == 0 ? 0 : P2.lvl_s0[l];
                    h->neg_zero_rows.emplace_back(s0, P2.lvl_s0[l] + (int)P2.lvl_ns[l] - s0);
                }
        }
        stage("engine choice");
        if (h->engine == SCFR_ENGINE_LEVELS && predictive(h->variant) && h->mode == SCFR_MODE_ALT) {
            const char* nb = std::getenv("SCFR_NO_BCUR");
            h->bcur_on = !(nb && nb[0] == '1');
            if (h->bcur_on) h->P[0].bcur.alloc(val_slots((size_t)h->P[0].S * h->B, h->f32));
        }
        if (h->engine == SCFR_ENGINE_LEVELS && !h->rowshard()) {
            // forced leaf levels: skip their top-down launches (k_expand_leaf)
            const bool l1 = leaf_single(h.get(), h->P[0]), l2 = leaf_single(h.get(), h->P[1]);
            h->leaf_x = l1 || l2;
            if (l2) build_iter_indices(h.get(), h->U, h->P[1]);   // U's columns: player 2's sequences
            if (l1) build_iter_indices(h.get(), h->UT, h->P[0]);  // Uᵀ's columns: player 1's
            stage("leaf columns");
            // top-down passes recompute the top's x from ancestor chains
            prepare_top(h.get(), 0);
            prepare_top(h.get(), 1);
            prepare_cur_top(h.get());
            stage("top");
            // alt mode: player 1's next overlaps player 2's observe
            const char* nov = std::getenv("SCFR_NO_OVERLAP");
            if (h->mode == SCFR_MODE_ALT && h->fuse && !(nov && nov[0] == '1') && h->P[0].J > 0 &&
                h->P[1].J > 0) {
                CUDA_OK(cudaStreamCreateWithFlags(&h->stream2, cudaStreamNonBlocking));
                CUDA_OK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
                CUDA_OK(cudaEventCreateWithFlags(&h->ev_a, cudaEventDisableTiming));
                CUDA_OK(cudaEventCreateWithFlags(&h->ev_b, cudaEventDisableTiming));
                if (subtree) {  // stream 2's root exchanges on a second communicator
                    ncclComm_t c2 = nullptr;
                    NCCL_OK(nccl().CommSplit((ncclComm_t)h->comm, 0, h->rank, &c2, nullptr));
                    h->comm2 = c2;
                }
                // predictive variants, opt-in (SCFR_OBS_SIDE=1; measured slower, 130.5 vs
                // 122.9 us: the graph's third branch delays PRED2's level 2 behind
                // stream A's work): player 2's small observe levels on a third
                // stream beside PRED2's deep ones, PRED in its own value buffer
                const char* os3 = std::getenv("SCFR_OBS_SIDE");
                if (predictive(h->variant) && os3 && os3[0] == '1') {
                    for (Player& P : h->P) P.PV.alloc(val_slots((size_t)std::max(P.J, 1) * h->B, h->f32));
                    CUDA_OK(cudaStreamCreateWithFlags(&h->stream3, cudaStreamNonBlocking));
                    CUDA_OK(cudaEventCreateWithFlags(&h->ev_side, cudaEventDisableTiming));
                    for (auto& e : h->ev_lv) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                }
                h->overlap = true;
                int lo = 0, hi = 0;
                const char* npr2 = std::getenv("SCFR_NO_PRIO");
                if (!(npr2 && npr2[0] == '1') && cudaDeviceGetStreamPriorityRange(&lo, &hi) == cudaSuccess) h->prio_hi = hi;
                if (const char* pn = std::getenv("SCFR_PRIO_NJ")) h->prio_nj = std::atoll(pn);
            }
        }
        if (subtree) plan_subtree_mode(h.get(), U);
        stage("streams");
        CUDA_OK(cudaStreamSynchronize(h->stream));
        for (Player& P : h->P) P.h_seq_ptr = P.h_dp_parent = nullptr;  // scratch is reused
        stage("engine");
        *out = h.release();
    }
}

int scfr_create(const scfr_tfsdp* p1, const scfr_tfsdp* p2, const scfr_csr* U, const scfr_csr* UT,
                const scfr_config* cfg, int device, scfr_handle** out) {
    return guarded([&] { create_impl(p1, p2, U, UT, cfg, device, nullptr, 0, 1, out); });
}

int scfr_create_subtree(const scfr_tfsdp* p1, const scfr_tfsdp* p2, const scfr_csr* U,
                        const scfr_csr* UT, const scfr_config* cfg, int device,
                        const char* nccl_id, int rank, int world, scfr_handle** out) {
    return guarded([&] {
        if (!nccl_id) fail(SCFR_EINVAL, "NULL NCCL unique id");
        create_impl(p1, p2, U, UT, cfg, device, nccl_id, rank, world, out, true);
    });
}

int scfr_nccl_unique_id(char* out) {
    return guarded([&] {
        if (!out) fail(SCFR_EINVAL, "NULL argument");
        ncclUniqueId id;
        NCCL_OK(nccl().GetUniqueId(&id));
        std::memcpy(out, &id, sizeof id);
    });
}

int scfr_create_sharded(const scfr_tfsdp* p1, const scfr_tfsdp* p2, const scfr_csr* U,
                        const scfr_csr* UT, const scfr_config* cfg, int device,
                        const char* nccl_id, int rank, int world, scfr_handle** out) {
    return guarded([&] {
        if (!nccl_id) fail(SCFR_EINVAL, "NULL NCCL unique id");
        create_impl(p1, p2, U, UT, cfg, device, nccl_id, rank, world, out);
    });
}

int scfr_engine(const scfr_handle* h, int* engine) {
    return guarded([&] {
        if (!h || !engine) fail(SCFR_EINVAL, "NULL argument");
        *engine = h->engine;
    });
}

int scfr_step(scfr_handle* h, int64_t n) {
    NvtxRange nvtx("scfr_step");
    return guarded([&] {
        if (!h) fail(SCFR_EINVAL, "handle is NULL");
        if (n < 0) fail(SCFR_EINVAL, "n_iter must be >= 0");
        if (n == 0) return;
        set_device(h);
        add_weights(h, n);
        preset_constant_rows(h);
        CUDA_OK(cudaEventRecord(h->ev0, h->stream));
        if (is_persistent(h->engine)) {
            h->launches += launch_persistent(h, n);
        } else if (h->use_graph && h->overlap) {
            // prologue, n - 1 overlapped bodies, epilogue: the state is back at
            // an iteration boundary when the call returns
            if (!h->exec_body) build_overlap_graphs(h);
            CUDA_OK(cudaGraphLaunch(h->exec_pro, h->stream));
            for (int64_t i = 1; i < n; ++i) CUDA_OK(cudaGraphLaunch(h->exec_body, h->stream));
            CUDA_OK(cudaGraphLaunch(h->exec_epi, h->stream));
            h->launches += h->nodes_pro + (n - 1) * h->nodes_body + h->nodes_epi;
        } else if (h->use_graph) {
            if (!h->exec) build_graph(h);
            for (int64_t i = 0; i < n; ++i) CUDA_OK(cudaGraphLaunch(h->exec, h->stream));
            h->launches += n * h->nodes_per_iter;
        } else {
            Launcher L(h);
            for (int64_t i = 0; i < n; ++i) L.iteration();
            CUDA_OK(cudaGetLastError());
            h->launches += L.count;
        }
        CUDA_OK(cudaEventRecord(h->ev1, h->stream));
        h->timed = true;
        h->t += n;
        h->sub_stale = h->subtree;
    });
}

int scfr_profile_step(scfr_handle* h, int64_t n, scfr_kernel_stat* out, int cap, int* count) {
    return guarded([&] {
        if (!h || !out || !count || cap < KK_COUNT) fail(SCFR_EINVAL, "bad arguments");
        if (n < 1) fail(SCFR_EINVAL, "n_iter must be >= 1");
        set_device(h);
        add_weights(h, n);
        preset_constant_rows(h);
        std::vector<KernelRecord> recs;
        int64_t issued = 0;
        if (is_persistent(h->engine)) {
            KernelRecord r;
            r.kind = KK_PERSIST;
            r.bytes = persistent_bytes_per_iter(h) * (double)n;
            CUDA_OK(cudaEventCreate(&r.e0));
            CUDA_OK(cudaEventCreate(&r.e1));
            CUDA_OK(cudaEventRecord(r.e0, h->stream));
            issued = launch_persistent(h, n);
            CUDA_OK(cudaEventRecord(r.e1, h->stream));
            recs.push_back(r);
        } else {
            Launcher L(h);
            L.prof = &recs;
            for (int64_t i = 0; i < n; ++i) L.iteration();
            issued = L.count;
        }
        CUDA_OK(cudaGetLastError());
        CUDA_OK(cudaStreamSynchronize(h->stream));
        h->timed = false;
        h->t += n;
        h->sub_stale = h->subtree;
        h->launches += issued;
        for (int k = 0; k < KK_COUNT; ++k) {
            std::snprintf(out[k].name, sizeof out[k].name, "%s", kKernelNames[k]);
            out[k].launches = 0;
            out[k].ms = 0.0;
            out[k].bytes = 0.0;
        }
        for (auto& r : recs) {
            float ms = 0.f;
            CUDA_OK(cudaEventElapsedTime(&ms, r.e0, r.e1));
            out[r.kind].launches++;
            out[r.kind].ms += ms;
            out[r.kind].bytes += r.bytes;
            cudaEventDestroy(r.e0);
            cudaEventDestroy(r.e1);
        }
        *count = KK_COUNT;
    });
}

int scfr_timeline(scfr_handle* h, int64_t n, scfr_kernel_span* out, int cap, int* count) {
    NvtxRange nvtx("scfr_timeline");
    return guarded([&] {
        if (!h || !out || !count) fail(SCFR_EINVAL, "bad arguments");
        if (n < 1 || (h->overlap && n < 2)) fail(SCFR_EINVAL, "n_iter must be >= 1 (>= 2 when overlapped)");
        if (is_persistent(h->engine)) fail(SCFR_EINVAL, "the timeline covers the level engine's launches");
        set_device(h);
        add_weights(h, n);
        preset_constant_rows(h);
        // a recording copy of the iteration graph (the overlapped body when
        // the handle runs overlapped iterations: prologue, n - 1 recorded
        // bodies, epilogue)
        std::vector<LaunchBase::TlRec> kinds;
        DevBuf<unsigned long long> buf;
        {
            AllocStream alloc_on(h->stream);
            buf.alloc(2 * 4096);
        }
        Launcher L(h);
        L.tl = buf.p;
        L.tl_kinds = &kinds;
        cudaGraph_t graph;
        cudaGraphExec_t exec;
        CUDA_OK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
        if (h->overlap) L.body();
        else L.iteration();
        CUDA_OK(cudaStreamEndCapture(h->stream, &graph));
        CUDA_OK(cudaGraphInstantiate(&exec, graph, cudaGraphInstantiateFlagUseNodePriority));
        cudaGraphDestroy(graph);
        const int m = (int)kinds.size();
        if (m > 4096 || m > cap) {
            cudaGraphExecDestroy(exec);
            fail(SCFR_EINVAL, "%d launches per iteration exceed the output capacity", m);
        }
        if (h->overlap) {
            if (!h->exec_body) build_overlap_graphs(h);
            CUDA_OK(cudaGraphLaunch(h->exec_pro, h->stream));
        }
        const int64_t rec = h->overlap ? n - 1 : n;
        std::vector<unsigned long long> host(2 * m);
        std::vector<double> st(m, 0.0), en(m, 0.0);
        for (int64_t i = 0; i < rec; ++i) {
            CUDA_OK(cudaMemsetAsync(buf.p, 0, 2 * m * sizeof(unsigned long long), h->stream));
            CUDA_OK(cudaGraphLaunch(exec, h->stream));
            CUDA_OK(cudaMemcpyAsync(host.data(), buf.p, 2 * m * sizeof(unsigned long long),
                                    cudaMemcpyDeviceToHost, h->stream));
            CUDA_OK(cudaStreamSynchronize(h->stream));
            unsigned long long t0 = ~0ull;
            for (int k = 0; k < m; ++k) t0 = std::min(t0, ~host[2 * k]);
            for (int k = 0; k < m; ++k) {
                st[k] += (double)(long long)(~host[2 * k] - t0) / 1e3;
                en[k] += (double)(long long)(host[2 * k + 1] - t0) / 1e3;
            }
        }
        if (h->overlap) CUDA_OK(cudaGraphLaunch(h->exec_epi, h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));
        cudaGraphExecDestroy(exec);
        h->timed = false;
        h->t += n;
        h->sub_stale = h->subtree;
        h->launches += h->overlap ? h->nodes_pro + rec * m + h->nodes_epi : n * m;
        for (int k = 0; k < m; ++k) {
            std::snprintf(out[k].name, sizeof out[k].name, "%s", kKernelNames[kinds[k].kind]);
            out[k].kind = kinds[k].kind;
            out[k].stream = kinds[k].stream;
            out[k].bytes = kinds[k].bytes;
            out[k].start_us = st[k] / (double)rec;
            out[k].end_us = en[k] / (double)rec;
        }
        *count = m;
    });
}

int scfr_set_schedule(scfr_handle* h, int solve, const double* w, const double* pf, const double* nf, int64_t n) {
    return guarded([&] {
        if (!h) fail(SCFR_EINVAL, "handle is NULL");
        if (n < 0) fail(SCFR_EINVAL, "n must be >= 0");
        if (solve < -1 || solve >= h->B) fail(SCFR_EINVAL, "solve out of range");
        if (n == 0 || (!w && !pf && !nf)) return;
        for (int64_t i = 0; i < n; ++i)
            if ((w && !std::isfinite(w[i])) || (pf && !std::isfinite(pf[i])) || (nf && !std::isfinite(nf[i])))
                fail(SCFR_EINVAL, "schedule entry %lld is not finite", (long long)i);
        set_device(h);
        ensure_schedule(h, h->t + n);
        for (int k = solve < 0 ? 0 : solve; k < (solve < 0 ? h->B : solve + 1); ++k)
            for (int64_t i = 0; i < n; ++i) {
                const size_t q = (size_t)k * h->cap + h->t + i;
                if (w) h->w_host[q] = w[i];
                if (pf) h->pf_host[q] = pf[i];
                if (nf) h->nf_host[q] = nf[i];
            }
        upload_schedule(h);
    });
}

int scfr_synchronize(scfr_handle* h) {
    return guarded([&] {
        if (!h) fail(SCFR_EINVAL, "handle is NULL");
        set_device(h);
        CUDA_OK(cudaStreamSynchronize(h->stream));
    });
}

// Device-side copy of the whole iteration state (every solve of the batch)
// and of the host counters: a coarse-to-fine time-to-target search replays
// from it instead of paying a best response after every iteration.
int scfr_snapshot(scfr_handle* h, int restore) {
    NvtxRange nvtx("scfr_snapshot");
    return guarded([&] {
        if (!h) fail(SCFR_EINVAL, "handle is NULL");
        if (restore != 0 && restore != 1) fail(SCFR_EINVAL, "restore must be 0 (save) or 1 (restore)");
        set_device(h);
        Snapshot& sn = h->snap;
        if (restore && !sn.valid) fail(SCFR_EINVAL, "no snapshot saved");
        AllocStream alloc_on(h->stream);
        auto copy = [&](DevBuf<double>& live, DevBuf<double>& saved) {
            if (!restore && saved.n != live.n) saved.alloc(live.n);
            if (live.n)
                CUDA_OK(cudaMemcpyAsync(restore ? live.p : saved.p, restore ? saved.p : live.p,
                                        live.n * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
        };
        for (int k = 0; k < 2; ++k) {
            Player& P = h->P[k];
            DevBuf<double>* live[] = {&P.r, &P.b, &P.x, &P.xpost, &P.avg, &P.u, &P.V};
            for (int a = 0; a < 7; ++a) copy(*live[a], sn.buf[k][a]);
        }
        if (!restore) {
            if (!sn.tdev.n) sn.tdev.alloc(1);
            CUDA_OK(cudaMemcpyAsync(sn.tdev.p, h->tdev.p, sizeof(long long), cudaMemcpyDeviceToDevice, h->stream));
            sn.t = h->t;
            sn.avg_weight = h->avg_weight;
            sn.valid = true;
        } else {
            CUDA_OK(cudaMemcpyAsync(h->tdev.p, sn.tdev.p, sizeof(long long), cudaMemcpyDeviceToDevice, h->stream));
            h->t = sn.t;
            h->avg_weight = sn.avg_weight;
            h->sub_stale = h->subtree;
        }
    });
}

int scfr_iterations(const scfr_handle* h, int64_t* out) {
    return guarded([&] {
        if (!h || !out) fail(SCFR_EINVAL, "NULL argument");
        *out = h->t;
    });
}

int scfr_avg_weight(const scfr_handle* h, int player, int solve, double* out) {
    return guarded([&] {
        check_player(h, player, solve);
        if (!out) fail(SCFR_EINVAL, "NULL argument");
        *out = h->avg_weight[solve];
    });
}

int scfr_read_state(scfr_handle* h, int player, int solve, int which, double* host_out) {
    NvtxRange nvtx("scfr_read_state");
    return guarded([&] {
        check_player(h, player, solve);
        if (!host_out) fail(SCFR_EINVAL, "NULL argument");
        set_device(h);
        gather_subtrees(h);
        Player& P = h->P[player - 1];
        const double* src = nullptr;
        size_t off = 0, cnt = P.S;
        switch (which) {
            case SCFR_STATE_REGRETS: src = P.r.p; off = 1; cnt = P.S - 1; break;
            // Non-predictive variants regret-match inside OBS, so this is the
            // behaviour the *next* iteration will play.
            case SCFR_STATE_BEHAVIOR: src = P.b.p; off = 1; cnt = P.S - 1; break;
            case SCFR_STATE_ACCUM:
                expand_leaves(h, player, P.avg, solve);
                src = P.avg.p;
                break;
            case SCFR_STATE_UTILITY: src = P.u.p; break;
            default: fail(SCFR_EINVAL, "unknown state selector");
        }
        src = orig_order(h, player, src, solve);
        read_to_host(h, host_out, src + off, cnt);
    });
}

int scfr_read_average(scfr_handle* h, int player, int solve, double* host_out) {
    NvtxRange nvtx("scfr_read_average");
    return guarded([&] {
        check_player(h, player, solve);
        if (!host_out) fail(SCFR_EINVAL, "NULL argument");
        if (h->avg_weight[solve] == 0.0) fail(SCFR_EINVAL, "no strategies accumulated yet");
        set_device(h);
        gather_subtrees(h);
        Player& P = h->P[player - 1];
        // avg_accum / avg_weight (IEEE division, as the reference's numpy divide)
        expand_leaves(h, player, P.avg, solve);
        const double* avg = orig_order(h, player, P.avg.p, solve);
        k_normalize<<<grid_for(P.S), TPB, 0, h->stream>>>(avg, h->avg_weight[solve], P.xbar.p, P.S);
        CUDA_OK(cudaGetLastError());
        read_to_host(h, host_out, P.xbar.p, P.S);
    });
}

int scfr_read_averages(scfr_handle* h, int solve, double* host_out1, double* host_out2) {
    NvtxRange nvtx("scfr_read_averages");
    return guarded([&] {
        check_player(h, 1, solve);
        if (!host_out1 || !host_out2) fail(SCFR_EINVAL, "NULL argument");
        if (h->avg_weight[solve] == 0.0) fail(SCFR_EINVAL, "no strategies accumulated yet");
        set_device(h);
        gather_subtrees(h);
        ReadSeg seg[2];
        for (int k = 0; k < 2; ++k) {  // both normalisations queued before the first DMA
            Player& P = h->P[k];
            expand_leaves(h, k + 1, P.avg, solve);
            const double* avg = orig_order(h, k + 1, P.avg.p, solve);
            k_normalize<<<grid_for(P.S), TPB, 0, h->stream>>>(avg, h->avg_weight[solve], P.xbar.p, P.S);
            CUDA_OK(cudaGetLastError());
            seg[k] = ReadSeg{k == 0 ? host_out1 : host_out2, P.xbar.p, (size_t)P.S};
        }
        read_to_host_multi(h, seg, 2);
    });
}

int scfr_read_current(scfr_handle* h, int player, int solve, double* host_out) {
    return guarded([&] {
        check_player(h, player, solve);
        if (!host_out) fail(SCFR_EINVAL, "NULL argument");
        if (h->t == 0) fail(SCFR_EINVAL, "no iteration has run yet");
        set_device(h);
        gather_subtrees(h);
        Player& P = h->P[player - 1];
        expand_leaves(h, player, P.x, solve);
        read_to_host(h, host_out, orig_order(h, player, P.x.p, solve), P.S);
    });
}

int scfr_exploitability(scfr_handle* h, int solve, int which, double* expl, double* br1, double* br2) {
    NvtxRange nvtx("scfr_exploitability");
    return guarded([&] {
        check_player(h, 1, solve);
        if (which != 0 && which != 1) fail(SCFR_EINVAL, "which must be 0 (average) or 1 (current)");
        if (which == 1 && h->t == 0) fail(SCFR_EINVAL, "no iteration has run yet");
        set_device(h);
        gather_subtrees(h);
        // br1 against x2, then br2 against x1 (pkg/metrics.py:59-68); xbar
        // buffers are per player so both profiles can be live at once.
        const double* x2 = profile(h, 2, solve, which);
        const double b1 = best_response(h, 1, x2);
        const double* x1 = profile(h, 1, solve, which);
        const double b2 = best_response(h, 2, x1);
        if (br1) *br1 = b1;
        if (br2) *br2 = b2;
        if (expl) *expl = (b1 + b2) / 2.0;
    });
}

static double host_dot(const std::vector<double>& x, const std::vector<double>& g) {
    double acc = 0.0;  // Backend.dot: sequential (pkg/kernels.py:278-283)
    for (size_t i = 0; i < x.size(); ++i) acc = acc + x[i] * g[i];
    return acc;
}

int scfr_expected_value(scfr_handle* h, int solve, double* out) {
    return guarded([&] {
        check_player(h, 1, solve);
        if (!out) fail(SCFR_EINVAL, "NULL argument");
        set_device(h);
        gather_subtrees(h);
        const double* x2 = profile(h, 2, solve, 0);
        Player& A = h->P[0];
        solve_spmv(h, h->U, x2, A.g.p, false);
        profile(h, 1, solve, 0);
        std::vector<double> g(A.S), x(A.S);
        CUDA_OK(copy_async(g.data(), A.g.p, A.S * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        CUDA_OK(copy_async(x.data(), A.xbar.p, A.S * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));
        *out = host_dot(x, g);
    });
}

int scfr_best_response_values(scfr_handle* h, const double* x1, const double* x2, double* br1,
                              double* br2) {
    return guarded([&] {
        if (!h || !x1 || !x2) fail(SCFR_EINVAL, "NULL argument");
        set_device(h);
        Player& A = h->P[0];
        Player& Bp = h->P[1];
        CUDA_OK(copy_async(A.xbar.p, x1, A.S * sizeof(double), cudaMemcpyHostToDevice, h->stream));
        CUDA_OK(copy_async(Bp.xbar.p, x2, Bp.S * sizeof(double), cudaMemcpyHostToDevice, h->stream));
        const double b1 = best_response(h, 1, Bp.xbar.p);
        const double b2 = best_response(h, 2, A.xbar.p);
        if (br1) *br1 = b1;
        if (br2) *br2 = b2;
    });
}

int scfr_expected_value_of(scfr_handle* h, const double* x1, const double* x2, double* out) {
    return guarded([&] {
        if (!h || !x1 || !x2 || !out) fail(SCFR_EINVAL, "NULL argument");
        set_device(h);
        Player& A = h->P[0];
        Player& Bp = h->P[1];
        CUDA_OK(copy_async(Bp.xbar.p, x2, Bp.S * sizeof(double), cudaMemcpyHostToDevice, h->stream));
        solve_spmv(h, h->U, Bp.xbar.p, A.g.p, false);
        std::vector<double> g(A.S), x(x1, x1 + A.S);
        CUDA_OK(copy_async(g.data(), A.g.p, A.S * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));
        *out = host_dot(x, g);
    });
}

int scfr_status(scfr_handle* h, int* nonfinite) {
    return guarded([&] {
        if (!h || !nonfinite) fail(SCFR_EINVAL, "NULL argument");
        set_device(h);
        int v = 0;
        CUDA_OK(copy_async(&v, h->nonfinite.p, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));
        *nonfinite = v;
    });
}

int scfr_device_bytes(const scfr_handle* h, int64_t* out) {
    return guarded([&] {
        if (!h || !out) fail(SCFR_EINVAL, "NULL argument");
        int64_t s = 0;
        for (const Player& P : h->P) {
            s += P.seq_ptr.bytes() + P.dp_parent.bytes() + P.child.bytes();
            for (const DevBuf<double>* b : {&P.r, &P.b, &P.x, &P.xpost, &P.avg, &P.u, &P.V, &P.g, &P.W, &P.xbar})
                s += b->bytes();
        }
        for (const DevCsr* m : {&h->U, &h->UT, &h->tM[0], &h->tM[1]})
            s += m->indptr.bytes() + m->indices.bytes() + m->data.bytes();
        for (const TilePlayer& tp : h->tp)
            s += tp.seq_ptr.bytes() + tp.dp_parent.bytes() + tp.off.bytes() + tp.sperm.bytes() +
                 tp.child.bytes() + tp.shape.bytes() + tp.ticket.bytes() + tp.gat.bytes();
        s += h->wsched.bytes() + h->pfsched.bytes() + h->nfsched.bytes();
        *out = s;
    });
}

int scfr_launch_count(const scfr_handle* h, int64_t* out) {
    return guarded([&] {
        if (!h || !out) fail(SCFR_EINVAL, "NULL argument");
        *out = h->launches;
    });
}

int scfr_last_step_ms(scfr_handle* h, double* total_ms) {
    return guarded([&] {
        if (!h || !total_ms) fail(SCFR_EINVAL, "NULL argument");
        if (!h->timed) fail(SCFR_EINVAL, "no timed step has run yet");
        set_device(h);
        CUDA_OK(cudaEventSynchronize(h->ev1));
        float ms = 0.f;
        CUDA_OK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
        *total_ms = ms;
    });
}

int scfr_transfer_bytes(int64_t* h2d, int64_t* d2h) {
    return guarded([&] {
        if (!h2d || !d2h) fail(SCFR_EINVAL, "NULL argument");
        *h2d = g_h2d.load();
        *d2h = g_d2h.load();
    });
}

int scfr_destroy(scfr_handle* h) {
    return guarded([&] {
        if (!h) return;
        cudaSetDevice(h->device);
        delete h;  // ~scfr_handle drains the stream and destroys the communicator
    });
}

}  // extern "C"
