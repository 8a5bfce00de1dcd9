// Forest mode of the level engine: one streaming kernel per pass.
//
// The level engine runs one launch per DP level and pass (23 launches per
// Goofspiel-5 PCFR+ iteration), and every level's V / x makes a round trip
// through HBM to the next launch.  Here each player's decision process is cut
// at a split level `ls`:
//
//   * Forest (levels [ls, L)).  Breadth-first numbering makes the
//     descendants of a contiguous range of level-ls DPs (roots) a contiguous
//     range at every deeper level (pkg/decision_process.py:9-13).  The host
//     records, for every root boundary, the DP / sequence / payoff-nnz
//     position per level (`tab`), and cuts the roots into items whose
//     subtrees fit a shared-memory stage.  A persistent CTA streams its items
//     through two stages: one thread issues TMA bulk copies (cp.async.bulk,
//     mbarrier completion) of the next item's contiguous r / b / u / avg /
//     payoff / table ranges while the CTA computes the current one.  Inside
//     an item every warp owns a contiguous range of roots and walks their
//     subtrees level by level with only __syncwarp between levels: lanes run
//     the group-mode per-DP code (kernels.cuh, lane = (DP, action)) on
//     shared-memory windows, so inner V / x never leave the chip; results go
//     out with coalesced stores.
//   * Top (levels [0, ls), a few thousand DPs).  Bottom-up passes finish it
//     by last arrival: a root (or top DP) publishes its V, fences, and bumps
//     its parent DP's counter; the warp that completes a parent computes it
//     (warp-per-DP code, L2 loads) and carries on upwards.  The warp that
//     completes the empty sequence of the last solve advances the iteration
//     counter.  Top-down passes recompute a top sequence's x from its
//     ancestor chain (x = b_a·(…·(b_0·1.0))): every root parent on the fly,
//     and every top sequence once (x, average) across the grid.
//
// Per-DP arithmetic is the code of the other engines, so the iterates stay
// bit-identical to the reference.  A predictive alt iteration is 5 launches
// (PRED both players, TD + average both, OBS₁, TD of bcur into x₁', OBS₂).
//
// The forest needs, below the split, every DP of level k+1 to hang under a
// sequence of level k with non-decreasing parents (children of consecutive
// sequences consecutive).  Trees without it (e.g. merged levels whose DPs
// sit at two node depths) keep the plain level engine.

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <type_traits>
#include <vector>

#include "host_par.h"
#include "runtime.h"

namespace scfr {

// Forest CTA: kFW independent warp pipelines (two shared-memory stages each).
constexpr int kFW = 4;
constexpr int kFT = kFW * 32;
constexpr int kFMinB = 6;    // CTAs per SM the register budget allows

// Phase trace (scfr_trace_*; tuning only): CTA 0 of a launch records
// (clock64 << 8 | tag) values.
__device__ long long* g_trace = nullptr;
__device__ int g_trace_cap = 0;
__device__ int g_trace_n = 0;
__device__ __forceinline__ void trace(int tag) {
    if (g_trace && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
        const int i = atomicAdd(&g_trace_n, 1);
        if (i < g_trace_cap) g_trace[i] = ((long long)clock64() << 8) | tag;
    }
}

// ---------------------------------------------------------------------------
// TMA bulk copies (global -> shared) completing on an mbarrier.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Generic-proxy accesses to a stage are ordered before the async proxy (the
// next bulk copy) overwrites it.
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

// ---------------------------------------------------------------------------
// Stage layout: the same function sizes stages on the host and carves them
// on the device.  A stage is [FHdr per level][FItem][table rows][level
// arrays].  Staged arrays are read as whole 16-byte granules (alo = the
// first element of the granule holding the range's first element), so a
// stage holds a slightly wider window of each; computed arrays are exact
// windows.  Indices are >= 0 and E is a power of two.

__host__ __device__ inline int f_alo(int e, int E) { return e & ~(E - 1); }
__host__ __device__ inline int f_ahi(int e, int E) { return (e + E - 1) & ~(E - 1); }
__host__ __device__ inline int f_up16(int b) { return (b + 15) & ~15; }

struct FItem {  // one stage's item: root range and the staged table rows
    int r0, r1;
    int tab_off, tab_alo, tab_cnt;
};

__host__ __device__ inline int f_hdr_bytes(int nla) { return f_up16(nla * (int)sizeof(FHdr) + (int)sizeof(FItem)); }

// Arrays of forest level L (bounds in h) for one pass, from offset `cur`.
// leaf: the level is the deepest one and all forced moves into end nodes
// (kernels.cuh leaf_note): PRED does not touch it (the parent reads the
// prediction itself) and OBS only computes its utilities (the parent reads
// them as the child values).  `so`: the per-solve element offset of
// seq-indexed state (alignment only).  Returns the staged bytes.
__host__ __device__ inline int layout_level(int pass, const FLev& L, FHdr& h, int v, int so, bool leaf, int& cur) {
    int tx = 0;
    auto staged = [&](int a, int lo, int hi, int esz, int base) {
        const int E = 16 / esz;
        const int al = f_alo(base + lo, E), ah = f_ahi(base + hi, E);
        h.off[a] = cur;
        h.alo[a] = al - base;
        h.cnt[a] = hi > lo ? ah - al : 0;
        tx += h.cnt[a] * esz;
        cur = f_up16(cur + h.cnt[a] * esz);
    };
    auto window = [&](int a, int n, int esz) {
        h.off[a] = cur;
        h.alo[a] = 0;
        h.cnt[a] = 0;  // computed here, not staged
        cur = f_up16(cur + n * esz);
    };
    for (int a = 0; a < FA_N; ++a) h.cnt[a] = 0;
    const int ns = h.s1 - h.s0, nj = h.j1 - h.j0;
    const bool single = L.un == 1;
    if (pass == FP_OBS || pass == FP_PRED) {
        if (L.rows) {
            if (pass == FP_OBS) {  // fused payoff rows: indices and values staged, x gathered
                staged(FA_IX, h.k0, h.k1, 4, 0);
                staged(FA_D, h.k0, h.k1, v, 0);
                if (L.rc <= 0) staged(FA_IP, h.s0, h.s1 + 1, 4, 0);
                window(FA_U, ns, v);
            } else {
                staged(FA_M, h.s0, h.s1, v, so);
            }
        }
        if (leaf) return tx;
        if (!single) {
            staged(FA_R, h.s0, h.s1, v, so);
            staged(FA_B, h.s0, h.s1, v, so);
        }
        if (L.un <= 0) staged(FA_SP, h.j0, h.j1 + 1, 4, 0);
        if (L.cn < 0) staged(FA_CH, h.s0, h.s1, 8, 0);
        window(FA_V, nj, v);
    } else {
        if (!single) staged(FA_B, h.s0, h.s1, v, so);
        if (pass == FP_TDAVG) staged(FA_AVG, h.s0, h.s1, v, so);
        if (L.un <= 0) staged(FA_SP, h.j0, h.j1 + 1, 4, 0);
        if (L.pc <= 0) staged(FA_PAR, h.j0, h.j1, 4, 0);
        window(FA_X, ns, v);
    }
    return tx;
}

// Whole-stage layout (host sizing, worst-case alignment slack via `so`).
inline int forest_layout(int pass, int nl, int nla, const FLev* lv, bool leaf, FItem& it, FHdr* hd, int v, int so) {
    const int lo = it.r0 * nla * 3, hi = (it.r1 + 1) * nla * 3;
    const int al = f_alo(lo, 4), ah = f_ahi(hi, 4);
    it.tab_off = f_hdr_bytes(nla);
    it.tab_alo = al;
    it.tab_cnt = ah - al;
    int cur = f_up16(it.tab_off + it.tab_cnt * 4);
    for (int k = 0; k < nl; ++k) layout_level(pass, lv[k], hd[k], v, so, leaf && k == nl - 1, cur);
    return cur;
}

// ---------------------------------------------------------------------------
// Forest kernel.

template <class T>
__device__ __forceinline__ T* at(unsigned char* stage, const FHdr& h, int a) {
    return reinterpret_cast<T*>(stage + h.off[a]) - h.alo[a];
}

// Root range [r0, r1) of item `item`.
template <class R>
__device__ __forceinline__ void item_roots(const ForestTaskT<R>& t, int item, int& r0, int& r1) {
    if (t.aff) {
        r0 = item * t.aR;
        r1 = min(r0 + t.aR, t.nroots);
    } else {
        r0 = __ldg(t.items + item);
        r1 = __ldg(t.items + item + 1);
    }
}

// The whole warp lays out `item` into stage `st` (lane k: level k) and
// issues its bulk copies on `bar`.
template <int PASS, class R>
__device__ __forceinline__ void forest_issue(const ForestTaskT<R>& t, const FLev* lvs, int item, unsigned char* st,
                                             uint64_t* bar, int so) {
    const int lane = threadIdx.x & 31;
    FHdr* hd = reinterpret_cast<FHdr*>(st);
    FItem* fi = reinterpret_cast<FItem*>(st + t.nla * sizeof(FHdr));
    FItem it;
    item_roots(t, item, it.r0, it.r1);
    it.tab_off = f_hdr_bytes(t.nla);
    it.tab_alo = 0;
    it.tab_cnt = 0;
    const int base0 = it.tab_off;
    FHdr h;
    int lb = 0, tx = 0;
    if (lane < t.nl) {
        const FLev& L = lvs[lane];
        if (t.aff) {  // affine forest: positions linear in the root index
            h.j0 = L.aj0 + it.r0 * L.dj;
            h.s0 = L.as0 + it.r0 * L.ds;
            h.k0 = L.ak0 + it.r0 * L.dk;
            h.j1 = L.aj0 + it.r1 * L.dj;
            h.s1 = L.as0 + it.r1 * L.ds;
            h.k1 = L.ak0 + it.r1 * L.dk;
        } else {
            const int* ta = t.tab + (size_t)it.r0 * t.nla * 3 + 3 * lane;
            const int* tb = t.tab + (size_t)it.r1 * t.nla * 3 + 3 * lane;
            h.j0 = __ldg(ta);
            h.s0 = __ldg(ta + 1);
            h.k0 = __ldg(ta + 2);
            h.j1 = __ldg(tb);
            h.s1 = __ldg(tb + 1);
            h.k1 = __ldg(tb + 2);
        }
        tx = layout_level(PASS, lvs[lane], h, (int)sizeof(R), so, t.leaf && lane == t.nl - 1, lb);
    }
    int base = lb;  // inclusive scan of the level sizes over lanes 0..nl-1
    for (int d = 1; d < kFMax; d <<= 1) {
        const int y = __shfl_up_sync(kFullMask, base, d);
        if (lane >= d) base += y;
    }
    base = base0 + base - lb;
    for (int d = 16; d > 0; d >>= 1) tx += __shfl_xor_sync(kFullMask, tx, d);
    if (lane < t.nl) {
        for (int a = 0; a < FA_N; ++a) h.off[a] += base;
        hd[lane] = h;
    }
    if (lane == 0) {
        *fi = it;
        mbar_expect_tx(bar, (uint32_t)tx);
    }
    __syncwarp();
    if (lane < t.nl) {
        auto go = [&](int a, const void* src, int esz) {
            if (h.cnt[a] > 0)
                bulk_g2s(st + h.off[a], static_cast<const unsigned char*>(src) + (ptrdiff_t)h.alo[a] * esz,
                         (uint32_t)(h.cnt[a] * esz), bar);
        };
        if (PASS == FP_OBS || PASS == FP_PRED) {
            go(FA_R, t.r + so, sizeof(R));
            go(FA_B, t.b + so, sizeof(R));
            go(FA_M, t.u + so, sizeof(R));
            go(FA_IX, t.ix, 4);
            go(FA_D, t.d, sizeof(R));
            go(FA_IP, t.ip, 4);
            go(FA_CH, t.child, 8);
        } else {
            go(FA_B, t.src + so, sizeof(R));
            go(FA_AVG, t.avg + so, sizeof(R));
            go(FA_PAR, t.dp_parent, 4);
        }
        go(FA_SP, t.seq_ptr, 4);
    }
}

template <class R>
__device__ __forceinline__ DevTree level_tree(const FLev& L, unsigned char* st, const FHdr& h) {
    DevTree T;
    T.seq_ptr = L.un <= 0 ? at<int>(st, h, FA_SP) : nullptr;
    T.child = L.cn < 0 ? at<int2>(st, h, FA_CH) : nullptr;
    T.dp_parent = L.pc <= 0 ? at<int>(st, h, FA_PAR) : nullptr;
    T.j_lo = L.j_lo;
    T.s_lo = L.s_lo;
    T.un = L.un;
    T.cn = L.cn;
    T.c_lo = L.c_lo;
    T.pc = L.pc;
    T.p_lo = L.p_lo;
    return T;
}

template <class R>
__device__ __forceinline__ DevTree top_tree(const ForestTaskT<R>& t, int l) {
    const FLev& L = t.tlv[l];
    DevTree T{t.seq_ptr, t.dp_parent, t.child};
    T.j_lo = L.j_lo;
    T.s_lo = L.s_lo;
    T.un = L.un;
    T.cn = L.cn;
    T.c_lo = L.c_lo;
    T.pc = L.pc;
    T.p_lo = L.p_lo;
    return T;
}

// DP of parent sequence p (p in the top): the virtual root index Jtop for the
// empty sequence.
template <class R>
__device__ __forceinline__ int parent_dp(const ForestTaskT<R>& t, int p) {
    return p == 0 ? t.Jtop : __ldg(t.top_sdp + p);
}

// Last arrival: the warp has published V of DPs whose parent DPs are in `q`
// (one per lane where `mine`); it completes every parent it is the last
// child of, then their parents, up to the empty sequence.
template <int PASS, class R>
__device__ __noinline__ void top_cascade(const ForestTaskT<R>& t, const KParams& kp, R pf, R nf, int q, bool mine,
                                         int so) {
    const int lane = threadIdx.x & 31;
    unsigned* cnt = t.cnt + (size_t)blockIdx.y * (t.Jtop + 1);
    bool last = false;
    if (mine) last = atomicAdd(cnt + q, 1u) == (unsigned)__ldg(t.nch + q) - 1u;
    unsigned m = __ballot_sync(kFullMask, last);
    while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        int d = __shfl_sync(kFullMask, q, src);
        while (true) {
            __threadfence();  // acquire: the siblings' V
            if (d == t.Jtop) {  // the empty sequence: the pass is complete for this solve
                if (lane == 0) {
                    cnt[d] = 0u;
                    if (t.tick) {
                        __threadfence();
                        if (atomicAdd(t.done, 1u) == (unsigned)t.ntick - 1u) {
                            *t.done = 0u;
                            *t.tick += 1;
                        }
                    }
                }
                break;
            }
            int l = 0;
            while (l + 1 < t.ls && d >= t.tlo[l + 1]) ++l;
            const DevTree T = top_tree(t, l);
            const FLev& L = t.tlv[l];
            R* V = t.V + (size_t)blockIdx.y * t.J;
            if constexpr (PASS == FP_OBS) {
                FuseUT<R> fu{};
                R* u = nullptr;
                if (L.rows) {
                    u = t.uo + so;
                    fu = FuseUT<R>{t.ip, t.ix, t.d, t.xo + (size_t)blockIdx.y * t.xo_sx, t.neg};
                    fu.rc = L.rc;
                    fu.rs0 = L.rs0;
                    fu.rk0 = L.rk0;
                }
                obs_dp_warp<LdL2s>(T, d, u, t.r + so, t.b + so, V, kp.post, pf, nf, t.do_rm != 0, kp.nonfinite,
                                   lane, fu, static_cast<const R*>(nullptr), t.bo == t.b ? nullptr : t.bo + so);
            } else {
                pred_dp_warp<LdL2s>(T, d, L.rows ? t.u + so : nullptr, t.r + so, t.b + so, V, kp.plus != 0, lane,
                                    static_cast<const R*>(nullptr));
            }
            __syncwarp();
            __threadfence();
            int up = 0;
            if (lane == 0) {
                cnt[d] = 0u;  // re-armed for the next launch
                const int nd = parent_dp(t, __ldg(t.dp_parent + d));
                up = atomicAdd(cnt + nd, 1u) == (unsigned)__ldg(t.nch + nd) - 1u ? nd + 1 : 0;
            }
            up = __shfl_sync(kFullMask, up, 0);
            if (!up) break;
            d = up - 1;
        }
    }
}

// Bottom-up pass (OBS or PRED) over one item, deep -> shallow.
template <int PASS, int MAXA, class R>
__device__ __forceinline__ void warp_up(const ForestTaskT<R>& t, const FLev* lvs, unsigned char* st,
                                        const KParams& kp, R pf, R nf, int so, const R* xo) {
    const int lane = threadIdx.x & 31;
    const FHdr* hd = reinterpret_cast<const FHdr*>(st);
    const R* Vc = nullptr;  // child values of the level being processed
    for (int k = t.nl - 1; k >= 0; --k) {
        const FHdr& h = hd[k];
        const FLev L = lvs[k];
        const bool single = L.un == 1;
        const bool leaf = t.leaf && k == t.nl - 1;
        R* us = nullptr;
        if (PASS == FP_OBS && L.rows) {
            // fused payoff rows: u[s] = (±) row s of M applied to the
            // opponent's x, summed in CSR order from 0.0 (pkg/kernels.py:149-154,
            // as spmv_range), gathers batched so several are in flight
            const int* ix = at<int>(st, h, FA_IX);
            const R* dd = at<R>(st, h, FA_D);
            R* u = reinterpret_cast<R*>(st + h.off[FA_U]) - h.s0;
            bool bad = false;
            if (L.rc == 1) {  // one non-zero per row: row s is entry k0 + (s - s0)
                constexpr int UR = 8;
                for (int sb = h.s0; sb < h.s1; sb += 32 * UR) {
                    R xv[UR];
#pragma unroll
                    for (int i = 0; i < UR; ++i) {
                        const int s = sb + i * 32 + lane;
                        if (s < h.s1) xv[i] = xo[ix[h.k0 + (s - h.s0)]];
                    }
#pragma unroll
                    for (int i = 0; i < UR; ++i) {
                        const int s = sb + i * 32 + lane;
                        if (s < h.s1) {
                            R acc = dadd(R(0), dmul(dd[h.k0 + (s - h.s0)], xv[i]));
                            if (t.neg) acc = dmul(R(-1), acc);
                            bad |= !isfinite(acc);
                            u[s] = acc;
                            t.uo[so + s] = acc;  // the next iteration's prediction
                        }
                    }
                }
            } else {
                const int* ip = L.rc > 0 ? nullptr : at<int>(st, h, FA_IP);
                for (int s = h.s0 + lane; s < h.s1; s += 32) {
                    int q0, q1;
                    if (L.rc > 0) {
                        q0 = h.k0 + (s - h.s0) * L.rc;
                        q1 = q0 + L.rc;
                    } else {
                        q0 = ip[s];
                        q1 = ip[s + 1];
                    }
                    R acc = R(0);
                    int q = q0;
                    for (; q + 4 <= q1; q += 4) {  // loads first, adds in order
                        const R x0 = xo[ix[q]], x1 = xo[ix[q + 1]], x2 = xo[ix[q + 2]], x3 = xo[ix[q + 3]];
                        acc = dadd(dadd(dadd(dadd(acc, dmul(dd[q], x0)), dmul(dd[q + 1], x1)), dmul(dd[q + 2], x2)),
                                   dmul(dd[q + 3], x3));
                    }
                    for (; q < q1; ++q) acc = dadd(acc, dmul(dd[q], xo[ix[q]]));
                    if (t.neg) acc = dmul(R(-1), acc);
                    bad |= !isfinite(acc);
                    u[s] = acc;
                    t.uo[so + s] = acc;
                }
            }
            if (bad) atomicOr(kp.nonfinite, 1);
            __syncwarp();
            us = u;
        } else if (PASS == FP_PRED && L.rows) {
            us = at<R>(st, h, FA_M);
        }
        if (leaf) {  // the parent reads the utility / prediction as the child value
            const int sh = L.s_lo - L.j_lo;
            Vc = (us ? us : (PASS == FP_OBS ? t.uo : t.u) + so) + sh;
            continue;
        }
        R* const Vs = reinterpret_cast<R*>(st + h.off[FA_V]) - h.j0;
        const DevTree T = level_tree<R>(L, st, h);
        R* rs = single ? nullptr : at<R>(st, h, FA_R);
        R* bs = single ? nullptr : at<R>(st, h, FA_B);
        if (L.un >= 2 && L.un <= 16) {  // group mode: lane = (DP, action)
            auto run = [&](auto width) {
                constexpr int N = decltype(width)::value;
                const int n = N > 0 ? N : L.un, G = 32 / n, g = lane / n, a = lane - g * n, gb = g * n;
                for (int base = h.j0; base < h.j1; base += G) {
                    const int j = base + g;
                    const bool valid = g < G && j < h.j1;
                    if constexpr (PASS == FP_OBS)
                        obs_dp_group<LdS, N>(T, valid ? j : h.j0, valid, a, gb, n, us, rs, bs, Vs, kp.post, pf, nf,
                                             t.do_rm != 0, kp.nonfinite, FuseUT<R>{}, Vc);
                    else
                        pred_dp_group<LdS, N>(T, valid ? j : h.j0, valid, a, gb, n, us, rs, bs, Vs, kp.plus != 0,
                                              Vc);
                }
            };
            switch (L.un) {
                case 2: run(std::integral_constant<int, 2>{}); break;
                case 3: run(std::integral_constant<int, 3>{}); break;
                case 4: run(std::integral_constant<int, 4>{}); break;
                default: run(std::integral_constant<int, 0>{}); break;
            }
        } else {
            for (int j = h.j0 + lane; j < h.j1; j += 32) {
                if constexpr (PASS == FP_OBS)
                    obs_dp<MAXA, LdS>(T, j, us, rs, bs, Vs, kp.post, pf, nf, t.do_rm != 0, kp.nonfinite,
                                      FuseUT<R>{}, Vc);
                else
                    pred_dp<MAXA, LdS>(T, j, us, rs, bs, Vs, kp.plus != 0, Vc);
            }
        }
        __syncwarp();
        if (!single) {  // coalesced write-back
            const bool wr = PASS == FP_OBS, wb = PASS == FP_PRED || t.do_rm;
            for (int s = h.s0 + lane; s < h.s1; s += 32) {
                if (wr) t.r[so + s] = rs[s];
                if (wb) t.bo[so + s] = bs[s];
            }
        }
        Vc = Vs;
        if (k == 0) {  // the roots: publish V (the top is completed after the warp's last item)
            R* Vg = t.V + (size_t)blockIdx.y * t.J;
            for (int j = h.j0 + lane; j < h.j1; j += 32) Vg[j] = Vs[j];
        }
    }
}

// x of top sequence p from its ancestor chain: b_a0·1.0, then b_a1·that, ...
// (the level engine's x[s] = b[s]·x[parent], with x[0] = 1.0; a forced
// level's b is 1.0 and is not read).
template <class R>
__device__ __forceinline__ R top_x(const ForestTaskT<R>& t, const R* src, int p) {
    if (p == 0) return R(1);
    const int* an = t.top_anc + (size_t)p * t.ls;
    int a[kTopMax];
    R bv[kTopMax];
#pragma unroll
    for (int l = 0; l < kTopMax; ++l) a[l] = l < t.ls ? __ldg(an + l) : -1;
#pragma unroll
    for (int l = 0; l < kTopMax; ++l) bv[l] = a[l] >= 0 && !(a[l] & (1 << 30)) ? src[a[l] & ~(1 << 30)] : R(1);
    R x = R(1);
#pragma unroll
    for (int l = 0; l < kTopMax; ++l)
        if (a[l] >= 0) x = dmul(bv[l], x);
    return x;
}

// Top-down pass (TD + average, TD) over one item, shallow -> deep; the
// per-sequence operations are td_dp's (kernels.cuh).
template <int PASS, class R>
__device__ __forceinline__ void warp_down(const ForestTaskT<R>& t, const FLev* lvs, unsigned char* st, R w, int so) {
    const int lane = threadIdx.x & 31;
    const FHdr* hd = reinterpret_cast<const FHdr*>(st);
    const R* srcg = t.src + so;
    for (int k = 0; k < t.nl; ++k) {
        const FHdr& h = hd[k];
        const FLev L = lvs[k];
        const bool single = L.un == 1;
        R* const xs = reinterpret_cast<R*>(st + h.off[FA_X]) - h.s0;
        const R* const xin = k == 0 ? nullptr : reinterpret_cast<const R*>(st + hd[k - 1].off[FA_X]) - hd[k - 1].s0;
        const R* src = single ? nullptr : at<R>(st, h, FA_B);
        R* av = PASS == FP_TDAVG ? at<R>(st, h, FA_AVG) : nullptr;
        const DevTree T = level_tree<R>(L, st, h);
        auto seq = [&](int s, R xp) {
            const R xa = dmul(single ? R(1) : src[s], xp);
            xs[s] = xa;
            if (PASS == FP_TDAVG) av[s] = dadd(dmul(w, xa), av[s]);
        };
        if (L.un >= 1 && L.un <= 16) {  // lane = (DP, action)
            const int n = L.un, G = 32 / n, g = lane / n, a = lane - g * n;
            for (int base = h.j0; base < h.j1; base += G) {
                const int j = base + g;
                if (g < G && j < h.j1) {
                    const int p = parent_of<LdS>(T, j);
                    seq(T.s_lo + (j - T.j_lo) * n + a, k == 0 ? top_x(t, srcg, p) : xin[p]);
                }
            }
        } else {
            for (int j = h.j0 + lane; j < h.j1; j += 32) {
                int s0, n;
                dp_range<LdS>(T, j, s0, n);
                const int p = parent_of<LdS>(T, j);
                const R xp = k == 0 ? top_x(t, srcg, p) : xin[p];
                for (int s = s0; s < s0 + n; ++s) seq(s, xp);
            }
        }
        __syncwarp();
        for (int s = h.s0 + lane; s < h.s1; s += 32) {
            t.x[so + s] = xs[s];
            if (PASS == FP_TDAVG) t.avg[so + s] = av[s];
        }
    }
}

// One task's share of a forest launch.  Every warp is an independent
// pipeline over its own items (item = gw, gw + nw, ...): it issues the
// next item's bulk copies into one of its two stages, then walks the
// current item's subtrees from the other.
template <int PASS, int MAXA, class R>
__device__ __forceinline__ void forest_body(const ForestTaskT<R>& t, int blk, const KParams& kp) {
    extern __shared__ __align__(128) unsigned char fsm[];
    __shared__ __align__(8) uint64_t full[kFW][2];
    __shared__ FLev slv[kFMax];
    const int so = (int)blockIdx.y * t.S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        mbar_init(&full[warp][0], 1);
        mbar_init(&full[warp][1], 1);
        fence_mbar_init();
    }
    if (threadIdx.x < kFMax) slv[threadIdx.x] = t.lv[threadIdx.x];
    __syncthreads();
    pdl_launch_dependents();
    pdl_wait();  // the previous pass's results are visible from here
    trace(1);
    R w = R(0), pf = R(1), nf = R(1);
    if (PASS == FP_TDAVG) w = (R)kp.wsched[(size_t)blockIdx.y * kp.cap + *kp.tdev];
    if (PASS == FP_OBS && kp.post == POST_DCFR) {
        const size_t q = (size_t)blockIdx.y * kp.cap + *kp.tdev;
        pf = (R)kp.pfsched[q];
        nf = (R)kp.nfsched[q];
    }
    const R* xo = PASS == FP_OBS ? t.xo + (size_t)blockIdx.y * t.xo_sx : nullptr;
    const int gw = blk * kFW + warp, nw = t.nblk * kFW;
    unsigned char* stage[2] = {fsm + (size_t)(2 * warp) * t.stage_bytes,
                               fsm + (size_t)(2 * warp + 1) * t.stage_bytes};
    int item = gw;
    if (item < t.nitems) forest_issue<PASS, R>(t, slv, item, stage[0], &full[warp][0], so);
    if (PASS == FP_OBS && t.row0 && blk == 0 && threadIdx.x == 0) {  // the empty sequence's row: u[0]
        FuseUT<R> f0{t.ip, t.ix, t.d, xo, t.neg};
        bool bad = false;
        fused_u<LdL1>(f0, t.uo + so, 0, bad);
        if (bad) atomicOr(kp.nonfinite, 1);
    }
    if (PASS == FP_TDAVG || PASS == FP_TD) {  // the top's x (and average), once, across the task's CTAs
        const R* srcg = t.src + so;
        for (int s = 1 + blk * kFT + (int)threadIdx.x; s < t.Stop; s += t.nblk * kFT) {
            const R xa = top_x(t, srcg, s);
            t.x[so + s] = xa;
            if (PASS == FP_TDAVG) t.avg[so + s] = dadd(dmul(w, xa), t.avg[so + s]);
        }
        if (PASS == FP_TDAVG && blk == 0 && threadIdx.x == 0)  // the reference axpy also covers x[0] = 1
            t.avg[so] = dadd(dmul(w, t.x[so]), t.avg[so]);
    }
    for (int it = 0; item < t.nitems; ++it, item += nw) {
        const int s = it & 1;
        const int next = item + nw;
        if (next < t.nitems) forest_issue<PASS, R>(t, slv, next, stage[s ^ 1], &full[warp][s ^ 1], so);
        trace(2);
        mbar_wait(&full[warp][s], (uint32_t)((it >> 1) & 1));
        trace(3);
        if constexpr (PASS == FP_OBS || PASS == FP_PRED)
            warp_up<PASS, MAXA, R>(t, slv, stage[s], kp, pf, nf, so, xo);
        else
            warp_down<PASS, R>(t, slv, stage[s], w, so);
        trace(4);
        fence_proxy_async();  // this warp's accesses to the stage before the next bulk copy into it
        __syncwarp();
    }
    if constexpr (PASS == FP_OBS || PASS == FP_PRED) {
        // every root V this warp published, then one arrival per root at its
        // parent DP; last arrivals complete the top (top_cascade)
        __threadfence();
        __syncwarp();
        const int j_root = t.lv[0].j_lo;
        for (int q = gw; q < t.nitems; q += nw) {
            int r0, r1;
            item_roots(t, q, r0, r1);
            for (int base = r0; base < r1; base += 32) {
                const int r = base + lane;
                const bool mine = r < r1;
                const int pd = mine ? parent_dp(t, __ldg(t.dp_parent + j_root + r)) : 0;
                top_cascade<PASS, R>(t, kp, pf, nf, pd, mine, so);
            }
        }
        trace(5);
    }
}

template <int PASS, int MAXA, class R>
__global__ void __launch_bounds__(kFT, kFMinB) k_forest(const __grid_constant__ ForestTaskT<R> t0,
                                                        const __grid_constant__ ForestTaskT<R> t1,
                                                        const __grid_constant__ KParams kp) {
    // (a branch per task, so parameter offsets stay compile-time constants)
    if ((int)blockIdx.x < t0.nblk) forest_body<PASS, MAXA, R>(t0, blockIdx.x, kp);
    else forest_body<PASS, MAXA, R>(t1, blockIdx.x - t0.nblk, kp);
}

// ---------------------------------------------------------------------------
// Host: planning.

// Algorithmic bytes of one forest pass (what the kernel moves to and from
// HBM: staged ranges at their exact size, results, payoff gathers; the inner
// V / x stay on chip).  v: bytes per value.
static double forest_bytes(int pass, int nl, const FLev* lv, const FHdr* hd, int v, bool do_rm) {
    double b = 0;
    for (int k = 0; k < nl; ++k) {
        const FHdr& h = hd[k];
        const FLev& L = lv[k];
        const double ns = h.s1 - h.s0, nj = h.j1 - h.j0, nz = h.k1 - h.k0;
        const bool single = L.un == 1;
        if (L.un <= 0) b += 4 * (nj + 1);
        if (pass == FP_OBS || pass == FP_PRED) {
            if (L.cn < 0) b += 8 * ns;
            if (!single) b += 2 * v * ns + v * ns * (pass == FP_OBS ? (do_rm ? 2 : 1) : 1);
            if (L.rows && pass == FP_OBS) b += (4.0 + v) * nz + v * nz + v * ns + (L.rc > 0 ? 0 : 4 * (ns + 1));
            else if (L.rows) b += v * ns;
            if (k == 0) b += v * nj;
        } else {
            if (L.pc <= 0) b += 4 * nj;
            if (!single) b += v * ns;
            b += v * ns * (pass == FP_TDAVG ? 3 : 1);
        }
    }
    return b;
}

// Level pair (k, k+1) is forest-compatible: every DP of level k+1 hangs under
// a sequence of level k, with non-decreasing parent sequences.
static bool pair_ok(const Player& P, const std::vector<int>& par, int k) {
    const int s_lo = P.lvl_s0[k], s_hi = s_lo + (int)P.lvl_ns[k];
    const int j0 = P.lvl[k + 1], j1 = P.lvl[k + 2];
    const int T = host_threads();
    std::vector<char> bad(T, 0);
    parallel_chunks(j1 - j0, 1 << 16, [&](int c, int64_t lo, int64_t hi) {
        for (int64_t q = j0 + lo; q < j0 + hi; ++q) {
            const int p = par[q];
            if (p < s_lo || p >= s_hi || (q > j0 && par[q - 1] > p)) {
                bad[c] = 1;
                return;
            }
        }
    });
    for (char x : bad)
        if (x) return false;
    return true;
}

struct FPlanIn {
    const Player* P;
    const std::vector<int>* sp;
    const std::vector<int>* par;
    const int64_t* indptr;  // the player's payoff rows (U for player 1, Uᵀ for player 2)
    int ls, nl;
};

// Positions (J, S, K per forest level) of the subtree boundary in front of
// level-ls DP a.
static void f_pos(const FPlanIn& in, int a, int* row) {
    const Player& P = *in.P;
    int J = a;
    for (int k = 0; k < in.nl; ++k) {
        const int S = (*in.sp)[J];
        row[3 * k] = J;
        row[3 * k + 1] = S;
        row[3 * k + 2] = (int)in.indptr[S];
        if (k + 1 < in.nl) {
            const int l = in.ls + k + 1;
            const int* b = in.par->data() + P.lvl[l];
            const int* e = in.par->data() + P.lvl[l + 1];
            J = (int)(std::lower_bound(b, e, S) - in.par->data());
        }
    }
}

// Largest stage any pass needs for roots [a, b) (worst-case alignment slack).
static int f_stage_bytes(int nl, const FLev* lv, bool leaf, const std::vector<int>& tab, int a, int b, int v) {
    FHdr hd[kFMax];
    for (int k = 0; k < nl; ++k) {
        const int* ra = &tab[((size_t)a * nl + k) * 3];
        const int* rb = &tab[((size_t)b * nl + k) * 3];
        hd[k].j0 = ra[0];
        hd[k].s0 = ra[1];
        hd[k].k0 = ra[2];
        hd[k].j1 = rb[0];
        hd[k].s1 = rb[1];
        hd[k].k1 = rb[2];
    }
    int mx = 0;
    for (int pass = 0; pass < FP_COUNT; ++pass)
        for (int so : {0, 1, 2, 3}) {
            FItem it{a, b, 0, 0, 0};
            mx = std::max(mx, forest_layout(pass, nl, nl, lv, leaf, it, hd, v, so));
        }
    return mx;
}

static FLev level_of(const Player& P, const DevCsr& M, const int64_t* indptr, bool affine_rows, int l) {
    const DevTree& sh = P.lvl_shape[l];
    FLev f{};
    f.j_lo = sh.j_lo;
    f.s_lo = sh.s_lo;
    f.un = sh.un;
    f.cn = sh.cn;
    f.c_lo = sh.c_lo;
    f.pc = sh.pc;
    f.p_lo = sh.p_lo;
    const int s0 = l == 0 ? 0 : sh.s_lo, s1 = sh.s_lo + (int)P.lvl_ns[l];
    f.rows = indptr[s1] - indptr[s0] > 0 ? 1 : 0;
    f.rc = affine_rows && l < (int)M.lvl_rowc.size() ? std::max(0, M.lvl_rowc[l]) : 0;
    f.rs0 = sh.s_lo;
    f.rk0 = (int)indptr[sh.s_lo];
    return f;
}

// Plans one player: the split level, the levels' shapes, the root table and
// the items.  Returns false when the tree has no forest-compatible split.
static bool plan_forest_player(scfr_handle* h, int k, const int64_t* indptr, const DevCsr& M, ForestPlayer& fp) {
    const Player& P = h->P[k];
    const int L = P.levels();
    if (L < 2 || !P.h_seq_ptr || !P.h_dp_parent) return false;
    const std::vector<int>& sp = *P.h_seq_ptr;
    const std::vector<int>& par = *P.h_dp_parent;
    const int v = h->f32 ? 4 : 8;
    int deepest_bad = -1;  // largest q with pair (q, q+1) incompatible
    for (int q = L - 2; q >= 0; --q)
        if (!pair_ok(P, par, q)) {
            deepest_bad = q;
            break;
        }
    int budget = 6 * 1024;
    if (const char* e = std::getenv("SCFR_FOREST_STAGE")) budget = std::max(2048, std::atoi(e));
    const int min_roots = 4 * h->num_sms;
    for (int ls = std::max(1, deepest_bad + 1); ls < L; ++ls) {
        const int nl = L - ls;
        if (ls > kTopMax || nl > kFMax) continue;
        const int Jtop = P.lvl[ls];
        if (Jtop > kTopMaxDPs || sp[Jtop] > (1 << 22)) break;  // the top is for few DPs
        const int a0 = P.lvl[ls], a1 = P.lvl[ls + 1], nroots = a1 - a0;
        if (nroots < min_roots && ls + 1 < L) continue;  // too little parallelism: split deeper
        FPlanIn in{&P, &sp, &par, indptr, ls, nl};
        FLev lv[kFMax];
        for (int q = 0; q < nl; ++q) {
            lv[q] = level_of(P, M, indptr, h->affine_rows, ls + q);
            if (q + 1 == nl) lv[q].cn = 0;  // the deepest level has no child DPs
        }
        const bool leaf = nl >= 2 && lv[nl - 1].un == 1;  // the deepest level: forced moves into end nodes
        std::vector<int> tab((size_t)(nroots + 1) * nl * 3);
        parallel_chunks(nroots + 1, 1 << 12, [&](int, int64_t lo, int64_t hi) {
            for (int64_t r = lo; r < hi; ++r) f_pos(in, a0 + (int)r, &tab[(size_t)r * nl * 3]);
        });
        // items (one warp each): consecutive roots within the budget; fewer,
        // bigger items than the warps can keep busy would starve them, so
        // aim for >= 48 per SM
        const double total = (double)f_stage_bytes(nl, lv, leaf, tab, 0, nroots, v);
        const int eff = (int)std::max(1024.0, std::min((double)budget, total / (48.0 * h->num_sms)));
        // affine forest: every level's positions linear in the root index
        bool aff = nroots >= 2;
        for (int q = 0; q < nl && aff; ++q)
            aff = lv[q].un > 0 && lv[q].cn >= 0 && lv[q].pc > 0 && (!lv[q].rows || lv[q].rc > 0);
        for (int r = 2; r <= nroots && aff; ++r)
            for (int c = 0; c < nl * 3 && aff; ++c)
                aff = tab[(size_t)r * nl * 3 + c] == tab[c] + r * (tab[nl * 3 + c] - tab[c]);
        std::vector<int> items{0};
        bool fits = true;
        if (aff) {  // uniform items of aR roots
            int R = 1;
            while (R < nroots && f_stage_bytes(nl, lv, leaf, tab, 0, R + 1, v) <= eff) ++R;
            fits = f_stage_bytes(nl, lv, leaf, tab, 0, 1, v) <= budget;
            for (int a = R; a < nroots; a += R) items.push_back(a);
            items.push_back(nroots);
            fp.aR = R;
        }
        for (int a = 0; a < nroots && !aff;) {
            if (f_stage_bytes(nl, lv, leaf, tab, a, a + 1, v) > budget) {
                fits = false;
                break;
            }
            int lo = a + 1, hi = nroots;  // largest b with the stage within eff
            while (lo < hi) {
                const int mid = lo + (hi - lo + 1) / 2;
                if (f_stage_bytes(nl, lv, leaf, tab, a, mid, v) <= eff) lo = mid;
                else hi = mid - 1;
            }
            a = lo;
            items.push_back(a);
        }
        if (!fits) continue;
        fp.ls = ls;
        fp.nl = nl;
        fp.leaf = leaf;
        fp.nroots = nroots;
        fp.nitems = (int)items.size() - 1;
        fp.Jtop = Jtop;
        fp.Stop = sp[Jtop];
        for (int q = 0; q < nl; ++q) fp.lv[q] = lv[q];
        for (int q = 0; q < ls; ++q) fp.tlv[q] = level_of(P, M, indptr, h->affine_rows, q);
        fp.aff = aff;
        fp.stage = 0;
        if (aff) {
            fp.stage = f_stage_bytes(nl, lv, leaf, tab, 0, fp.aR, v);  // (per-solve residues cover every item)
            for (int q = 0; q < nl; ++q) {
                FLev& f = fp.lv[q];
                f.aj0 = tab[q * 3];
                f.as0 = tab[q * 3 + 1];
                f.ak0 = tab[q * 3 + 2];
                f.dj = tab[nl * 3 + q * 3] - f.aj0;
                f.ds = tab[nl * 3 + q * 3 + 1] - f.as0;
                f.dk = tab[nl * 3 + q * 3 + 2] - f.ak0;
            }
        } else {
            for (int c = 0; c < fp.nitems; ++c)
                fp.stage = std::max(fp.stage, f_stage_bytes(nl, lv, leaf, tab, items[c], items[c + 1], v));
        }
        for (int q = 0; q < nl; ++q) {
            fp.all[q].j0 = tab[q * 3];
            fp.all[q].s0 = tab[q * 3 + 1];
            fp.all[q].k0 = tab[q * 3 + 2];
            fp.all[q].j1 = tab[((size_t)nroots * nl + q) * 3];
            fp.all[q].s1 = tab[((size_t)nroots * nl + q) * 3 + 1];
            fp.all[q].k1 = tab[((size_t)nroots * nl + q) * 3 + 2];
        }
        fp.maxa = 1;
        for (int q = ls; q < L; ++q) fp.maxa = std::max(fp.maxa, P.lvl_maxa[q]);
        // the top: sequence -> DP, ancestor chains, child-DP counts
        const int Stop = fp.Stop;
        fp.h_sdp.assign(std::max(Stop, 1), -1);
        for (int q = 0; q < Jtop; ++q)
            for (int s = sp[q]; s < sp[q + 1]; ++s) fp.h_sdp[s] = q;
        std::vector<int> lvl_of(Jtop, 0);
        for (int l = 0; l < ls; ++l)
            for (int q = P.lvl[l]; q < P.lvl[l + 1]; ++q) lvl_of[q] = l;
        fp.h_anc.assign((size_t)std::max(Stop, 1) * ls, -1);
        for (int s = 1; s < Stop; ++s) {
            int chain[kTopMax + 1], n = 0;
            for (int a = s; a != 0 && n <= kTopMax; a = par[fp.h_sdp[a]]) chain[n++] = a;
            if (n > ls) return false;  // deeper than the top's levels: not a DP-level tree
            for (int i = 0; i < n; ++i) {
                const int a = chain[n - 1 - i];
                const bool single = P.lvl_shape[lvl_of[fp.h_sdp[a]]].un == 1;
                fp.h_anc[(size_t)s * ls + i] = a | (single ? 1 << 30 : 0);
            }
        }
        fp.h_nch.assign(Jtop + 1, 0);
        for (int q = 0; q < P.J; ++q) {
            const int p = par[q];
            if (p == 0) fp.h_nch[Jtop]++;
            else if (p < Stop) fp.h_nch[fp.h_sdp[p]]++;
        }
        fp.h_tab.swap(tab);
        fp.h_items.swap(items);
        return true;
    }
    return false;
}

bool prepare_forest(scfr_handle* h, const scfr_csr* U, const scfr_csr* UT) {
    const char* off = std::getenv("SCFR_NO_FOREST");
    if (off && off[0] == '1') return false;
    if (h->comm || h->engine != SCFR_ENGINE_LEVELS || !h->fuse || !h->u_empty_skip || h->P[0].J == 0 ||
        h->P[1].J == 0)
        return false;
    // predictive alt mode: CUR is a TD over bcur (OBS₁ regret-matches into it)
    if (predictive(h->variant) && h->mode == SCFR_MODE_ALT && !h->bcur_on) return false;
    ForestPlayer fp[2];
    for (int k = 0; k < 2; ++k)
        if (!plan_forest_player(h, k, (k == 0 ? U : UT)->indptr, k == 0 ? h->U : h->UT, fp[k])) return false;
    const int v = h->f32 ? 4 : 8;
    for (int k = 0; k < 2; ++k) {
        ForestPlayer& d = h->fp[k];  // (DevBuf is not movable: fill in place)
        ForestPlayer& s = fp[k];
        d.ls = s.ls;
        d.nl = s.nl;
        d.leaf = s.leaf;
        d.aff = s.aff;
        d.aR = s.aR;
        // top-down passes skip a forced leaf level whose x / avg are parent
        // copies (solver.cu leaf_x)
        d.nl_down = s.nl - (h->leaf_x && leaf_single(h, h->P[k]) ? 1 : 0);
        d.nroots = s.nroots;
        d.nitems = s.nitems;
        d.stage = s.stage;
        d.maxa = s.maxa;
        d.Jtop = s.Jtop;
        d.Stop = s.Stop;
        std::copy(s.lv, s.lv + kFMax, d.lv);
        std::copy(s.tlv, s.tlv + kTopMax, d.tlv);
        std::copy(s.all, s.all + kFMax, d.all);
        for (int p = 0; p < FP_COUNT; ++p)
            d.bytes[p] = forest_bytes(p, p >= FP_TDAVG ? d.nl_down : d.nl, d.lv, d.all, v, p == FP_OBS);
        d.bytes_obs_norm = forest_bytes(FP_OBS, d.nl, d.lv, d.all, v, false);
        auto up = [&](DevBuf<int>& dst, const std::vector<int>& src) {
            dst.alloc(std::max<size_t>(src.size(), 1));
            if (!src.empty())
                CUDA_OK(copy_async(dst.p, src.data(), src.size() * sizeof(int), cudaMemcpyHostToDevice, h->stream));
        };
        up(d.tab, s.h_tab);
        up(d.items, s.h_items);
        up(d.top_sdp, s.h_sdp);
        up(d.top_anc, s.h_anc);
        up(d.nch, s.h_nch);
        d.cnt.alloc((size_t)(d.Jtop + 1) * h->B);
        d.cnt.zero(h->stream);
    }
    CUDA_OK(cudaStreamSynchronize(h->stream));  // the host vectors die here
    h->forest = true;
    return true;
}

// ---------------------------------------------------------------------------
// Host: per-iteration launches.

template <int PASS, class R>
static void (*pick_forest(int maxa))(ForestTaskT<R>, ForestTaskT<R>, KParams) {
    if (maxa <= 2) return k_forest<PASS, 2, R>;
    if (maxa <= 4) return k_forest<PASS, 4, R>;
    return k_forest<PASS, 8, R>;
}

template <class R>
struct ForestLauncher {
    LaunchBase& L;
    scfr_handle* h;

    ForestTaskT<R> task(int k, int pass) {
        ForestPlayer& fp = h->fp[k];
        Player& P = h->P[k];
        const DevCsr& M = k == 0 ? h->U : h->UT;
        ForestTaskT<R> t{};
        t.nl = pass >= FP_TDAVG ? fp.nl_down : fp.nl;
        t.leaf = pass >= FP_TDAVG ? 0 : fp.leaf;
        t.nla = fp.nl;
        t.nitems = fp.nitems;
        t.nroots = fp.nroots;
        t.aff = fp.aff ? 1 : 0;
        t.aR = fp.aR;
        t.items = fp.items.p;
        t.tab = fp.tab.p;
        std::copy(fp.lv, fp.lv + kFMax, t.lv);
        t.ls = fp.ls;
        t.Jtop = fp.Jtop;
        t.Stop = fp.Stop;
        t.row0 = fp.tlv[0].rows;
        for (int l = 0; l <= fp.ls; ++l) t.tlo[l] = P.lvl[l];
        std::copy(fp.tlv, fp.tlv + kTopMax, t.tlv);
        t.top_sdp = fp.top_sdp.p;
        t.top_anc = fp.top_anc.p;
        t.nch = fp.nch.p;
        t.cnt = fp.cnt.p;
        t.done = h->fdone.p;
        t.S = P.S;
        t.J = P.J;
        t.seq_ptr = P.seq_ptr.p;
        t.dp_parent = P.dp_parent.p;
        t.child = P.child.p;
        t.ip = M.indptr.p;
        t.ix = M.iter_indices();
        if constexpr (sizeof(R) == 4) t.d = M.data32.p;
        else t.d = M.data.p;
        t.neg = k;
        t.r = vals<R>(P.r);
        t.b = vals<R>(P.b);
        t.bo = t.b;
        t.u = vals<R>(P.u);
        t.uo = vals<R>(P.u);
        t.x = vals<R>(P.x);
        t.avg = vals<R>(P.avg);
        t.V = vals<R>(P.V);
        t.src = t.b;
        return t;
    }

    template <class K>
    int resident(K kern, size_t smem) {
        const void* key = reinterpret_cast<const void*>(kern);
        for (const auto& e : h->tile_occ)
            if (e.first == key) return e.second * h->num_sms;
        int occ = 0;
        CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kFT, smem));
        if (occ < 1) fail(SCFR_ECUDA, "forest kernel cannot be resident (%zu B shared memory)", smem);
        h->tile_occ.emplace_back(key, occ);
        return occ * h->num_sms;
    }

    // One forest pass over player tasks a (and b, when both players run).
    template <int PASS>
    void pass(int kk, ForestTaskT<R> a, ForestTaskT<R>* b, bool do_rm, bool tick, double bytes) {
        ForestTaskT<R> t1 = b ? *b : ForestTaskT<R>{};
        if (!b) t1.nitems = 0;
        a.do_rm = t1.do_rm = do_rm ? 1 : 0;
        const int st = std::max(h->fp[0].stage, h->fp[1].stage);
        a.stage_bytes = t1.stage_bytes = st;
        const int ntask = b ? 2 : 1;
        a.tick = t1.tick = tick ? h->tdev.p : nullptr;
        a.ntick = t1.ntick = ntask * h->B;
        const int maxa = std::max(h->fp[0].maxa, h->fp[1].maxa);
        auto kern = pick_forest<PASS, R>(maxa);
        const size_t smem = 2 * kFW * (size_t)st;
        const int wave = std::max(2, resident(kern, smem) / h->B);  // per solve (blockIdx.y)
        // CTAs in proportion to each task's items, one resident wave in all
        const int tot = a.nitems + t1.nitems;
        a.nblk = std::max(1, std::min(a.nitems, (int)((int64_t)wave * a.nitems / std::max(1, tot))));
        t1.nblk = t1.nitems > 0 ? std::max(1, std::min(t1.nitems, wave - a.nblk)) : 0;
        const KParams kp = L.kparams(do_rm);
        L.launch(kk, bytes, [&] { L.run_ex(kern, dim3(a.nblk + t1.nblk, h->B), kFT, smem, a, t1, kp); });
    }

    // Bytes of the top levels of one pass (kernels.cuh per-DP terms).
    double top_bytes(int k, bool up) {
        const Player& P = h->P[k];
        const double v = sizeof(R);
        double b = 0;
        for (int l = 0; l < h->fp[k].ls; ++l) {
            const double ns = P.lvl_ns[l], nj = P.lvl_nj[l], nc = P.lvl_nc[l];
            b += up ? 4 * v * ns + v * nj + v * nc : 3 * v * ns;
        }
        return b;
    }

    void iteration() {
        Player& A = h->P[0];
        Player& Bp = h->P[1];
        const bool pr = predictive(h->variant);
        const bool alt = h->mode == SCFR_MODE_ALT;
        const ForestPlayer& fa = h->fp[0];
        const ForestPlayer& fb = h->fp[1];
        // next_strategy of both players: [PRED], then TD + average
        if (pr) {
            ForestTaskT<R> a = task(0, FP_PRED), b = task(1, FP_PRED);
            pass<FP_PRED>(KK_PRED, a, &b, false, false,
                          fa.bytes[FP_PRED] + fb.bytes[FP_PRED] + top_bytes(0, true) + top_bytes(1, true));
        }
        {
            ForestTaskT<R> a = task(0, FP_TDAVG), b = task(1, FP_TDAVG);
            pass<FP_TDAVG>(KK_TD_AVG, a, &b, false, false,
                           fa.bytes[FP_TDAVG] + fb.bytes[FP_TDAVG] + 2 * (top_bytes(0, false) + top_bytes(1, false)));
        }
        // observe: payoff rows fused (u1 = U x2, u2 = -Uᵀ x1 / x1')
        const int kobs = pr ? KK_OBS : KK_OBS_RM;
        auto obs = [&](int k) {
            ForestTaskT<R> t = task(k, FP_OBS);
            t.xo = k == 0 ? vals<R>(Bp.x) : (alt ? vals<R>(A.xpost) : vals<R>(A.x));
            t.xo_sx = k == 0 ? Bp.S : A.S;
            return t;
        };
        const double ob_a = (pr && !alt ? fa.bytes_obs_norm : fa.bytes[FP_OBS]) + top_bytes(0, true);
        const double ob_b = (pr ? fb.bytes_obs_norm : fb.bytes[FP_OBS]) + top_bytes(1, true);
        if (!alt) {
            ForestTaskT<R> a = obs(0), b = obs(1);
            pass<FP_OBS>(kobs, a, &b, !pr, true, ob_a + ob_b);
            return;
        }
        {
            // OBS₁ regret-matches into b (non-predictive) or into bcur, which
            // current_strategy then multiplies down into xpost
            ForestTaskT<R> a = obs(0);
            if (pr) a.bo = vals<R>(A.bcur);
            pass<FP_OBS>(kobs, a, nullptr, true, false, ob_a);
            ForestTaskT<R> c = task(0, FP_TD);
            c.x = vals<R>(A.xpost);
            c.src = pr ? vals<R>(A.bcur) : vals<R>(A.b);
            pass<FP_TD>(pr ? KK_CUR : KK_TD, c, nullptr, false, false, fa.bytes[FP_TD] + top_bytes(0, false));
        }
        {
            ForestTaskT<R> b = obs(1);
            pass<FP_OBS>(kobs, b, nullptr, !pr, true, ob_b);
        }
    }
};

static DevBuf<long long> g_trace_buf;

template <class R>
void forest_iteration(LaunchBase& L) {
    ForestLauncher<R> F{L, L.h};
    F.iteration();
}
template void forest_iteration<double>(LaunchBase&);
template void forest_iteration<float>(LaunchBase&);

}  // namespace scfr

// Phase trace of the forest kernels (tuning aid): CTA 0 of every launch
// appends (clock64 << 8 | tag) values.  scfr_trace_start(cap) arms a buffer
// of cap entries (0 disarms); scfr_trace_read copies them out.
int scfr_trace_start(int cap) {
    return scfr::guarded([&] {
        using namespace scfr;
        long long* p = nullptr;
        if (cap > 0) {
            g_trace_buf.alloc((size_t)cap);
            p = g_trace_buf.p;
        } else {
            g_trace_buf.free();
            cap = 0;
        }
        const int zero = 0;
        CUDA_OK(cudaMemcpyToSymbol(g_trace, &p, sizeof p));
        CUDA_OK(cudaMemcpyToSymbol(g_trace_cap, &cap, sizeof cap));
        CUDA_OK(cudaMemcpyToSymbol(g_trace_n, &zero, sizeof zero));
    });
}

int scfr_trace_read(int64_t* out, int cap, int* n) {
    return scfr::guarded([&] {
        using namespace scfr;
        if (!out || !n) fail(SCFR_EINVAL, "NULL argument");
        CUDA_OK(cudaDeviceSynchronize());
        int m = 0;
        CUDA_OK(cudaMemcpyFromSymbol(&m, g_trace_n, sizeof m));
        m = std::min(m, std::min(cap, (int)g_trace_buf.n));
        if (m > 0) CUDA_OK(cudaMemcpy(out, g_trace_buf.p, (size_t)m * sizeof(long long), cudaMemcpyDeviceToHost));
        *n = m;
    });
}
