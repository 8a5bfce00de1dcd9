// sm_100a device functions for one CFR iteration, per decision point (DP).
//
// Bit-faithful fp64: every operation is an explicit round-to-nearest
// intrinsic in the exact association order of the reference (SURVEY.md
// §8(a) "exact arithmetic contract"); the translation units are also
// compiled with -fmad=false so nothing is contracted into an FMA.  Sums are
// sequential per output element and exactly one thread owns each output, so
// results are deterministic and equal to the numba loops bit for bit.
//
// Layout (per player, per solve; solves of a batch are strided copies):
//   seq-indexed fp64 vectors over Σ (slot 0 = empty sequence): r, b, x,
//     xpost, avg, u, g   — r/b slot 0 unused (reference Σ+ index = s-1)
//   dp-indexed fp64 temporaries over J: V (sum pass), W (max pass)
//   structure (int32, read-only): seq_ptr[J+1] (action range of DP j),
//     dp_parent[J] (parent sequence), child[S] = {lo, cnt} (child-DP range of
//     sequence s: cnt 0 = end node, 1 = a single DP, >1 = observation point)
//   DP levels: DPs grouped by process-tree depth; BFS numbering makes each
//     level a contiguous j range (pkg/decision_process.py:9-13).
//
// Loads go through the policy `Ld`: structure via the read-only path
// (__ldg) and mutable state with plain (L1-cacheable) loads where every
// producer ran in an earlier launch or in the same CTA (LdL1: level engine,
// CTA-persistent engine); L2-only loads (ld.global.cg) in the grid-persistent
// engine whose producers are other SMs in the same launch (LdL2); plain loads
// of everything when state and structure live in shared memory (LdS).
#pragma once

#include <cstdint>

namespace scfr {

struct DevTree {
    const int* __restrict__ seq_ptr;    // [J+1]
    const int* __restrict__ dp_parent;  // [J]
    const int2* __restrict__ child;     // [S]
    // Optional affine shape of the level being processed, set by the host
    // when it holds exactly (then the index is computed, not loaded):
    //   un > 0:  DP j has un actions, s0 = s_lo + (j - j_lo) * un
    //   cn >= 0: sequence s has cn child DPs starting at c_lo + (s - s_lo) * cn
    //   pc > 0:  DP j's parent sequence is p_lo + (j - j_lo) / pc
    int j_lo = 0, s_lo = 0, un = 0, cn = -1, c_lo = 0, pc = 0, p_lo = 0;
};

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
// fp32 mode: the same operation sequence, every operation rounded to fp32
// (no FMA contraction either way; the fp32 oracle restates it op for op).
__device__ __forceinline__ float dadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float dmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float ddiv(float a, float b) { return __fdiv_rn(a, b); }

// kChunk: child loads a lane keeps in flight in the warp-per-DP variants
// (deep for HBM/L2 latency, shallow for shared memory).
struct LdL1 {
    static constexpr int kChunk = 32;
    template <class V>
    static __device__ __forceinline__ V ld(const V* p) { return *p; }
    template <class X>
    static __device__ __forceinline__ X st(const X* p) { return __ldg(p); }
};
struct LdL2 {
    static constexpr int kChunk = 32;
    template <class V>
    static __device__ __forceinline__ V ld(const V* p) { return __ldcg(p); }
    template <class X>
    static __device__ __forceinline__ X st(const X* p) { return __ldg(p); }
};
// L1 loads with a shallow chunk (group mode: 6 CTAs per SM at 80 registers).
struct LdL1s : LdL1 {
    static constexpr int kChunk = 8;
};
// L2-only loads with a shallow chunk: the tile engine's top pass, which
// shares a kernel (and so a register budget) with the tile walk.
struct LdL2s {
    static constexpr int kChunk = 8;
    template <class V>
    static __device__ __forceinline__ V ld(const V* p) { return __ldcg(p); }
    template <class X>
    static __device__ __forceinline__ X st(const X* p) { return __ldg(p); }
};
// Shared-memory resident state and structure (CTA-resident small-game engine).
struct LdS {
    static constexpr int kChunk = 8;
    template <class V>
    static __device__ __forceinline__ V ld(const V* p) { return *p; }
    template <class X>
    static __device__ __forceinline__ X st(const X* p) { return *p; }
};

enum : int { POST_NONE = 0, POST_PLUS = 1, POST_DCFR = 2 };

// Non-deduced context: scalars and optional pointers take the state's type.
template <class T>
struct nd {
    using type = T;
};

template <class Ld>
__device__ __forceinline__ void dp_range(const DevTree& T, int j, int& s0, int& n) {
    if (T.un > 0) {
        s0 = T.s_lo + (j - T.j_lo) * T.un;
        n = T.un;
    } else {
        s0 = Ld::st(T.seq_ptr + j);
        n = Ld::st(T.seq_ptr + j + 1) - s0;
    }
}
template <class Ld>
__device__ __forceinline__ int2 child_of(const DevTree& T, int s) {
    if (T.cn >= 0) return make_int2(T.c_lo + (s - T.s_lo) * T.cn, T.cn);
    return Ld::st(T.child + s);
}
template <class Ld>
__device__ __forceinline__ int parent_of(const DevTree& T, int j) {
    if (T.pc > 0) return T.p_lo + (j - T.j_lo) / T.pc;
    return Ld::st(T.dp_parent + j);
}

// Value flowing up into a sequence from the DPs below it, given its child
// range c and (already loaded) V of its first child `v0`:
//   end node: 0.0 (the zero-initialised v); one DP: V of that DP;
//   observation point: ((0.0 + V_lo) + V_lo+1) + ... in j order
// (pkg/solvers.py:195-199, pkg/oracle.py:91-95).
template <class Ld, class R>
__device__ __forceinline__ R child_value(int2 c, R v0, const R* __restrict__ V) {
    if (c.y == 0) return R(0);
    if (c.y == 1) return v0;
    R acc = dadd(R(0), v0);
    int k = 1;
    for (; k + 4 <= c.y; k += 4) {  // loads first, adds in order
        const R a0 = Ld::ld(V + c.x + k), a1 = Ld::ld(V + c.x + k + 1);
        const R a2 = Ld::ld(V + c.x + k + 2), a3 = Ld::ld(V + c.x + k + 3);
        acc = dadd(dadd(dadd(dadd(acc, a0), a1), a2), a3);
    }
    for (; k < c.y; ++k) acc = dadd(acc, Ld::ld(V + c.x + k));
    return acc;
}

template <class Ld, class R>
__device__ __forceinline__ R child_sum(int2 c, const R* __restrict__ V) {
    return child_value<Ld>(c, c.y > 0 ? Ld::ld(V + c.x) : R(0), V);
}

// Utility / prediction of sequence s.  u == nullptr: the level's payoff rows
// are structurally empty, so u is the constant ±0.0 (+0.0 player 1, -0.0 =
// -1.0*0.0 player 2) and every use adds it to 0.0 first: +0.0 either way.
template <class Ld, class R>
__device__ __forceinline__ R ld_u(const R* u, int s) {
    return u ? Ld::ld(u + s) : R(0);
}

// Entries [k0, k1) of a CSR row: ((0.0 + d0*x0) + d1*x1) + ... in order.
template <class Ld, class R>
__device__ __forceinline__ R spmv_range(const int* __restrict__ indices, const R* __restrict__ data,
                                        const R* __restrict__ x, int k0, int k1) {
    R acc = R(0);
    int k = k0;
    for (; k + 2 <= k1; k += 2) {
        const R d0 = __ldg(data + k), d1 = __ldg(data + k + 1);
        const R x0 = Ld::ld(x + __ldg(indices + k)), x1 = Ld::ld(x + __ldg(indices + k + 1));
        acc = dadd(dadd(acc, dmul(d0, x0)), dmul(d1, x1));
    }
    if (k < k1) acc = dadd(acc, dmul(__ldg(data + k), Ld::ld(x + __ldg(indices + k))));
    return acc;
}

// Payoff SpMV row: ((0.0 + d0*x[c0]) + d1*x[c1]) + ... (pkg/kernels.py:149-154).
template <class Ld, class R>
__device__ __forceinline__ R spmv_row(const int* __restrict__ indptr,
                                           const int* __restrict__ indices,
                                           const R* __restrict__ data,
                                           const R* __restrict__ x, int row) {
    return spmv_range<Ld>(indices, data, x, __ldg(indptr + row), __ldg(indptr + row + 1));
}

// Optional fusion of the payoff SpMV into the observe pass: when `ip` is set
// the utility of sequence s is computed here as row s of M applied to the
// opponent's strategy x (scaled by -1 for player 2, pkg/solvers.py:359,368),
// stored to u[s] (it is the next iteration's prediction), and used directly.
template <class R>
struct FuseUT {
    const int* ip;
    const int* ix;
    const R* d;
    const R* x;
    int neg;
    // rc > 0: every row of this launch's level holds rc non-zeros, so row s
    // starts at rk0 + (s - rs0) * rc and indptr is not loaded (Goofspiel's
    // terminal rows: one each).  Same k range, same sum order.
    int rc = 0, rs0 = 0, rk0 = 0;
};
using FuseU = FuseUT<double>;

template <class Ld, class R>
__device__ __forceinline__ R fused_u(const FuseUT<R>& f, R* u, int s, bool& bad) {
    R v;
    if (f.rc > 0) {
        const int k0 = f.rk0 + (s - f.rs0) * f.rc;
        v = spmv_range<Ld>(f.ix, f.d, f.x, k0, k0 + f.rc);
    } else {
        v = spmv_row<Ld>(f.ip, f.ix, f.d, f.x, s);
    }
    if (f.neg) v = dmul(R(-1), v);
    bad |= !isfinite(v);
    u[s] = v;
    return v;
}

// q[a] = (0.0 + u[s0+a]) + C_{s0+a} for a < n <= MAXA, all loads issued
// before the dependent adds ((w + v)[node(s)] read back through Bᵀ,
// pkg/solvers.py:192-202).
template <int MAXA, class Ld, class R>
__device__ __forceinline__ void load_q(const DevTree& T, const R* __restrict__ u,
                                       const R* __restrict__ V, int s0, int n,
                                       R (&q)[MAXA], const FuseUT<R> f = FuseUT<R>{},
                                       bool* bad = nullptr) {
    int2 c[MAXA];
    R uu[MAXA], v0[MAXA];
#pragma unroll
    for (int a = 0; a < MAXA; ++a)
        if (a < n) {
            c[a] = child_of<Ld>(T, s0 + a);
            uu[a] = f.ip ? fused_u<Ld>(f, const_cast<R*>(u), s0 + a, *bad) : ld_u<Ld>(u, s0 + a);
        }
#pragma unroll
    for (int a = 0; a < MAXA; ++a)
        if (a < n) v0[a] = c[a].y > 0 ? Ld::ld(V + c[a].x) : R(0);
#pragma unroll
    for (int a = 0; a < MAXA; ++a)
        if (a < n) q[a] = dadd(dadd(R(0), uu[a]), child_value<Ld>(c[a], v0[a], V));
}

template <class Ld, class R>
__device__ __forceinline__ R qval(const DevTree& T, const R* __restrict__ u,
                                       const R* __restrict__ V, int s) {
    return dadd(dadd(R(0), ld_u<Ld>(u, s)), child_sum<Ld>(child_of<Ld>(T, s), V));
}

template <class R>
__device__ __forceinline__ R post_op(R rv, int post, R pf, R nf) {
    if (post == POST_PLUS) return rv > R(0) ? rv : R(0);
    if (post == POST_DCFR) return rv > R(0) ? dmul(rv, pf) : (rv < R(0) ? dmul(rv, nf) : rv);
    return rv;
}

// Regret matching of one block (pkg/solvers.py:156-160): positive part,
// sequential sum from 0.0, IEEE division, uniform 1.0/n fallback.
template <class R>
__device__ __forceinline__ R rm_prob(R rv, R S, int n) {
    const R p = rv > R(0) ? rv : R(0);
    const bool z = S == R(0);  // one division either way: p / S, or 1.0 / n
    return ddiv(z ? R(1) : p, z ? R(n) : S);
}


// single_action_note — a DP with exactly one action (a forced move) keeps
// b = 1.0 and r = +0.0 for ever, in every variant, bit for bit:
//   RM: S = 0.0 + max(r, 0) = 0.0 -> b = 1.0/1 = 1.0 (and r/r = 1.0 if r > 0);
//   E = 0.0 + 1.0*q;  r' = r + ((-1.0*(0.0+E)) + q) = r + (+0.0) = r
//   (r starts at +0.0; the floor and the DCFR scale map +0.0 to +0.0).
// When the host marks a whole level single-action (DevTree::un == 1) the
// passes therefore skip the r/b traffic and only produce V (and u, x, avg).
// A non-finite q still raises the FloatingPointError flag; the run aborts
// there exactly as the reference would.

// leaf_note — a level of single-action DPs whose sequences end the tree
// (no child DPs) gives, in the PRED pass, V_j = 0.0 + 1.0*((0.0 + m_s) + 0.0)
// = m_s with -0.0 turned into +0.0.  A parent reads child values either as
// the lone child (added to 0.0 + u, which is never -0.0) or through a sum
// that starts from 0.0, so +0.0 and -0.0 give the same bits: the parent can
// read m_s directly and that PRED level need not run.

// ---------------------------------------------------------------------------
// OBS: counterfactual values + regret update (+ variant post-op) (+ regret
// matching of the updated regrets into b for the next iteration).
// pkg/solvers.py:178-224 and :143-160, fused per decision point.
// MAXA: actions held in registers; wider DPs take the generic (recompute) path.
template <int MAXA, class Ld, class R>
__device__ __forceinline__ void obs_dp(const DevTree& T, int j, const R* __restrict__ u,
                                       R* __restrict__ r, R* __restrict__ b,
                                       R* __restrict__ V, int post, typename nd<R>::type pf, typename nd<R>::type nf,
                                       bool do_rm, int* nonfinite, FuseUT<R> fuse = FuseUT<R>{},
                                       const R* Vc = nullptr, bool skip_v = false, R* bw = nullptr) {
    // bw: where regret matching writes (default b; CUR's matched strategy in
    // the predictive alt mode, solver.cu bcur)
    R* const bo = bw ? bw : b;
    // Vc: where child values are read (default V; the level engine points it
    // at u when the child level is a forced leaf level, kernels.cuh
    // leaf_note).  skip_v: that leaf level itself, whose V nobody reads.
    const R* Vr = Vc ? Vc : V;
    int s0, n;
    dp_range<Ld>(T, j, s0, n);
    bool bad = false;
    if (T.un == 1) {  // single-action level: r and b are constants (see single_action_note)
        const R uu = fuse.ip ? fused_u<Ld>(fuse, const_cast<R*>(u), s0, bad) : ld_u<Ld>(u, s0);
        const R q = dadd(dadd(R(0), uu), child_sum<Ld>(child_of<Ld>(T, s0), Vr));
        if (!skip_v) V[j] = dadd(R(0), dmul(R(1), q));
        bad |= !isfinite(q);
        if (bad) atomicOr(nonfinite, 1);
        return;
    }
    if (n <= MAXA) {
        R q[MAXA], bb[MAXA], rr[MAXA];
        load_q<MAXA, Ld>(T, u, Vr, s0, n, q, fuse, &bad);
#pragma unroll
        for (int a = 0; a < MAXA; ++a)
            if (a < n) {
                bb[a] = Ld::ld(b + s0 + a);
                rr[a] = Ld::ld(r + s0 + a);
            }
        R E = R(0);
#pragma unroll
        for (int a = 0; a < MAXA; ++a)
            if (a < n) E = dadd(E, dmul(bb[a], q[a]));
        V[j] = E;
        const R negE = dmul(R(-1), dadd(R(0), E));
        R S = R(0);
#pragma unroll
        for (int a = 0; a < MAXA; ++a)
            if (a < n) {
                bad |= !isfinite(q[a]);
                const R rv = post_op(dadd(rr[a], dadd(negE, q[a])), post, pf, nf);
                bad |= !isfinite(rv);
                rr[a] = rv;
                r[s0 + a] = rv;
                S = dadd(S, rv > R(0) ? rv : R(0));
            }
        if (do_rm) {
#pragma unroll
            for (int a = 0; a < MAXA; ++a)
                if (a < n) bo[s0 + a] = rm_prob(rr[a], S, n);
        }
    } else {
        if (fuse.ip)  // wide DP: materialise u first, then the generic path re-reads it
            for (int s = s0; s < s0 + n; ++s) fused_u<Ld>(fuse, const_cast<R*>(u), s, bad);
        R E = R(0);
        for (int s = s0; s < s0 + n; ++s) E = dadd(E, dmul(Ld::ld(b + s), qval<Ld>(T, u, Vr, s)));
        V[j] = E;
        const R negE = dmul(R(-1), dadd(R(0), E));
        R S = R(0);
        for (int s = s0; s < s0 + n; ++s) {
            const R q = qval<Ld>(T, u, Vr, s);
            bad |= !isfinite(q);
            const R rv = post_op(dadd(Ld::ld(r + s), dadd(negE, q)), post, pf, nf);
            bad |= !isfinite(rv);
            r[s] = rv;
            S = dadd(S, rv > R(0) ? rv : R(0));
        }
        if (do_rm)
            for (int s = s0; s < s0 + n; ++s) bo[s] = rm_prob(Ld::ld(r + s), S, n);
    }
    if (bad) atomicOr(nonfinite, 1);
}

// PRED: observe the prediction m against the previous behaviour, floor if
// plus, regret-match the predicted regrets into b; r itself is untouched
// (the snapshot/restore of pkg/solvers.py:227-245 without the copy).
// MAXA: actions held in registers; wider DPs take the generic (recompute) path.
template <int MAXA, class Ld, class R>
__device__ __forceinline__ void pred_dp(const DevTree& T, int j, const R* __restrict__ m,
                                        const R* __restrict__ r, R* __restrict__ b,
                                        R* __restrict__ V, bool plus, const R* Vc = nullptr) {
    // Vc: where the child DPs' values are read (default V).  The level engine
    // points it at the prediction itself when the child level is all
    // forced moves into end nodes: their V would be exactly 0.0 + m, and a
    // parent's child sum cannot tell that from m (see leaf_note).
    const R* Vr = Vc ? Vc : V;
    int s0, n;
    dp_range<Ld>(T, j, s0, n);
    if (T.un == 1) {  // single-action level: b stays R(1) (see single_action_note)
        const R q = dadd(dadd(R(0), ld_u<Ld>(m, s0)), child_sum<Ld>(child_of<Ld>(T, s0), Vr));
        V[j] = dadd(R(0), dmul(R(1), q));
        return;
    }
    if (n <= MAXA) {
        R q[MAXA], bb[MAXA], rr[MAXA];
        load_q<MAXA, Ld>(T, m, Vr, s0, n, q);
#pragma unroll
        for (int a = 0; a < MAXA; ++a)
            if (a < n) {
                bb[a] = Ld::ld(b + s0 + a);
                rr[a] = Ld::ld(r + s0 + a);
            }
        R E = R(0);
#pragma unroll
        for (int a = 0; a < MAXA; ++a)
            if (a < n) E = dadd(E, dmul(bb[a], q[a]));
        V[j] = E;
        const R negE = dmul(R(-1), dadd(R(0), E));
        R S = R(0);
#pragma unroll
        for (int a = 0; a < MAXA; ++a)
            if (a < n) {
                R rv = dadd(rr[a], dadd(negE, q[a]));
                if (plus) rv = rv > R(0) ? rv : R(0);
                rr[a] = rv;
                S = dadd(S, rv > R(0) ? rv : R(0));
            }
#pragma unroll
        for (int a = 0; a < MAXA; ++a)
            if (a < n) b[s0 + a] = rm_prob(rr[a], S, n);
    } else {
        R E = R(0);
        for (int s = s0; s < s0 + n; ++s) E = dadd(E, dmul(Ld::ld(b + s), qval<Ld>(T, m, Vr, s)));
        V[j] = E;
        const R negE = dmul(R(-1), dadd(R(0), E));
        R S = R(0);
        for (int s = s0; s < s0 + n; ++s) {
            R rv = dadd(Ld::ld(r + s), dadd(negE, qval<Ld>(T, m, Vr, s)));
            if (plus) rv = rv > R(0) ? rv : R(0);
            S = dadd(S, rv > R(0) ? rv : R(0));
        }
        for (int s = s0; s < s0 + n; ++s) {
            R rv = dadd(Ld::ld(r + s), dadd(negE, qval<Ld>(T, m, Vr, s)));
            if (plus) rv = rv > R(0) ? rv : R(0);
            b[s] = rm_prob(rv, S, n);
        }
    }
}

// TD: x[(j,a)] = b[(j,a)] * x[parent(j)] (pkg/solvers.py:163-170), with the
// fused average update avg = w*x + avg (pkg/solvers.py:172-174).
// xp_in: the parent sequence's x when the caller already has it (the level
// engine's top: recomputed from the ancestor chain), else loaded from x.
template <class Ld, class R>
__device__ __forceinline__ void td_dp(const DevTree& T, int j, const R* __restrict__ b,
                                      R* __restrict__ x, typename nd<R>::type* __restrict__ avg,
                                      typename nd<R>::type w, const R* xp_in = nullptr) {
    int s0, n;
    dp_range<Ld>(T, j, s0, n);
    const int s1 = s0 + n;
    const R xp = xp_in ? *xp_in : Ld::ld(x + parent_of<Ld>(T, j));
    if (T.un == 1) {  // single-action level: b == R(1), so x = R(1) * xp (single_action_note)
        const R xa = dmul(R(1), xp);
        x[s0] = xa;
        if (avg) avg[s0] = dadd(dmul(w, xa), Ld::ld(avg + s0));
        return;
    }
    for (int s = s0; s < s1; ++s) {
        const R xa = dmul(Ld::ld(b + s), xp);
        x[s] = xa;
        if (avg) avg[s] = dadd(dmul(w, xa), Ld::ld(avg + s));
    }
}

// TD on a wide level, warp per DP (lane = action): the same per-sequence
// product and average update as td_dp, with the actions in parallel instead
// of a serial chain of loads (Liar's dice: up to 12 actions per DP).
template <class Ld, class R>
__device__ __forceinline__ void td_dp_warp(const DevTree& T, int j, const R* __restrict__ b,
                                           R* __restrict__ x, typename nd<R>::type* __restrict__ avg,
                                           typename nd<R>::type w, int lane, const R* xp_in = nullptr) {
    int s0, n;
    dp_range<Ld>(T, j, s0, n);
    const R xp = xp_in ? *xp_in : Ld::ld(x + parent_of<Ld>(T, j));
    for (int a = lane; a < n; a += 32) {
        const int s = s0 + a;
        const R xa = T.un == 1 ? dmul(R(1), xp) : dmul(Ld::ld(b + s), xp);
        x[s] = xa;
        if (avg) avg[s] = dadd(dmul(w, xa), Ld::ld(avg + s));
    }
}

// CUR: side-effect-free current strategy (pkg/solvers.py:270-291): regret
// matching on the fly, then the top-down product into x.
// MAXA: actions held in registers; wider DPs take the generic (recompute) path.
template <int MAXA, class Ld, class R>
__device__ __forceinline__ void cur_dp(const DevTree& T, int j, const R* __restrict__ r,
                                       R* __restrict__ x) {
    int s0, n;
    dp_range<Ld>(T, j, s0, n);
    const R xp = Ld::ld(x + parent_of<Ld>(T, j));
    if (T.un == 1) {  // single-action level: r == +R(0), RM gives R(1) (single_action_note)
        x[s0] = dmul(R(1), xp);
        return;
    }
    if (n <= MAXA) {
        R rr[MAXA];
#pragma unroll
        for (int a = 0; a < MAXA; ++a)
            if (a < n) rr[a] = Ld::ld(r + s0 + a);
        R S = R(0);
#pragma unroll
        for (int a = 0; a < MAXA; ++a)
            if (a < n) S = dadd(S, rr[a] > R(0) ? rr[a] : R(0));
#pragma unroll
        for (int a = 0; a < MAXA; ++a)
            if (a < n) x[s0 + a] = dmul(rm_prob(rr[a], S, n), xp);
    } else {
        R S = R(0);
        for (int s = s0; s < s0 + n; ++s) {
            const R v = Ld::ld(r + s);
            S = dadd(S, v > R(0) ? v : R(0));
        }
        for (int s = s0; s < s0 + n; ++s) x[s] = dmul(rm_prob(Ld::ld(r + s), S, n), xp);
    }
}

// BR: best response to gradient g (pkg/oracle.py:186-221): strict '>' from
// -inf in action order; value g + C_s with C_s the child sum as above.
template <class Ld, class R>
__device__ __forceinline__ void br_dp(const DevTree& T, int j, const R* __restrict__ g,
                                      R* __restrict__ W) {
    int s0, n;
    dp_range<Ld>(T, j, s0, n);
    const int s1 = s0 + n;
    R best = R(-INFINITY);
    for (int s = s0; s < s1; ++s) {
        const R v = dadd(Ld::ld(g + s), child_sum<Ld>(child_of<Ld>(T, s), W));
        if (v > best) best = v;
    }
    W[j] = best;
}

// ---------------------------------------------------------------------------
// Warp-per-DP variants for "fat" levels (few DPs, many child DPs per action,
// e.g. the top rounds of Goofspiel: 5 actions x 20 observed outcomes).  A
// thread-per-DP walk of those is a serial chain of dependent loads; here lane
// a owns action a, issues all of its child loads at once (32 in flight), sums
// them in order, and the per-DP sums run over lanes in action order through
// shuffles — the same association order, so still bit-exact.  All 32 lanes
// must call these together (j is warp-uniform).

constexpr unsigned kFullMask = 0xffffffffu;

template <class Ld, class R>
__device__ __forceinline__ R lane_child_value(int2 c, const R* __restrict__ V) {
    if (c.y == 0) return R(0);
    if (c.y == 1) return Ld::ld(V + c.x);
    if (c.y <= 4) {  // the common small observation points, unpredicated (same order)
        const R v0 = Ld::ld(V + c.x), v1 = Ld::ld(V + c.x + 1);
        if (c.y == 2) return dadd(dadd(R(0), v0), v1);
        const R v2 = Ld::ld(V + c.x + 2);
        if (c.y == 3) return dadd(dadd(dadd(R(0), v0), v1), v2);
        const R v3 = Ld::ld(V + c.x + 3);
        return dadd(dadd(dadd(dadd(R(0), v0), v1), v2), v3);
    }
    constexpr int CH = Ld::kChunk;
    R acc = R(0);
    for (int base = 0; base < c.y; base += CH) {
        R vv[CH];
#pragma unroll
        for (int k = 0; k < CH; ++k)
            if (base + k < c.y) vv[k] = Ld::ld(V + c.x + base + k);
#pragma unroll
        for (int k = 0; k < CH; ++k)
            if (base + k < c.y) acc = dadd(acc, vv[k]);
    }
    return acc;
}

// Sequential sum over lanes 0..n-1 of v: ((0.0 + v0) + v1) + ...
template <class R>
__device__ __forceinline__ R lane_seq_sum(R v, int n) {
    R acc = R(0);
    for (int a = 0; a < n; ++a) acc = dadd(acc, __shfl_sync(kFullMask, v, a));
    return acc;
}

// ---------------------------------------------------------------------------
// Group mode: on a big level whose DPs all have n = T.un actions (2..16), a
// warp runs G = 32/n DPs side by side, lane = (DP g, action a), so that
// consecutive lanes touch consecutive sequences (coalesced r / b / u / x /
// avg, and child ranges adjacent across lanes) instead of one thread walking
// its DP's n sequences.  The per-sequence arithmetic and the in-order sums
// are those of the thread and warp paths: group_seq_sum adds the group's n
// lanes from 0.0 in action order.  Every lane of the warp executes the
// shuffles (n is warp-uniform); `valid` masks the lanes past the level's end
// and the 32 - G*n idle lanes.

// N > 0: the group width is a compile-time constant (the common 2..4-action
// levels), so the shuffles unroll with no loop around them; N == 0: width n
// at run time.
template <int N = 0, class R>
__device__ __forceinline__ R group_seq_sum(R v, int gb, int n) {
    R acc = R(0);
    if constexpr (N == 2) {  // one shuffle: the partner's value (groups are aligned pairs)
        const R o = __shfl_xor_sync(kFullMask, v, 1);
        const bool first = ((threadIdx.x & 31) - gb) == 0;
        return dadd(dadd(R(0), first ? v : o), first ? o : v);
    } else if constexpr (N == 3) {  // two shuffles: the other two members, by rotation
        const int a = (int)(threadIdx.x & 31) - gb;
        const R n1 = __shfl_sync(kFullMask, v, gb + (a == 2 ? 0 : a + 1));
        const R n2 = __shfl_sync(kFullMask, v, gb + (a == 0 ? 2 : a - 1));
        // member values in group order: a = 0 -> (v, n1, n2), 1 -> (n2, v, n1), 2 -> (n1, n2, v)
        const R v0 = a == 0 ? v : a == 1 ? n2 : n1;
        const R v1 = a == 0 ? n1 : a == 1 ? v : n2;
        const R v2 = a == 0 ? n2 : a == 1 ? n1 : v;
        return dadd(dadd(dadd(R(0), v0), v1), v2);
    } else if constexpr (N > 0) {
#pragma unroll
        for (int a = 0; a < N; ++a) acc = dadd(acc, __shfl_sync(kFullMask, v, gb + a));
    } else {
        for (int a = 0; a < n; ++a) acc = dadd(acc, __shfl_sync(kFullMask, v, gb + a));
    }
    return acc;
}

template <class Ld, int N = 0, class R>
__device__ __forceinline__ void obs_dp_group(const DevTree& T, int j, bool valid, int a, int gb, int n,
                                             const R* __restrict__ u, R* __restrict__ r, R* __restrict__ b,
                                             R* __restrict__ V, int post, typename nd<R>::type pf,
                                             typename nd<R>::type nf, bool do_rm, int* nonfinite,
                                             FuseUT<R> fuse, const R* Vc, R* bw = nullptr, R* r_out = nullptr,
                                             const FuseUT<R>* cfu = nullptr, R* cu = nullptr, int cshift = 0) {
    // cfu: the child level is a forced leaf level whose utilities are
    // computed here (its fused payoff rows, written to cu) and used as the
    // child values directly (leaf_note); child DP c is sequence c + cshift
    if constexpr (N > 0) n = N;
    const R* Vr = Vc ? Vc : V;
    const int s = T.s_lo + (j - T.j_lo) * n + a;
    R q = R(0), bb = R(0), rr = R(0);
    bool bad = false;
    if (valid) {
        const int2 c = child_of<Ld>(T, s);
        const R uu = fuse.ip ? fused_u<Ld>(fuse, const_cast<R*>(u), s, bad) : ld_u<Ld>(u, s);
        bb = Ld::ld(b + s);
        rr = Ld::ld(r + s);
        R cv;
        if (cfu) {  // in-order child sum, as lane_child_value
            auto row = [&](int sc) {  // (±) payoff row sc, as fused_u without the store
                R v;
                if (cfu->rc > 0) {
                    const int k0 = cfu->rk0 + (sc - cfu->rs0) * cfu->rc;
                    v = spmv_range<Ld>(cfu->ix, cfu->d, cfu->x, k0, k0 + cfu->rc);
                } else {
                    v = spmv_row<Ld>(cfu->ip, cfu->ix, cfu->d, cfu->x, sc);
                }
                if (cfu->neg) v = dmul(R(-1), v);
                bad |= !isfinite(v);
                return v;
            };
            const int c0 = c.x + cshift;
            if (c.y == 1) {
                cv = row(c0);
                cu[c0] = cv;
            } else if (c.y == 2) {  // both rows' loads in flight before the stores
                const R v0 = row(c0), v1 = row(c0 + 1);
                cu[c0] = v0;
                cu[c0 + 1] = v1;
                cv = dadd(dadd(R(0), v0), v1);
            } else {
                cv = R(0);
                for (int k = 0; k < c.y; ++k) {
                    const R v = row(c0 + k);
                    cu[c0 + k] = v;
                    cv = dadd(cv, v);
                }
            }
        } else {
            cv = lane_child_value<Ld>(c, Vr);
        }
        q = dadd(dadd(R(0), uu), cv);
    }
    const R E = group_seq_sum<N>(dmul(bb, q), gb, n);
    if (valid && a == 0) V[j] = E;
    const R negE = dmul(R(-1), dadd(R(0), E));
    R rv = R(0);
    if (valid) {
        bad |= !isfinite(q);
        rv = post_op(dadd(rr, dadd(negE, q)), post, pf, nf);
        bad |= !isfinite(rv);
        (r_out ? r_out : r)[s] = rv;
    }
    const R S = group_seq_sum<N>(rv > R(0) ? rv : R(0), gb, n);
    if (do_rm && valid) (bw ? bw : b)[s] = rm_prob(rv, S, n);
    if (bad) atomicOr(nonfinite, 1);
}

template <class Ld, int N = 0, class R>
__device__ __forceinline__ void pred_dp_group(const DevTree& T, int j, bool valid, int a, int gb, int n,
                                              const R* __restrict__ m, const R* __restrict__ r,
                                              R* __restrict__ b, R* __restrict__ V, bool plus, const R* Vc,
                                              R* b_out = nullptr) {
    if constexpr (N > 0) n = N;
    const R* Vr = Vc ? Vc : V;
    const int s = T.s_lo + (j - T.j_lo) * n + a;
    R q = R(0), bb = R(0), rr = R(0);
    if (valid) {
        const int2 c = child_of<Ld>(T, s);
        const R mm = ld_u<Ld>(m, s);
        bb = Ld::ld(b + s);
        rr = Ld::ld(r + s);
        q = dadd(dadd(R(0), mm), lane_child_value<Ld>(c, Vr));
    }
    const R E = group_seq_sum<N>(dmul(bb, q), gb, n);
    if (valid && a == 0) V[j] = E;
    const R negE = dmul(R(-1), dadd(R(0), E));
    R rv = R(0);
    if (valid) {
        rv = dadd(rr, dadd(negE, q));
        if (plus) rv = rv > R(0) ? rv : R(0);
    }
    const R S = group_seq_sum<N>(rv > R(0) ? rv : R(0), gb, n);
    if (valid) (b_out ? b_out : b)[s] = rm_prob(rv, S, n);
}

// TD (+ average): x[s] = b[s] * x[parent(j)], avg[s] = w*x[s] + avg[s].
template <class Ld, class R>
__device__ __forceinline__ void td_dp_group(const DevTree& T, int j, bool valid, int a, int n,
                                            const R* __restrict__ b, R* __restrict__ x,
                                            typename nd<R>::type* __restrict__ avg, typename nd<R>::type w,
                                            const R* xp_in = nullptr) {
    if (!valid) return;
    const int s = T.s_lo + (j - T.j_lo) * n + a;
    const R xa = dmul(Ld::ld(b + s), xp_in ? *xp_in : Ld::ld(x + parent_of<Ld>(T, j)));
    x[s] = xa;
    if (avg) avg[s] = dadd(dmul(w, xa), Ld::ld(avg + s));
}

// CUR: regret matching on the fly, then the top-down product.
template <class Ld, int N = 0, class R>
__device__ __forceinline__ void cur_dp_group(const DevTree& T, int j, bool valid, int a, int gb, int n,
                                             const R* __restrict__ r, R* __restrict__ x) {
    if constexpr (N > 0) n = N;
    const int s = T.s_lo + (j - T.j_lo) * n + a;
    const R rv = valid ? Ld::ld(r + s) : R(0);
    const R S = group_seq_sum<N>(rv > R(0) ? rv : R(0), gb, n);
    if (valid) x[s] = dmul(rm_prob(rv, S, n), Ld::ld(x + parent_of<Ld>(T, j)));
}

// Out-of-line single-lane paths for DPs wider than a warp (rare): kept out
// of the warp kernels' register allocation (they run at 80 registers so 6
// CTAs fit per SM).
template <class Ld, class R>
__device__ __noinline__ void obs_dp_wide(const DevTree& T, int j, const R* __restrict__ u, R* __restrict__ r,
                                         R* __restrict__ b, R* __restrict__ V, int post,
                                         typename nd<R>::type pf, typename nd<R>::type nf, bool do_rm,
                                         int* nonfinite, FuseUT<R> fuse, const R* Vc, R* bw) {
    obs_dp<1, Ld>(T, j, u, r, b, V, post, pf, nf, do_rm, nonfinite, fuse, Vc, false, bw);
}
template <class Ld, class R>
__device__ __noinline__ void pred_dp_wide(const DevTree& T, int j, const R* __restrict__ m,
                                          const R* __restrict__ r, R* __restrict__ b, R* __restrict__ V,
                                          bool plus, const R* Vc) {
    pred_dp<1, Ld>(T, j, m, r, b, V, plus, Vc);
}

template <class Ld, class R>
__device__ __forceinline__ void obs_dp_warp(const DevTree& T, int j, const R* __restrict__ u,
                                            R* __restrict__ r, R* __restrict__ b,
                                            R* __restrict__ V, int post, typename nd<R>::type pf, typename nd<R>::type nf,
                                            bool do_rm, int* nonfinite, int lane,
                                            FuseUT<R> fuse = FuseUT<R>{}, const R* Vc = nullptr,
                                            R* bw = nullptr) {
    const R* Vr = Vc ? Vc : V;
    int s0, n;
    dp_range<Ld>(T, j, s0, n);
    if (n > 32) {  // wider than a warp: single-lane generic path
        if (lane == 0) obs_dp_wide<Ld>(T, j, u, r, b, V, post, pf, nf, do_rm, nonfinite, fuse, Vc, bw);
        return;
    }
    R q = R(0), bb = R(0), rr = R(0);
    bool bad = false;
    if (lane < n) {
        const int s = s0 + lane;
        const int2 c = child_of<Ld>(T, s);
        const R uu = fuse.ip ? fused_u<Ld>(fuse, const_cast<R*>(u), s, bad) : ld_u<Ld>(u, s);
        bb = Ld::ld(b + s);
        rr = Ld::ld(r + s);
        q = dadd(dadd(R(0), uu), lane_child_value<Ld>(c, Vr));
    }
    const R E = lane_seq_sum(dmul(bb, q), n);
    if (lane == 0) V[j] = E;
    const R negE = dmul(R(-1), dadd(R(0), E));
    R rv = R(0);
    if (lane < n) {
        bad |= !isfinite(q);
        rv = post_op(dadd(rr, dadd(negE, q)), post, pf, nf);
        bad |= !isfinite(rv);
        r[s0 + lane] = rv;
    }
    const R S = lane_seq_sum(rv > R(0) ? rv : R(0), n);
    if (do_rm && lane < n) (bw ? bw : b)[s0 + lane] = rm_prob(rv, S, n);
    if (__any_sync(kFullMask, bad) && lane == 0) atomicOr(nonfinite, 1);
}

template <class Ld, class R>
__device__ __forceinline__ void pred_dp_warp(const DevTree& T, int j, const R* __restrict__ m,
                                             const R* __restrict__ r, R* __restrict__ b,
                                             R* __restrict__ V, bool plus, int lane,
                                             const R* Vc = nullptr) {
    const R* Vr = Vc ? Vc : V;
    int s0, n;
    dp_range<Ld>(T, j, s0, n);
    if (n > 32) {
        if (lane == 0) pred_dp_wide<Ld>(T, j, m, r, b, V, plus, Vc);
        return;
    }
    R q = R(0), bb = R(0), rr = R(0);
    if (lane < n) {
        const int s = s0 + lane;
        const int2 c = child_of<Ld>(T, s);
        const R mm = ld_u<Ld>(m, s);
        bb = Ld::ld(b + s);
        rr = Ld::ld(r + s);
        q = dadd(dadd(R(0), mm), lane_child_value<Ld>(c, Vr));
    }
    const R E = lane_seq_sum(dmul(bb, q), n);
    if (lane == 0) V[j] = E;
    const R negE = dmul(R(-1), dadd(R(0), E));
    R rv = R(0);
    if (lane < n) {
        rv = dadd(rr, dadd(negE, q));
        if (plus) rv = rv > R(0) ? rv : R(0);
    }
    const R S = lane_seq_sum(rv > R(0) ? rv : R(0), n);
    if (lane < n) b[s0 + lane] = rm_prob(rv, S, n);
}

template <class Ld, class R>
__device__ __forceinline__ void br_dp_warp(const DevTree& T, int j, const R* __restrict__ g,
                                           R* __restrict__ W, int lane) {
    int s0, n;
    dp_range<Ld>(T, j, s0, n);
    if (n > 32) {
        if (lane == 0) br_dp<Ld>(T, j, g, W);
        return;
    }
    R v = R(0);
    if (lane < n) v = dadd(Ld::ld(g + s0 + lane), lane_child_value<Ld>(child_of<Ld>(T, s0 + lane), W));
    R best = R(-INFINITY);
    for (int a = 0; a < n; ++a) {
        const R x = __shfl_sync(kFullMask, v, a);
        if (x > best) best = x;
    }
    if (lane == 0) W[j] = best;
}

}  // namespace scfr
