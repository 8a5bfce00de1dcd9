// sm_100a kernels for one CFR iteration over per-DP-level index arrays.
//
// Bit-faithful fp64: every operation is an explicit round-to-nearest
// intrinsic in the exact association order of the reference (SURVEY.md
// §8(a) "exact arithmetic contract"); the translation unit is also compiled
// with -fmad=false so nothing is contracted into an FMA.  Sums are
// sequential per output element, exactly one thread owns each output, so
// results are deterministic and equal to the numba loops bit for bit.
//
// Layout (per player, per solve; all solves of a batch are strided copies):
//   seq-indexed fp64 vectors over Σ (slot 0 = empty sequence): r, b, x,
//     xpost, avg, u, g   — r/b slot 0 unused (reference Σ+ index = s-1)
//   dp-indexed fp64 temporaries over J: V (sum pass), W (max pass)
//   structure (int32, read-only): seq_ptr[J+1] (action range of DP j),
//     dp_parent[J] (parent sequence), child[S] = {lo, cnt} (child-DP range of
//     sequence s: cnt 0 = end node, 1 = a single DP, >1 = observation point)
//   DP levels: DPs grouped by process-tree depth; BFS numbering makes each
//     level a contiguous j range (pkg/decision_process.py:9-13).
#pragma once

#include <cstdint>

namespace scfr {

struct DevTree {
    const int* __restrict__ seq_ptr;    // [J+1]
    const int* __restrict__ dp_parent;  // [J]
    const int2* __restrict__ child;     // [S]
};

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// Value flowing up into sequence s from the decision points below it.
// End node: the zero-initialised v (0.0).  One DP: v of that DP node (its
// V).  Observation point: sequential sum over its child DPs in j order
// starting at 0.0 (pkg/solvers.py:195-199 / pkg/oracle.py:91-95).
__device__ __forceinline__ double child_sum(int2 c, const double* __restrict__ V) {
    if (c.y == 0) return 0.0;
    if (c.y == 1) return __ldcg(V + c.x);
    double acc = 0.0;
    for (int k = 0; k < c.y; ++k) acc = dadd(acc, __ldcg(V + c.x + k));
    return acc;
}

// Counterfactual value of action s: q = (0.0 + u[s]) + C_s, which is
// (w + v)[node(s)] read back through Bᵀ (pkg/solvers.py:192-202).
__device__ __forceinline__ double qval(const DevTree& T, const double* __restrict__ u,
                                       const double* __restrict__ V, int s) {
    return dadd(dadd(0.0, __ldcg(u + s)), child_sum(__ldg(T.child + s), V));
}

enum : int { POST_NONE = 0, POST_PLUS = 1, POST_DCFR = 2 };

// Regret matching of one DP block (pkg/solvers.py:156-160): positive part,
// sequential block sum from 0.0, IEEE division, uniform 1.0/n fallback.
__device__ __forceinline__ double rm_sum(const double* __restrict__ r, int s0, int s1) {
    double S = 0.0;
    for (int s = s0; s < s1; ++s) {
        const double v = __ldcg(r + s);
        S = dadd(S, v > 0.0 ? v : 0.0);
    }
    return S;
}
__device__ __forceinline__ double rm_prob(double rv, double S, int n) {
    const double p = rv > 0.0 ? rv : 0.0;
    return S != 0.0 ? ddiv(p, S) : ddiv(1.0, (double)n);
}

// ---------------------------------------------------------------------------
// OBS: bottom-up counterfactual values + regret update (+ variant post-op)
// (+ regret matching of the updated regrets into b for the next iteration).
// pkg/solvers.py:178-224 and :143-160, fused per decision point.
__device__ __forceinline__ void obs_dp(const DevTree& T, int j, const double* __restrict__ u,
                                       double* __restrict__ r, double* __restrict__ b,
                                       double* __restrict__ V, int post, double pf, double nf,
                                       bool do_rm, int* nonfinite) {
    const int s0 = __ldg(T.seq_ptr + j), s1 = __ldg(T.seq_ptr + j + 1);
    double E = 0.0;
    for (int s = s0; s < s1; ++s) E = dadd(E, dmul(__ldcg(b + s), qval(T, u, V, s)));
    V[j] = E;
    const double negE = dmul(-1.0, dadd(0.0, E));
    bool bad = false;
    for (int s = s0; s < s1; ++s) {
        const double q = qval(T, u, V, s);
        bad |= !isfinite(q);
        double rv = dadd(__ldcg(r + s), dadd(negE, q));
        if (post == POST_PLUS) {
            rv = rv > 0.0 ? rv : 0.0;
        } else if (post == POST_DCFR) {
            rv = rv > 0.0 ? dmul(rv, pf) : (rv < 0.0 ? dmul(rv, nf) : rv);
        }
        bad |= !isfinite(rv);
        r[s] = rv;
    }
    if (bad) atomicOr(nonfinite, 1);
    if (do_rm) {
        const double S = rm_sum(r, s0, s1);
        for (int s = s0; s < s1; ++s) b[s] = rm_prob(__ldcg(r + s), S, s1 - s0);
    }
}

// PRED: observe the prediction m against the previous behaviour, floor if
// plus, regret-match the predicted regrets into b; r itself is untouched
// (snapshot/restore of pkg/solvers.py:227-245 without the copy).
__device__ __forceinline__ void pred_dp(const DevTree& T, int j, const double* __restrict__ m,
                                        const double* __restrict__ r, double* __restrict__ b,
                                        double* __restrict__ V, bool plus) {
    const int s0 = __ldg(T.seq_ptr + j), s1 = __ldg(T.seq_ptr + j + 1);
    double E = 0.0;
    for (int s = s0; s < s1; ++s) E = dadd(E, dmul(__ldcg(b + s), qval(T, m, V, s)));
    V[j] = E;
    const double negE = dmul(-1.0, dadd(0.0, E));
    double S = 0.0;
    for (int s = s0; s < s1; ++s) {
        double rv = dadd(__ldcg(r + s), dadd(negE, qval(T, m, V, s)));
        if (plus) rv = rv > 0.0 ? rv : 0.0;
        S = dadd(S, rv > 0.0 ? rv : 0.0);
    }
    for (int s = s0; s < s1; ++s) {
        double rv = dadd(__ldcg(r + s), dadd(negE, qval(T, m, V, s)));
        if (plus) rv = rv > 0.0 ? rv : 0.0;
        b[s] = rm_prob(rv, S, s1 - s0);
    }
}

// TD: x[(j,a)] = b[(j,a)] * x[parent(j)] (pkg/solvers.py:163-170), with the
// fused average update avg = w*x + avg (pkg/solvers.py:172-174).
__device__ __forceinline__ void td_dp(const DevTree& T, int j, const double* __restrict__ b,
                                      double* __restrict__ x, double* __restrict__ avg,
                                      double w) {
    const int s0 = __ldg(T.seq_ptr + j), s1 = __ldg(T.seq_ptr + j + 1);
    const double xp = __ldcg(x + __ldg(T.dp_parent + j));
    for (int s = s0; s < s1; ++s) {
        const double xa = dmul(__ldcg(b + s), xp);
        x[s] = xa;
        if (avg) avg[s] = dadd(dmul(w, xa), __ldcg(avg + s));
    }
}

// CUR: side-effect-free current strategy (pkg/solvers.py:270-291): regret
// matching on the fly, then the top-down product into xpost.
__device__ __forceinline__ void cur_dp(const DevTree& T, int j, const double* __restrict__ r,
                                       double* __restrict__ x) {
    const int s0 = __ldg(T.seq_ptr + j), s1 = __ldg(T.seq_ptr + j + 1);
    const double S = rm_sum(r, s0, s1);
    const double xp = __ldcg(x + __ldg(T.dp_parent + j));
    for (int s = s0; s < s1; ++s) x[s] = dmul(rm_prob(__ldcg(r + s), S, s1 - s0), xp);
}

// BR: best response to gradient g (pkg/oracle.py:186-221): strict '>' from
// -inf in action order; s = g + C_s with C_s the child-DP sum as above.
__device__ __forceinline__ void br_dp(const DevTree& T, int j, const double* __restrict__ g,
                                      double* __restrict__ W) {
    const int s0 = __ldg(T.seq_ptr + j), s1 = __ldg(T.seq_ptr + j + 1);
    double best = -INFINITY;
    for (int s = s0; s < s1; ++s) {
        const double v = dadd(__ldcg(g + s), child_sum(__ldg(T.child + s), W));
        if (v > best) best = v;
    }
    W[j] = best;
}

// Payoff SpMV row: ((0.0 + d0*x[c0]) + d1*x[c1]) + ... (pkg/kernels.py:149-154),
// optionally scaled by -1.0 (backend.scale(-1.0, ...), pkg/solvers.py:359,368).
__device__ __forceinline__ double spmv_row(const int* __restrict__ indptr,
                                           const int* __restrict__ indices,
                                           const double* __restrict__ data,
                                           const double* __restrict__ x, int row) {
    const int k0 = __ldg(indptr + row), k1 = __ldg(indptr + row + 1);
    double acc = 0.0;
    for (int k = k0; k < k1; ++k) acc = dadd(acc, dmul(__ldg(data + k), __ldcg(x + __ldg(indices + k))));
    return acc;
}

}  // namespace scfr
