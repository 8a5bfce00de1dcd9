// Subtree partition for the subtree-sharded mode (subtree.h).  Host code only:
// scfr_create_subtree runs it on the structure it already converted, and the
// C-ABI scfr_subtree_plan runs it without a GPU (tests, planning tools).
#include "subtree.h"

#include <algorithm>
#include <cstdlib>

#include "common.h"

namespace scfr {

void host_levels(const scfr_tfsdp* p, std::vector<int>& seq_ptr, std::vector<int>& dp_parent,
                 std::vector<int>& lvl) {
    if (!p || p->num_seqs < 1 || p->num_decisions < 0) fail(SCFR_EINVAL, "bad tfsdp sizes");
    if (p->num_seqs >= (1ll << 31) / 2) fail(SCFR_EINVAL, "tfsdp too large for int32 indexing");
    if (!p->depth || !p->dp_node || !p->dp_first_seq || !p->dp_parent_seq) fail(SCFR_EINVAL, "tfsdp has a NULL array");
    const int J = (int)p->num_decisions;
    seq_ptr.assign(J + 1, (int)p->num_seqs);
    dp_parent.assign(J, 0);
    lvl.clear();
    int64_t prev = -1;
    for (int j = 0; j < J; ++j) {
        seq_ptr[j] = (int)p->dp_first_seq[j];
        dp_parent[j] = (int)p->dp_parent_seq[j];
        const int64_t d = p->depth[p->dp_node[j]];
        if (j == 0 || d != prev) lvl.push_back(j);
        prev = d;
    }
    lvl.push_back(J);
    // merge_levels (solver.cu): level l joins the current range unless one of
    // its DPs hangs under a sequence of that range
    const char* e = std::getenv("SCFR_NO_LEVEL_MERGE");
    const int L = (int)lvl.size() - 1;
    if ((e && e[0] == '1') || L < 2) return;
    std::vector<int> merged{0};
    int start = 0;
    for (int l = 1; l < L; ++l) {
        int mx = -1;
        for (int j = lvl[l]; j < lvl[l + 1]; ++j) mx = std::max(mx, dp_parent[j]);
        if (mx >= seq_ptr[start]) {
            start = lvl[l];
            merged.push_back(start);
        }
    }
    merged.push_back(J);
    lvl.swap(merged);
}

namespace {

// Deepest level l in [1, L-2] with at most kTrunkDPs trunk DPs above it and
// every deeper DP under a sequence of a level >= l DP; -1 if none.
int split_level(const HostProcess& P) {
    const std::vector<int>& lvl = *P.lvl;
    const int L = (int)lvl.size() - 1;
    for (int l = std::min(L - 2, 64); l >= 1; --l) {
        if (lvl[l] > kTrunkDPs) continue;
        const int s0 = P.seq_ptr[lvl[l]];
        bool ok = true;
        for (int q = lvl[l + 1]; q < P.J && ok; ++q) ok = P.dp_parent[q] >= s0;
        if (ok) return l;
    }
    return -1;
}

}  // namespace

void plan_subtrees(const HostProcess P[2], const scfr_csr* U, int world, SubtreePlan& plan) {
    if (world < 1) fail(SCFR_EINVAL, "bad world size");
    if (!U || !U->indptr || (U->nnz && (!U->indices || !U->data))) fail(SCFR_EINVAL, "NULL payoff matrix");
    if (U->rows != P[0].S || U->cols != P[1].S) fail(SCFR_EINVAL, "payoff shape does not match the processes");
    plan = SubtreePlan{};
    plan.world = world;
    std::vector<int> rootS[2], rootJ[2];  // root of each forest sequence (s - sf0) / DP (q - lvl[ls])
    int sf0[2];
    for (int k = 0; k < 2; ++k) {
        const HostProcess& H = P[k];
        const std::vector<int>& lvl = *H.lvl;
        const int L = (int)lvl.size() - 1;
        const int ls = split_level(H);
        if (ls < 0)
            fail(SCFR_EINVAL, "player %d has no subtree split (a trunk of <= %d decision points over a forest)",
                 k + 1, kTrunkDPs);
        plan.ls[k] = ls;
        const int j0 = lvl[ls], j1 = lvl[ls + 1];
        plan.roots[k] = j1 - j0;
        sf0[k] = H.seq_ptr[j0];
        rootS[k].assign(H.S - sf0[k], -1);
        rootJ[k].assign(H.J - j0, 0);
        for (int q = j0; q < H.J; ++q) {
            const int r = q < j1 ? q - j0 : rootS[k][H.dp_parent[q] - sf0[k]];
            rootJ[k][q - j0] = r;
            for (int s = H.seq_ptr[q]; s < H.seq_ptr[q + 1]; ++s) rootS[k][s - sf0[k]] = r;
        }
        // a rank's DPs of a forest level must be one contiguous range
        for (int l = ls + 1; l < L; ++l)
            for (int q = lvl[l] + 1; q < lvl[l + 1]; ++q)
                if (rootJ[k][q - j0] < rootJ[k][q - 1 - j0])
                    fail(SCFR_EINVAL, "player %d: level %d is not ordered by subtree root", k + 1, l);
        plan.jb[k].assign(L, {});
        plan.sb[k].assign(L, {});
    }
    // payoff coupling: each player-1 root's range of player-2 roots
    const int R1 = plan.roots[0], R2 = plan.roots[1];
    std::vector<int> mx(R1, -1), mn(R1, R2);
    for (int64_t s1 = 0; s1 < U->rows; ++s1) {
        const bool f1 = s1 >= sf0[0];
        for (int64_t e = U->indptr[s1]; e < U->indptr[s1 + 1]; ++e) {
            const int64_t s2 = U->indices[e];
            const bool f2 = s2 >= sf0[1];
            if (f1 != f2)
                fail(SCFR_EINVAL, "the payoff couples a trunk sequence with a subtree sequence (row %lld, column %lld)",
                     (long long)s1, (long long)s2);
            if (!f1) continue;
            const int a = rootS[0][s1 - sf0[0]], b = rootS[1][s2 - sf0[1]];
            mx[a] = std::max(mx[a], b);
            mn[a] = std::min(mn[a], b);
        }
    }
    // forest sequences per root (the work measure of the balance)
    std::vector<int64_t> W[2];
    for (int k = 0; k < 2; ++k) {
        W[k].assign(plan.roots[k] + 1, 0);
        for (int r : rootS[k]) W[k][r + 1] += 1;
        for (int r = 0; r < plan.roots[k]; ++r) W[k][r + 1] += W[k][r];
    }
    // closed cuts (i, j): player-1 roots < i reference only player-2 roots < j,
    // roots >= i only roots >= j: max over [0, i) < j <= min over [i, R1)
    std::vector<int> pm(R1 + 1, -1), sm(R1 + 1, R2);
    for (int i = 0; i < R1; ++i) pm[i + 1] = std::max(pm[i], mx[i]);
    for (int i = R1 - 1; i >= 0; --i) sm[i] = std::min(sm[i + 1], mn[i]);
    const double total = (double)(W[0][R1] + W[1][R2]);
    for (int k = 0; k < 2; ++k) plan.cut[k].assign(world + 1, 0);
    plan.cut[0][world] = R1;
    plan.cut[1][world] = R2;
    int pi = 0, pj = 0;
    for (int r = 1; r < world; ++r) {
        const double target = total * r / world;
        double best = -1.0;
        int bi = -1, bj = -1;
        for (int i = pi + 1; i <= R1 - (world - r); ++i) {
            const int lo = std::max(pm[i] + 1, pj), hi = sm[i];
            if (lo > hi) continue;
            // player-2 cut nearest the target given i, clamped into [lo, hi]
            const double want = target - (double)W[0][i];
            int j = (int)(std::lower_bound(W[1].begin(), W[1].end(), (int64_t)std::max(0.0, want)) - W[1].begin());
            j = std::min(std::max(j, lo), hi);
            const double cost = std::abs((double)(W[0][i] + W[1][j]) - target);
            if (best < 0 || cost < best) {
                best = cost;
                bi = i;
                bj = j;
            }
        }
        if (bi < 0)
            fail(SCFR_EINVAL, "the payoff splits the subtrees into fewer than %d closed blocks", world);
        plan.cut[0][r] = pi = bi;
        plan.cut[1][r] = pj = bj;
    }
    for (int k = 0; k < 2; ++k) {
        const HostProcess& H = P[k];
        const std::vector<int>& lvl = *H.lvl;
        const int L = (int)lvl.size() - 1, ls = plan.ls[k], j0 = lvl[ls];
        const std::vector<int>& roots = rootJ[k];
        plan.seqs[k].assign(world, 0);
        for (int l = ls; l < L; ++l) {
            std::vector<int>& jb = plan.jb[k][l];
            std::vector<int>& sb = plan.sb[k][l];
            jb.assign(world + 1, lvl[l + 1]);
            for (int r = 0; r < world; ++r) {
                const auto first = roots.begin() + (lvl[l] - j0), last = roots.begin() + (lvl[l + 1] - j0);
                jb[r] = lvl[l] + (int)(std::lower_bound(first, last, (int)plan.cut[k][r]) - first);
            }
            sb.resize(world + 1);
            for (int r = 0; r <= world; ++r) sb[r] = H.seq_ptr[jb[r]];
            for (int r = 0; r < world; ++r) plan.seqs[k][r] += sb[r + 1] - sb[r];
        }
    }
}

}  // namespace scfr

using namespace scfr;

extern "C" int scfr_subtree_plan(const scfr_tfsdp* p1, const scfr_tfsdp* p2, const scfr_csr* U, int world,
                                 int32_t* ls_out, int64_t* cuts_out, int64_t* seqs_out) {
    return guarded([&] {
        if (!p1 || !p2 || !U || !ls_out || !cuts_out) fail(SCFR_EINVAL, "NULL argument");
        std::vector<int> sp[2], par[2], lvl[2];
        host_levels(p1, sp[0], par[0], lvl[0]);
        host_levels(p2, sp[1], par[1], lvl[1]);
        HostProcess H[2];
        for (int k = 0; k < 2; ++k)
            H[k] = HostProcess{sp[k].data(), par[k].data(), &lvl[k], (int)par[k].size(),
                               (int)(k == 0 ? p1 : p2)->num_seqs};
        SubtreePlan plan;
        plan_subtrees(H, U, world, plan);
        for (int k = 0; k < 2; ++k) {
            ls_out[k] = plan.ls[k];
            for (int r = 0; r <= world; ++r) cuts_out[(size_t)k * (world + 1) + r] = plan.cut[k][r];
            if (seqs_out)
                for (int r = 0; r < world; ++r) seqs_out[(size_t)k * world + r] = plan.seqs[k][r];
        }
    });
}
