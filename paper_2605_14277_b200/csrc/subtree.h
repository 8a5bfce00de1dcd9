// Subtree partition of the two decision processes for the subtree-sharded
// multi-GPU mode (scfr_create_subtree).
//
// The reference solves one tree on one device (pkg/decision_process.py
// :219-231 builds the level operators of the whole process)
// names the multi-GPU split: replicate the trunk, give each device whole
// subtrees.  Here the split level ls of each player is the deepest (merged)
// level whose trunk [0, ls) holds at most kTrunkDPs decision points and below
// which every DP hangs under a level->=ls sequence (a forest of level-ls
// roots).  Rank r owns the contiguous root range [cut[r], cut[r+1]) of each
// player; the cuts are chosen where no payoff entry couples a root of one
// rank's player-1 range with a root outside its player-2 range, so a rank's
// fused payoff rows read only its own subtrees' and the trunk's x.  Within
// every forest level the roots are non-decreasing in DP order, so a rank's
// DPs of that level are one contiguous range (jb) and its sequences too (sb).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/seqcfr_b200.h"

namespace scfr {

constexpr int kTrunkDPs = 4096;

struct SubtreePlan {
    int world = 1;
    int ls[2] = {-1, -1};          // first forest level of each player (merged level index)
    int roots[2] = {0, 0};         // level-ls DPs
    std::vector<int64_t> cut[2];   // [world + 1] root boundaries
    // per level l (empty below ls): [world + 1] DP / sequence boundaries
    std::vector<std::vector<int>> jb[2], sb[2];
    std::vector<int64_t> seqs[2];  // [world] forest sequences per rank
};

// One player's host structure: seq_ptr [J + 1], dp_parent [J], merged level
// starts [L + 1].
struct HostProcess {
    const int* seq_ptr;
    const int* dp_parent;
    const std::vector<int>* lvl;
    int J, S;
};

// Fills `plan`, or throws Error(SCFR_EINVAL, why) when the game has no split
// that the subtree mode can run (trunk rows coupled to subtree columns, too
// few closed root blocks for `world` ranks, ...).
void plan_subtrees(const HostProcess P[2], const scfr_csr* U, int world, SubtreePlan& plan);

// The merged level starts of a decision process, sequentially (the solver's
// merge_levels, solver.cu, is the parallel twin used at create).
void host_levels(const scfr_tfsdp* p, std::vector<int>& seq_ptr, std::vector<int>& dp_parent,
                 std::vector<int>& lvl);

}  // namespace scfr
