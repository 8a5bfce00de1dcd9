// Native generators for the large fixture games.
//
// They emit exactly the trees of paper_2605_14277_b200.games.liars_dice and
// .goofspiel (same DFS pre-order node ids, same child order, same chance
// probabilities, infoset ids interned by first appearance), which
// tests/test_compiler.py checks on small sizes.  Goofspiel-5 has 8.5 M nodes:
// building it as Python objects takes about a minute, this takes well under
// a second.

#include <cmath>
#include <cstdint>
#include <unordered_map>
#include <vector>

#include "common.h"

namespace {

struct Builder {
    std::vector<int8_t> kind, player;
    std::vector<int64_t> parent, infoset;
    std::vector<double> prob, payoff;

    int64_t add(int8_t k, int64_t par, double pr, int8_t pl = 0, int64_t inf = -1,
                double pay = NAN) {
        kind.push_back(k);
        parent.push_back(par);
        prob.push_back(pr);
        player.push_back(pl);
        infoset.push_back(inf);
        payoff.push_back(pay);
        return (int64_t)kind.size() - 1;
    }
};

struct FlatOwner {
    scfr_flat_game pub;
    std::vector<int8_t> kind, player;
    std::vector<int64_t> parent, infoset, child_ptr, child_idx;
    std::vector<double> prob, payoff;
};

scfr_flat_game* finish(Builder& b, int64_t num_infosets) {
    auto* o = new FlatOwner();
    const int64_t n = (int64_t)b.kind.size();
    o->kind.swap(b.kind);
    o->player.swap(b.player);
    o->parent.swap(b.parent);
    o->infoset.swap(b.infoset);
    o->prob.swap(b.prob);
    o->payoff.swap(b.payoff);
    // Children in creation (= increasing id) order: stable counting sort by parent.
    o->child_ptr.assign(n + 1, 0);
    for (int64_t i = 1; i < n; ++i) o->child_ptr[o->parent[i] + 1]++;
    for (int64_t i = 0; i < n; ++i) o->child_ptr[i + 1] += o->child_ptr[i];
    o->child_idx.assign(n > 0 ? n - 1 : 0, 0);
    std::vector<int64_t> fill(o->child_ptr.begin(), o->child_ptr.end() - 1);
    for (int64_t i = 1; i < n; ++i) o->child_idx[fill[o->parent[i]]++] = i;
    scfr_game& g = o->pub.game;
    g.num_nodes = n;
    g.kind = o->kind.data();
    g.parent = o->parent.data();
    g.child_ptr = o->child_ptr.data();
    g.child_idx = o->child_idx.data();
    g.player = o->player.data();
    g.infoset = o->infoset.data();
    g.prob = o->prob.data();
    g.payoff = o->payoff.data();
    o->pub.num_infosets = num_infosets;
    return &o->pub;
}

// --- Liar's dice, one die each ------------------------------------------
struct Liars {
    int F, nb;
    Builder b;
    std::unordered_map<uint64_t, int64_t> ids;
    int64_t intern(int actor, int own, uint64_t hist_mask) {
        const uint64_t key = ((hist_mask * 64 + (uint64_t)own) << 1) | (uint64_t)(actor - 1);
        auto it = ids.find(key);
        if (it != ids.end()) return it->second;
        const int64_t id = (int64_t)ids.size();
        ids.emplace(key, id);
        return id;
    }
    void expand(int64_t par, double pr, int actor, int d1, int d2, int last, uint64_t mask) {
        const int own = actor == 1 ? d1 : d2;
        const int64_t me = b.add(SCFR_NODE_DECISION, par, pr, (int8_t)actor, intern(actor, own, mask));
        for (int k = last + 1; k < nb; ++k) expand(me, NAN, 3 - actor, d1, d2, k, mask | (1ull << k));
        if (last >= 0) {
            const int q = last / F + 1, f = last % F + 1;
            const int hits = (d1 == f || d1 == F) + (d2 == f || d2 == F);
            const int bidder = 3 - actor;
            const bool bidder_wins = hits >= q;
            const bool p1_wins = bidder_wins == (bidder == 1);
            b.add(SCFR_NODE_TERMINAL, me, NAN, 0, -1, p1_wins ? 1.0 : -1.0);
        }
    }
};

// --- Goofspiel ----------------------------------------------------------
struct Goof {
    Builder b;
    int64_t next_id = 0;
    void round(int64_t par, const std::vector<int>& left, const std::vector<int>& h1,
               const std::vector<int>& h2, int score) {
        const int64_t ch = b.add(SCFR_NODE_CHANCE, par, NAN);
        for (int p : left) {
            std::vector<int> rest;
            for (int x : left)
                if (x != p) rest.push_back(x);
            const int64_t d1 = b.add(SCFR_NODE_DECISION, ch, 1.0 / (double)left.size(), 1, next_id++);
            int64_t p2_id = -1;
            for (int b1 : h1) {
                if (p2_id < 0) p2_id = next_id++;
                const int64_t d2 = b.add(SCFR_NODE_DECISION, d1, NAN, 2, p2_id);
                for (int b2 : h2) {
                    const int s = score + (b1 > b2 ? p : (b2 > b1 ? -p : 0));
                    if (!rest.empty()) {
                        std::vector<int> n1, n2;
                        for (int x : h1)
                            if (x != b1) n1.push_back(x);
                        for (int x : h2)
                            if (x != b2) n2.push_back(x);
                        round(d2, rest, n1, n2, s);
                    } else {
                        b.add(SCFR_NODE_TERMINAL, d2, NAN, 0, -1, (double)((s > 0) - (s < 0)));
                    }
                }
            }
        }
    }
};

}  // namespace

using namespace scfr;

extern "C" {

int scfr_generate_liars_dice(int faces, scfr_flat_game** out) {
    return guarded([&] {
        if (!out || faces < 1 || faces > 30) fail(SCFR_EINVAL, "faces must be in [1, 30]");
        Liars L;
        L.F = faces;
        L.nb = 2 * faces;
        const int64_t root = L.b.add(SCFR_NODE_CHANCE, -1, NAN);
        for (int d1 = 1; d1 <= faces; ++d1) {
            const int64_t mid = L.b.add(SCFR_NODE_CHANCE, root, 1.0 / faces);
            for (int d2 = 1; d2 <= faces; ++d2) L.expand(mid, 1.0 / faces, 1, d1, d2, -1, 0);
        }
        *out = finish(L.b, (int64_t)L.ids.size());
    });
}

int scfr_generate_goofspiel(int cards, scfr_flat_game** out) {
    return guarded([&] {
        if (!out || cards < 1 || cards > 6) fail(SCFR_EINVAL, "cards must be in [1, 6]");
        Goof G;
        std::vector<int> deck;
        for (int c = 1; c <= cards; ++c) deck.push_back(c);
        G.round(-1, deck, deck, deck, 0);
        *out = finish(G.b, G.next_id);
    });
}

void scfr_flat_game_free(scfr_flat_game* g) { delete reinterpret_cast<FlatOwner*>(g); }

}  // extern "C"
