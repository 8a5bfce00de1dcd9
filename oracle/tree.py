"""Pure-Python restatement of the reference compile step (TEST INFRASTRUCTURE).

Independent checker for the native tree compiler
(paper_2605_14277_b200/csrc/compiler.cpp).  Works on a FlatGame (so it sees
exactly what the C-ABI sees) and follows:

  DecisionProcess._extract   pkg/decision_process.py:76-242
  Game.chance_reach          pkg/games.py:93-103
  build_payoff_matrix        pkg/operators.py:164-180
  CsrMatrix.from_coo         pkg/kernels.py:95-112 (stable lexsort, bincount sums)
  CsrMatrix.transposed       pkg/kernels.py:114-127 (stable argsort)

Only tests/ and bench.py's CPU-baseline leg import this package.
"""

from __future__ import annotations

from collections import deque
from types import SimpleNamespace

import numpy as np

K_DEC, K_OBS, K_END = 0, 1, 2
G_CHANCE, G_DECISION, G_TERMINAL = 0, 1, 2


def extract(flat, player: int) -> SimpleNamespace:
    n = flat.num_nodes
    cp, ci = flat.child_ptr, flat.child_idx
    kind, pl, inf = flat.kind, flat.player, flat.infoset
    pid_of: dict[int, int] = {}
    first_key: list[int] = []
    parent_key: list[int] = []
    nact: list[int] = []
    first_node: list[int] = []
    kids_of_key: dict[int, list[int]] = {}
    prov = np.zeros(n, dtype=np.int64)
    next_key = 1
    order = [0]
    h = 0
    while h < len(order):
        order.extend(int(c) for c in ci[cp[order[h]]:cp[order[h] + 1]])
        h += 1
    for v in order:
        par = -1 if v == 0 else int(flat.parent[v])
        if v != 0:
            key = int(prov[par])
            if kind[par] == G_DECISION and pl[par] == player:
                kids = list(ci[cp[par]:cp[par + 1]])
                key = first_key[pid_of[int(inf[par])]] + kids.index(v)
            prov[v] = key
        if kind[v] == G_DECISION and pl[v] == player:
            key = int(prov[v])
            pid = pid_of.get(int(inf[v]))
            if pid is None:
                pid = len(first_key)
                pid_of[int(inf[v])] = pid
                first_key.append(next_key)
                parent_key.append(key)
                nact.append(int(cp[v + 1] - cp[v]))
                first_node.append(v)
                next_key += nact[-1]
                kids_of_key.setdefault(key, []).append(pid)
            elif parent_key[pid] != key:
                raise ValueError(f"perfect recall violated at node {v}")

    num_seqs = 1 + sum(nact)
    J = len(first_key)
    P = SimpleNamespace(kind=[], depth=[], parent=[], node_seq=[])
    seq_node = np.full(num_seqs, -1, dtype=np.int64)
    dp_node = np.zeros(J, dtype=np.int64)
    dp_first = np.zeros(J, dtype=np.int64)
    dp_nact = np.zeros(J, dtype=np.int64)
    dp_par = np.zeros(J, dtype=np.int64)
    j_of_pid = np.full(J, -1, dtype=np.int64)
    st = {"j": 0, "seq": 1}
    q: deque = deque([("seq", 0, -1, 0, kids_of_key.get(0, []))])

    def node(k, par, d, seq):
        nid = len(P.kind)
        P.kind.append(k)
        P.parent.append(par)
        P.depth.append(d)
        P.node_seq.append(seq)
        if seq >= 0:
            seq_node[seq] = nid
        return nid

    def open_dp(pid, par, d, parent_seq, seq):
        nid = node(K_DEC, par, d, seq)
        j = st["j"]
        st["j"] += 1
        j_of_pid[pid] = j
        dp_node[j], dp_first[j], dp_nact[j], dp_par[j] = nid, st["seq"], nact[pid], parent_seq
        for a in range(nact[pid]):
            q.append(("seq", st["seq"] + a, nid, d + 1, kids_of_key.get(first_key[pid] + a, [])))
        st["seq"] += nact[pid]

    while q:
        tag, a, par, d, rest = q.popleft()
        if tag == "seq":
            if not rest:
                node(K_END, par, d, a)
            elif len(rest) == 1:
                open_dp(rest[0], par, d, a, a)
            else:
                nid = node(K_OBS, par, d, a)
                for pid in rest:
                    q.append(("dp", pid, nid, d + 1, a))
        else:
            open_dp(a, par, d, rest, -1)

    depth = np.asarray(P.depth, dtype=np.int64)
    parent = np.asarray(P.parent, dtype=np.int64)
    height = int(depth.max())
    counts = np.bincount(parent[1:], minlength=len(depth)) if len(depth) > 1 else np.zeros(1, np.int64)
    fin = np.zeros(next_key, dtype=np.int64)
    for pid in range(J):
        j = j_of_pid[pid]
        fin[first_key[pid]:first_key[pid] + nact[pid]] = np.arange(dp_first[j], dp_first[j] + nact[pid])
    return SimpleNamespace(
        num_nodes=len(depth), num_decisions=J, num_seqs=num_seqs, height=height,
        degree=int(counts.max()) if counts.size else 0,
        kind=np.asarray(P.kind, dtype=np.int8), depth=depth, parent=parent,
        node_seq=np.asarray(P.node_seq, dtype=np.int64), seq_node=seq_node, dp_node=dp_node,
        dp_first_seq=dp_first, dp_num_actions=dp_nact, dp_parent_seq=dp_par,
        level_starts=np.searchsorted(depth, np.arange(height + 2)), game_seq=fin[prov])


def payoff(flat, p1, p2):
    reach = flat.chance_reach()
    z = flat.terminal_ids()
    r, c = p1.game_seq[z], p2.game_seq[z]
    v = flat.payoff[z] * reach[z]
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    if len(r):
        fresh = np.ones(len(r), dtype=bool)
        fresh[1:] = (np.diff(r) != 0) | (np.diff(c) != 0)
        grp = np.cumsum(fresh) - 1
        sums = np.zeros(grp[-1] + 1)
        for k in range(len(v)):  # sequential from 0.0, like np.bincount(weights=)
            sums[grp[k]] += v[k]
        v, r, c = sums, r[fresh], c[fresh]
    R, C = p1.num_seqs, p2.num_seqs
    indptr = np.zeros(R + 1, dtype=np.int64)
    np.add.at(indptr, r + 1, 1)
    indptr = np.cumsum(indptr)
    U = SimpleNamespace(rows=R, cols=C, indptr=indptr, indices=c.astype(np.int64), data=v,
                        nnz=len(v))
    row_of = np.repeat(np.arange(R, dtype=np.int64), np.diff(indptr))
    o = np.argsort(U.indices, kind="stable")
    tp = np.zeros(C + 1, dtype=np.int64)
    tp[1:] = np.cumsum(np.bincount(U.indices, minlength=C))
    UT = SimpleNamespace(rows=C, cols=R, indptr=tp, indices=row_of[o], data=U.data[o], nnz=len(v))
    return U, UT


def compile_flat(flat):
    p1, p2 = extract(flat, 1), extract(flat, 2)
    U, UT = payoff(flat, p1, p2)
    return SimpleNamespace(procs=(p1, p2), payoff=U, payoff_t=UT)
