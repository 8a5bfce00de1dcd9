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


# ---------------------------------------------------------------------------
# The same compile step in C (oracle/seqcfr_tree.c), plus the fixture-game
# generators, so the checker side can build Goofspiel-5 (8.5 M nodes) without
# the product library.  Pinned to the reference by tests/test_oracle_tree.py.

import ctypes as _C  # noqa: E402
import os as _os  # noqa: E402

_TREE_LIB = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "_build",
                          "libseqcfr_tree.so")
_tl = None


class _Game(_C.Structure):
    _fields_ = [("n", _C.c_int64), ("num_infosets", _C.c_int64),
                ("kind", _C.POINTER(_C.c_int8)), ("player", _C.POINTER(_C.c_int8)),
                ("parent", _C.POINTER(_C.c_int64)), ("child_ptr", _C.POINTER(_C.c_int64)),
                ("child_idx", _C.POINTER(_C.c_int64)), ("infoset", _C.POINTER(_C.c_int64)),
                ("prob", _C.POINTER(_C.c_double)), ("payoff", _C.POINTER(_C.c_double))]


class _Proc(_C.Structure):
    _fields_ = [(f, _C.c_int64) for f in ("num_nodes", "num_decisions", "num_seqs", "height",
                                          "degree")] + \
        [("kind", _C.POINTER(_C.c_int8))] + \
        [(f, _C.POINTER(_C.c_int64)) for f in ("depth", "parent", "node_seq", "seq_node",
                                              "dp_node", "dp_first_seq", "dp_num_actions",
                                              "dp_parent_seq", "level_starts", "game_seq")]


class _Csr(_C.Structure):
    _fields_ = [("rows", _C.c_int64), ("cols", _C.c_int64), ("nnz", _C.c_int64),
                ("indptr", _C.POINTER(_C.c_int64)), ("indices", _C.POINTER(_C.c_int64)),
                ("data", _C.POINTER(_C.c_double))]


def _tree_lib():
    global _tl
    if _tl is None:
        if not _os.path.exists(_TREE_LIB):
            import subprocess
            subprocess.run(["make", "-s", "-C", _os.path.dirname(_TREE_LIB) + "/.."], check=True)
        L = _C.CDLL(_TREE_LIB)
        P = _C.POINTER
        L.ot_goofspiel.restype = P(_Game)
        L.ot_goofspiel.argtypes = [_C.c_int]
        L.ot_liars_dice.restype = P(_Game)
        L.ot_liars_dice.argtypes = [_C.c_int]
        L.ot_game_free.argtypes = [P(_Game)]
        L.ot_extract.restype = P(_Proc)
        L.ot_extract.argtypes = [_C.c_int64, P(_C.c_int8), P(_C.c_int64), P(_C.c_int64),
                                 P(_C.c_int64), P(_C.c_int8), P(_C.c_int64), _C.c_int,
                                 P(_C.c_int)]
        L.ot_proc_free.argtypes = [P(_Proc)]
        L.ot_payoff.restype = _C.c_int
        L.ot_payoff.argtypes = [_C.c_int64, P(_C.c_int8), P(_C.c_int64), P(_C.c_double),
                                P(_C.c_double), P(_Proc), P(_Proc), P(P(_Csr)), P(P(_Csr))]
        L.ot_csr_free.argtypes = [P(_Csr)]
        _tl = L
    return _tl


def _np(ptr, n, dt):
    return np.ctypeslib.as_array(ptr, shape=(int(n),)).astype(dt, copy=True) if n else \
        np.zeros(0, dtype=dt)


def native_game(name: str, size: int) -> SimpleNamespace:
    """Flat arrays of ``goofspiel(size)`` or ``liars_dice(size)`` from the C
    generators (same trees as the product's games.py generators)."""
    L = _tree_lib()
    gp = {"goofspiel": L.ot_goofspiel, "liars_dice": L.ot_liars_dice}[name](int(size))
    if not gp:
        raise ValueError(f"oracle generator refused {name}({size})")
    g = gp.contents
    n = g.n
    try:
        flat = SimpleNamespace(
            num_nodes=int(n), kind=_np(g.kind, n, np.int8), player=_np(g.player, n, np.int8),
            parent=_np(g.parent, n, np.int64), child_ptr=_np(g.child_ptr, n + 1, np.int64),
            child_idx=_np(g.child_idx, max(n - 1, 0), np.int64),
            infoset=_np(g.infoset, n, np.int64), prob=_np(g.prob, n, np.float64),
            payoff=_np(g.payoff, n, np.float64))
    finally:
        L.ot_game_free(gp)
    return flat


def compile_native(flat) -> SimpleNamespace:
    """Reference compile step (DecisionProcess x2, U, U^T) on flat arrays, in C."""
    L = _tree_lib()
    P = _C.POINTER
    a = {f: np.ascontiguousarray(getattr(flat, f), dtype=dt) for f, dt in
         (("kind", np.int8), ("parent", np.int64), ("child_ptr", np.int64),
          ("child_idx", np.int64), ("player", np.int8), ("infoset", np.int64),
          ("prob", np.float64), ("payoff", np.float64))}
    ptr = {f: v.ctypes.data_as(P(_C.c_int8 if v.dtype == np.int8 else
                                  _C.c_double if v.dtype == np.float64 else _C.c_int64))
           for f, v in a.items()}
    n = int(a["kind"].shape[0])
    procs, raw = [], []
    try:
        for pl in (1, 2):
            err = _C.c_int(0)
            pp = L.ot_extract(n, ptr["kind"], ptr["parent"], ptr["child_ptr"], ptr["child_idx"],
                              ptr["player"], ptr["infoset"], pl, _C.byref(err))
            if not pp:
                raise ValueError(f"oracle compile failed for player {pl} (code {err.value})")
            raw.append(pp)
            p = pp.contents
            nn, nj, ns, h = p.num_nodes, p.num_decisions, p.num_seqs, p.height
            procs.append(SimpleNamespace(
                num_nodes=int(nn), num_decisions=int(nj), num_seqs=int(ns), height=int(h),
                degree=int(p.degree), kind=_np(p.kind, nn, np.int8),
                depth=_np(p.depth, nn, np.int64), parent=_np(p.parent, nn, np.int64),
                node_seq=_np(p.node_seq, nn, np.int64), seq_node=_np(p.seq_node, ns, np.int64),
                dp_node=_np(p.dp_node, nj, np.int64),
                dp_first_seq=_np(p.dp_first_seq, nj, np.int64),
                dp_num_actions=_np(p.dp_num_actions, nj, np.int64),
                dp_parent_seq=_np(p.dp_parent_seq, nj, np.int64),
                level_starts=_np(p.level_starts, h + 2, np.int64),
                game_seq=_np(p.game_seq, n, np.int64)))
        U, UT = P(_Csr)(), P(_Csr)()
        if L.ot_payoff(n, ptr["kind"], ptr["parent"], ptr["prob"], ptr["payoff"], raw[0], raw[1],
                       _C.byref(U), _C.byref(UT)):
            raise MemoryError("oracle payoff build failed")
        mats = []
        for m in (U, UT):
            c = m.contents
            mats.append(SimpleNamespace(rows=int(c.rows), cols=int(c.cols), nnz=int(c.nnz),
                                        indptr=_np(c.indptr, c.rows + 1, np.int64),
                                        indices=_np(c.indices, c.nnz, np.int64),
                                        data=_np(c.data, c.nnz, np.float64)))
            L.ot_csr_free(m)
    finally:
        for pp in raw:
            L.ot_proc_free(pp)
    return SimpleNamespace(procs=tuple(procs), payoff=mats[0], payoff_t=mats[1])


def native_bundle(name: str, size: int) -> SimpleNamespace:
    """Product-free bundle of a generated fixture game (the bench's reference
    arm and CPU baseline use this; no paper_2605_14277_b200 code runs)."""
    return compile_native(native_game(name, size))
