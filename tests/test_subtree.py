"""Subtree-sharded mode (C-ABI scfr_create_subtree / scfr_subtree_plan).

CPU: the native planner's partition (distributed.subtree_plan) checked on its
own terms — every subtree root owned by exactly one rank, each rank's DPs of
every level one contiguous range, payoff rows that read only the rank's own
subtrees and the trunk — and a gloo world-2 run of the sharded schedule: each
rank computes its payoff rows and a bottom-up value pass over its own
subtrees with every other rank's subtree state poisoned (NaN), the ranks
exchange the subtree roots' values, every rank finishes the trunk, and the
result must equal the one-process computation bit for bit.

GPU: the CUDA path over real NCCL at world 1, and the range-restricted
launches of a W-rank plan run back to back on one GPU (SCFR_SUBTREE_SIM=W),
both against the reference digests.
"""

import os
import socket

import numpy as np
import pytest

from conftest import ROOT, bundle, digest, golden_meta

# ---------------------------------------------------------------- structure


def _levels(p):
    """Merged level starts, as host_levels / merge_levels (csrc/subtree.cpp)."""
    J = p.num_decisions
    dpd = np.asarray(p.depth)[np.asarray(p.dp_node)]
    starts = [0] + (np.flatnonzero(np.diff(dpd)) + 1).tolist() + [J]
    sp = np.append(np.asarray(p.dp_first_seq), p.num_seqs)
    par = np.asarray(p.dp_parent_seq)
    merged, start = [0], 0
    for l in range(1, len(starts) - 1):
        if par[starts[l]:starts[l + 1]].max() >= sp[start]:
            start = starts[l]
            merged.append(start)
    return merged + [J]


def _roots(p, lvl, ls):
    """Subtree root of every DP and sequence (-1 in the trunk)."""
    J, S = p.num_decisions, p.num_seqs
    sp = np.append(np.asarray(p.dp_first_seq), S)
    par = np.asarray(p.dp_parent_seq)
    j0, j1 = lvl[ls], lvl[ls + 1]
    rj = np.full(J, -1, dtype=np.int64)
    rs = np.full(S, -1, dtype=np.int64)
    for q in range(j0, J):
        rj[q] = q - j0 if q < j1 else rs[par[q]]
        rs[sp[q]:sp[q + 1]] = rj[q]
    return rj, rs


def _owner(cuts, root):
    return np.searchsorted(np.asarray(cuts), root, side="right") - 1


@pytest.mark.parametrize("game", ["goof3", "goof4"])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_plan_partitions_the_forest(game, world):
    from paper_2605_14277_b200.distributed import subtree_plan
    b = bundle(game)
    plan = subtree_plan(b, world)
    rs_all = []
    for k, p in enumerate(b.procs):
        cuts = plan["cuts"][k]
        lvl = _levels(p)
        ls = plan["ls"][k]
        R = lvl[ls + 1] - lvl[ls]
        assert cuts[0] == 0 and cuts[-1] == R and all(a <= c for a, c in zip(cuts, cuts[1:]))
        assert all(a < c for a, c in zip(plan["cuts"][0], plan["cuts"][0][1:]))  # player 1: no empty rank
        assert lvl[ls] <= 4096
        rj, rs = _roots(p, lvl, ls)
        # every DP below the split hangs in a subtree; each level's DPs of a rank are contiguous
        assert (rj[lvl[ls]:] >= 0).all() and (rj[:lvl[ls]] == -1).all()
        for l in range(ls, len(lvl) - 1):
            own = _owner(cuts, rj[lvl[l]:lvl[l + 1]])
            assert (np.diff(own) >= 0).all()
        # the subtree sequences per rank the planner reports
        owners = _owner(cuts, rs[rs >= 0])
        assert np.bincount(owners, minlength=world).tolist() == plan["seqs"][k]
        rs_all.append(rs)
    # payoff closure: a forest row of rank r reads forest columns of rank r
    # only; trunk rows read trunk columns only
    U = b.payoff
    rows = np.repeat(np.arange(U.rows), np.diff(U.indptr))
    r1, r2 = rs_all[0][rows], rs_all[1][np.asarray(U.indices)]
    assert ((r1 >= 0) == (r2 >= 0)).all()
    f = r1 >= 0
    assert (_owner(plan["cuts"][0], r1[f]) == _owner(plan["cuts"][1], r2[f])).all()


@pytest.mark.parametrize("game,why", [("leduc", "couples a trunk sequence"), ("kuhn", "no subtree split"),
                                      ("liars3", "not ordered by subtree root")])
def test_plan_rejects_unsplittable_games(game, why):
    from paper_2605_14277_b200.distributed import subtree_plan
    with pytest.raises(ValueError, match=why):
        subtree_plan(bundle(game), 2)


def test_plan_rejects_more_ranks_than_blocks():
    from paper_2605_14277_b200.distributed import subtree_plan
    with pytest.raises(ValueError, match="closed blocks"):
        subtree_plan(bundle("goof3"), 64)


# ------------------------------------------------------- gloo world-2 schedule

WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rows(m, x, rows, neg):
    out = np.zeros(m.rows)
    for i in rows:
        acc = 0.0
        for k in range(m.indptr[i], m.indptr[i + 1]):
            acc += float(m.data[k]) * float(x[m.indices[k]])
        out[i] = -1.0 * acc if neg else acc
    return out


def _values(p, b, u, V, dps):
    """Bottom-up expected values of the DPs `dps` (descending): V[j] =
    sum_a b[s] (u[s] + sum of s's child DPs' V), fixed summation order."""
    sp = np.append(np.asarray(p.dp_first_seq), p.num_seqs)
    par = np.asarray(p.dp_parent_seq)
    kids = {}
    for q in range(p.num_decisions):
        kids.setdefault(int(par[q]), []).append(q)
    for j in dps:
        acc = 0.0
        for s in range(sp[j], sp[j + 1]):
            v = float(u[s])
            for c in kids.get(s, ()):
                v += float(V[c])
            acc += float(b[s]) * v
        V[j] = acc
    return V


def _worker(rank, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from oracle.oracle import OracleSolver
        from paper_2605_14277_b200.distributed import subtree_plan
        b = bundle("goof4")
        plan = subtree_plan(b, WORLD)
        o = OracleSolver(b, "cfr+")
        o.step(3)
        xs = [np.asarray(o.current(1), dtype=float), np.asarray(o.current(2), dtype=float)]
        info = []
        for k, p in enumerate(b.procs):
            lvl = _levels(p)
            rj, rs = _roots(p, lvl, plan["ls"][k])
            info.append((lvl, plan["ls"][k], rj, rs, _owner(plan["cuts"][k], np.maximum(rj, 0)),
                         _owner(plan["cuts"][k], np.maximum(rs, 0))))
        res = {}
        full = {}
        for k, p in enumerate(b.procs):
            lvl, ls, rj, rs, own_j, own_s = info[k]
            o_lvl, o_ls, o_rj, o_rs, o_own_j, o_own_s = info[1 - k]
            m = b.payoff if k == 0 else b.payoff_t
            # the opponent's strategy with every other rank's subtrees poisoned
            x = xs[1 - k].copy()
            x[(o_rs >= 0) & (o_own_s != rank)] = np.nan
            mine = np.flatnonzero((rs < 0) | (own_s == rank))
            u = _rows(m, x, mine, neg=k == 1)
            uf = _rows(m, xs[1 - k], range(m.rows), neg=k == 1)
            bb = xs[k]  # any behaviour-like vector: the current strategy
            V = np.full(p.num_decisions, np.nan)
            forest = [j for j in range(p.num_decisions - 1, lvl[ls] - 1, -1) if own_j[j] == rank]
            _values(p, bb, u, V, forest)
            # exchange the subtree roots' values (each rank's own slice)
            j0, j1 = lvl[ls], lvl[ls + 1]
            roots = torch.tensor(np.where(own_j[j0:j1] == rank, V[j0:j1], 0.0))
            got = [torch.zeros_like(roots) for _ in range(WORLD)]
            dist.all_gather(got, roots)
            for r in range(WORLD):
                sel = own_j[j0:j1] == r
                V[j0:j1][sel] = got[r].numpy()[sel]
            _values(p, bb, u, V, range(lvl[ls] - 1, -1, -1))  # the trunk
            Vf = _values(p, bb, uf, np.zeros(p.num_decisions), range(p.num_decisions - 1, -1, -1))
            res[k] = (u[mine], V[: lvl[ls]], V[forest])
            full[k] = (uf[mine], Vf[: lvl[ls]], Vf[forest])
        ok = all(np.array_equal(res[k][i], full[k][i]) for k in range(2) for i in range(3))
        finite = all(np.isfinite(res[k][i]).all() for k in range(2) for i in range(3))
        out = [None] * WORLD
        dist.all_gather_object(out, (ok, finite, len(res[0][2]) + len(res[1][2])))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_subtree_schedule_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [o[:2] for o in out] == [(True, True)] * WORLD
    b = bundle("goof4")
    assert sum(o[2] for o in out) == sum(p.num_decisions - _levels(p)[2] for p in b.procs)


# ---------------------------------------------------------------------- GPU

GOOF = [k for k in sorted(golden_meta()["lockstep"]) if k.startswith("goof")]


def _check(s, rec, key):
    from test_gpu_parity import _state
    for k, v in _state(s).items():
        assert digest(v) == rec["digests"][k], (key, k)
    e, br = s.exploitability("average")
    assert e == rec["expl"] and list(br) == rec["br_avg"]


@pytest.mark.gpu
@pytest.mark.parametrize("key", GOOF)
def test_subtree_world1_nccl_bit_exact(gpu, key):
    """scfr_create_subtree over a real 1-rank NCCL communicator (root-value
    broadcasts in the graph, gathers before the reads)."""
    from paper_2605_14277_b200 import Solver
    from paper_2605_14277_b200.distributed import nccl_unique_id
    from test_gpu_parity import _cfg
    rec = golden_meta()["lockstep"][key]
    s = Solver(bundle(rec["game"]), _cfg(rec), device=gpu, engine="levels", subtree=True,
               shard=(nccl_unique_id(), 0, 1))
    s.step(rec["iters"])
    _check(s, rec, key)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("key", ["goof3.pcfr+.alt.60", "goof3.dcfr.sim.60", "goof4.cfr.sim.10",
                                 "goof4.pcfr+.alt.10"])
def test_subtree_simulated_ranks_bit_exact(gpu, key, world, monkeypatch):
    """Every forest level launched as `world` range-restricted launches (one
    per rank of a world-rank plan; trunk once): the kernels' DP ranges, the
    top recompute on a partial range and the fused leaf rows per range."""
    from paper_2605_14277_b200 import Solver
    from paper_2605_14277_b200.distributed import nccl_unique_id
    from test_gpu_parity import _cfg
    monkeypatch.setenv("SCFR_SUBTREE_SIM", str(world))
    rec = golden_meta()["lockstep"][key]
    s = Solver(bundle(rec["game"]), _cfg(rec), device=gpu, engine="levels", subtree=True,
               shard=(nccl_unique_id(), 0, 1))
    s.step(rec["iters"])
    _check(s, rec, key)
