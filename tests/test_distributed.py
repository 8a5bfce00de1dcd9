"""Multi-process host logic of the multi-GPU modes (gloo, world size 2, CPU).

The CUDA kernels and NCCL need a GPU; here the sharding arithmetic and the
control plane are exercised exactly as the GPU path uses them:
  * the NCCL unique id is created on rank 0 and broadcast (distributed.py);
  * each rank computes its row slice (distributed.shard_rows) of u1 = U x2 and
    u2 = -Uᵀ x1 with row-sequential sums, the padded slices are all-gathered,
    and the result must equal the full product BIT FOR BIT (no reduction
    collective => sharding cannot change a single rounding);
  * the batched-sweep partition covers the grid exactly once, in order.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rows(m, x, r0, r1, neg):
    out = []
    for i in range(r0, r1):
        acc = 0.0
        for k in range(m.indptr[i], m.indptr[i + 1]):
            acc += float(m.data[k]) * float(x[m.indices[k]])
        out.append(-1.0 * acc if neg else acc)
    return out


def _worker(rank, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from oracle.oracle import OracleSolver
        from paper_2605_14277_b200 import GameBundle, leduc_poker
        from paper_2605_14277_b200.distributed import broadcast_unique_id, shard_rows, sweep_slice

        uid = broadcast_unique_id()
        ids = [None] * WORLD
        dist.all_gather_object(ids, uid)
        b = GameBundle(leduc_poker())
        # a non-trivial profile: the oracle's strategies after a few iterations
        o = OracleSolver(b, "cfr+")
        o.step(7)
        x1, x2 = o.current(1), o.current(2)
        res = {}
        for tag, m, x, neg in (("u1", b.payoff, x2, False), ("u2", b.payoff_t, x1, True)):
            r0, r1 = shard_rows(m.rows, WORLD, rank)
            chunk = (m.rows + WORLD - 1) // WORLD
            mine = _rows(m, x, r0, r1, neg) + [0.0] * (chunk - (r1 - r0))  # padded slice
            gathered = [torch.zeros(chunk, dtype=torch.float64) for _ in range(WORLD)]
            dist.all_gather(gathered, torch.tensor(mine, dtype=torch.float64))
            res[tag] = torch.cat(gathered).numpy()[:m.rows]
        grid = [(a, 0.0, g) for a in (0.5, 1.0, 1.5) for g in range(5)]
        part, lo = sweep_slice(grid, WORLD, rank)
        parts = [None] * WORLD
        dist.all_gather_object(parts, (lo, part))
        if rank == 0:
            import ctypes as C

            from oracle.oracle import _ptr
            from oracle.oracle import lib as olib
            full_u1 = np.empty(b.payoff.rows)
            xx = np.ascontiguousarray(x2)
            olib().oc_spmv(o._st, 0, _ptr(xx, C.c_double), _ptr(full_u1, C.c_double), 0)
            full_u2 = np.empty(b.payoff_t.rows)
            xx1 = np.ascontiguousarray(x1)
            olib().oc_spmv(o._st, 1, _ptr(xx1, C.c_double), _ptr(full_u2, C.c_double), 1)
            merged = [p for _, ps in sorted(parts) for p in ps]
            q.put({"ids_equal": all(i == ids[0] for i in ids) and len(ids[0]) == 128,
                   "u1": bool(np.array_equal(res["u1"], full_u1)),
                   "u2": bool(np.array_equal(res["u2"], full_u2)),
                   "sweep": merged == grid})
    finally:
        dist.destroy_process_group()


def test_sharded_spmv_and_sweep_partition_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out == {"ids_equal": True, "u1": True, "u2": True, "sweep": True}


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_rows_cover_every_row_once(world):
    from paper_2605_14277_b200.distributed import shard_rows
    for rows in (1, 2, 7, 1093, 2666026):
        spans = [shard_rows(rows, world, k) for k in range(world)]
        covered = np.zeros(rows, dtype=int)
        for r0, r1 in spans:
            covered[r0:r1] += 1
            assert r1 - r0 <= (rows + world - 1) // world
        assert (covered == 1).all()
