"""Multi-GPU plumbing (one process per GPU, torch.distributed for control).

Three modes:

* Row-sharded payoff SpMV for one big solve (BASELINE config 4):
  ``sharded_solver(bundle, config)``.  Every rank keeps the full
  decision-process state; rank k owns rows ``shard_rows(R, world, k)`` of U
  and of Uᵀ, computes its slice of u1 = U x2 and u2 = -Uᵀ x1 with the same
  row-sequential sums as one GPU, and the slices are all-gathered in place by
  NCCL inside the iteration (C-ABI ``scfr_create_sharded``) — no reduction
  collective, so iterates are bit-identical to one GPU.  torch.distributed
  only broadcasts the 128-byte NCCL unique id.
* Subtree-sharded tree passes for one big solve: ``subtree_solver(bundle,
  config)``.  Every rank computes the small trunk of each player; below each
  player's split level rank k owns a contiguous range of whole subtrees
  (``subtree_plan``), chosen so its payoff rows read only its own subtrees'
  strategies.  Launches cover only the rank's decision points; the subtree
  roots' values are exchanged (NCCL, in the graph) after each bottom-up
  launch of a split level, so iterates are bit-identical to one GPU.
* Independent solves (BASELINE config 5): ``sweep_slice(params, world, k)``
  gives rank k a contiguous slice of the (alpha, beta, gamma) grid, solved as
  one batched handle per GPU; no collective on the data path.
"""

from __future__ import annotations

import ctypes as C
import os

from . import native as N
from .compiler import GameBundle
from .solvers import Solver, SolverConfig


def shard_rows(rows: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [r0, r1) of a `rows`-row matrix owned by `rank`: equal chunks of
    ceil(rows/world) (the last rank may hold fewer, possibly none); the
    gathered vector is world*chunk long, padded at the end.  Mirrors
    upload_csr in csrc/solver.cu."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    chunk = (rows + world - 1) // world
    r0 = min(rows, chunk * rank)
    return r0, min(rows, r0 + chunk)


def sweep_slice(params, world: int, rank: int):
    """Contiguous, near-equal slice of a parameter grid for one rank."""
    n = len(params)
    lo = n * rank // world
    hi = n * (rank + 1) // world
    return list(params[lo:hi]), lo


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    N.check(N.lib().scfr_nccl_unique_id(buf))
    return buf.raw


def broadcast_unique_id(group=None) -> bytes:
    """Rank 0 creates the NCCL id; every rank returns it (torch.distributed
    must be initialised; any backend)."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def sharded_solver(bundle: GameBundle, config: SolverConfig, device: int | None = None,
                   group=None) -> Solver:
    """A Solver whose payoff SpMV is row-sharded over the torch.distributed
    group (one rank per GPU).  All ranks must step / query it together."""
    import torch.distributed as dist
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    uid = broadcast_unique_id(group)
    return Solver(bundle, config, device=device, engine="levels",
                  shard=(uid, dist.get_rank(group), dist.get_world_size(group)))


def subtree_plan(bundle: GameBundle, world: int) -> dict:
    """The subtree partition (C-ABI scfr_subtree_plan; host only, no GPU):
    ``ls`` = each player's split level (merged-level index), ``cuts[k]`` =
    the world+1 root boundaries of player k+1 (rank r owns level-ls roots
    [cuts[k][r], cuts[k][r+1])), ``seqs[k]`` = subtree sequences per rank.
    Raises ValueError (SCFR_EINVAL) for games the subtree mode cannot split."""
    import numpy as np
    if world < 1:
        raise ValueError("bad world size")
    p1, p2, U, _ = bundle._c
    ls = (C.c_int32 * 2)()
    cuts = np.zeros(2 * (world + 1), dtype=np.int64)
    seqs = np.zeros(2 * world, dtype=np.int64)
    N.check(N.lib().scfr_subtree_plan(C.byref(p1), C.byref(p2), C.byref(U), int(world), ls,
                                      N.ptr(cuts, C.c_int64), N.ptr(seqs, C.c_int64)))
    return {"ls": (int(ls[0]), int(ls[1])),
            "cuts": (cuts[:world + 1].tolist(), cuts[world + 1:].tolist()),
            "seqs": (seqs[:world].tolist(), seqs[world:].tolist())}


def subtree_solver(bundle: GameBundle, config: SolverConfig, device: int | None = None,
                   group=None) -> Solver:
    """A Solver whose tree passes are subtree-sharded over the torch.distributed
    group (C-ABI scfr_create_subtree): each rank computes the trunk and its own
    subtrees, exchanging the subtree roots' values over NCCL.  All ranks must
    step / query it together."""
    import torch.distributed as dist
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    uid = broadcast_unique_id(group)
    return Solver(bundle, config, device=device, engine="levels", subtree=True,
                  shard=(uid, dist.get_rank(group), dist.get_world_size(group)))
