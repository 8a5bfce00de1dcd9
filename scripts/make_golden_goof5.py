#!/usr/bin/env python
"""Goofspiel-5 golden fixtures produced by the REFERENCE seqcfr package.

This is the bench configuration (BASELINE.json configs[3]); round 1 pinned it
only through sizes and the oracle.  Run in the build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src:. \
        python scripts/make_golden_goof5.py [--target T]

Everything recorded comes from reference code paths:
  * tree                — the Appendix-A generator driven through the
                          reference GameBuilder (pkg/games.py:106-135)
  * structure digests   — GameBundle (pkg/solvers.py:314-323):
                          DecisionProcess (pkg/decision_process.py:76-242),
                          build_payoff_matrix + transposed (pkg/operators.py:164-180)
  * lockstep digests    — _step + RegretState (pkg/solvers.py:97-140,351-372),
                          PCFR+ alt at iterations 1, 2, 10, 30, 50 and CFR sim @10
  * exploitability      — metrics.best_response_values (pkg/metrics.py:59-75)
  * --target T          — run(iterations=T, checkpoints=[T-1, T])
                          (pkg/solvers.py:375-438): the first iteration at
                          which exploitability <= 1e-4, as found on the GPU,
                          checked against the reference itself.

The reference's parallel backend is bitwise identical to its serial one
(pkg/kernels.py:3-8), so it is used for speed.  Output:
tests/golden/goof5_meta.json (digests only: small enough to commit).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from seqcfr import games as G  # noqa: E402
from seqcfr import kernels, metrics, solvers  # noqa: E402
from seqcfr.solvers import RegretState, SolverConfig, _step  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden", "goof5_meta.json")
sys.path.insert(0, ROOT)
import paper_2605_14277_b200.games as MG  # noqa: E402  (generator body only)

PROC_FIELDS = ("kind", "depth", "parent", "node_seq", "seq_node", "dp_node",
               "dp_first_seq", "dp_num_actions", "dp_parent_seq",
               "level_starts", "game_seq")


def digest(a) -> str:
    a = np.asarray(a)
    a = a.astype("<i8") if a.dtype.kind in "iub" else a.astype("<f8")
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def reference_goofspiel(cards: int):
    """The Appendix-A generator body, with every node created by the
    reference's own GameBuilder."""
    saved = MG.GameBuilder
    MG.GameBuilder = G.GameBuilder
    try:
        return MG.goofspiel(cards)
    finally:
        MG.GameBuilder = saved


def load() -> dict:
    if os.path.exists(OUT):
        with open(OUT) as fh:
            return json.load(fh)
    return {"generator": "scripts/make_golden_goof5.py (reference seqcfr at "
                         "/root/reference/pkg/src)", "structure": {}, "lockstep": {},
            "target": {}}


def save(meta):
    with open(OUT, "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


def state_digests(s1, s2, x1, x2, p1, p2):
    return {"avg1": digest(s1.average_strategy()), "avg2": digest(s2.average_strategy()),
            "x1": digest(x1), "x2": digest(x2), "r1": digest(s1.regrets),
            "r2": digest(s2.regrets), "acc1": digest(s1.avg_accum),
            "acc2": digest(s2.avg_accum), "u1": digest(p1), "u2": digest(p2),
            "b1": digest(s1.behavior), "b2": digest(s2.behavior)}


def lockstep(bundle, be, variant, mode, marks, expl_at, meta):
    cfg = SolverConfig(variant=variant, mode=mode)
    s1 = RegretState(bundle.ops[0], cfg.gamma)
    s2 = RegretState(bundle.ops[1], cfg.gamma)
    p1 = p2 = x1 = x2 = None
    t0 = time.time()
    for it in range(1, max(marks) + 1):
        x1, x2, p1, p2 = _step(bundle, cfg, be, s1, s2, p1, p2)
        if it in marks:
            rec = {"variant": variant, "mode": cfg.mode, "gamma": cfg.gamma, "iters": it,
                   "avg_weight": [s1.avg_weight, s2.avg_weight],
                   "digests": state_digests(s1, s2, x1, x2, p1, p2)}
            if it in expl_at:
                avg1, avg2 = s1.average_strategy(), s2.average_strategy()
                br = metrics.best_response_values(bundle, avg1, avg2, be)
                brc = metrics.best_response_values(bundle, x1, x2, be)
                rec.update({"br_avg": list(br), "expl": (br[0] + br[1]) / 2.0,
                            "br_cur": list(brc), "expl_current": (brc[0] + brc[1]) / 2.0,
                            "value": metrics.expected_value(bundle.payoff, avg1, avg2, be)})
            meta["lockstep"][f"goof5.{variant}.{cfg.mode}.{it}"] = rec
            save(meta)
            print(f"{variant} {cfg.mode} @{it}: {time.time() - t0:.1f}s "
                  f"{rec.get('expl', '')}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--target", type=int, default=0,
                    help="check first-<=1e-4 iteration T of PCFR+ alt against the reference")
    ap.add_argument("--skip-lockstep", action="store_true")
    args = ap.parse_args()
    meta = load()
    be = kernels.parallel_backend(os.cpu_count() or 1)

    t0 = time.time()
    game = reference_goofspiel(5)
    print(f"generate: {time.time() - t0:.1f}s nodes={game.num_nodes}", flush=True)
    t0 = time.time()
    bundle = solvers.GameBundle(game)
    print(f"bundle: {time.time() - t0:.1f}s", flush=True)

    info = {"num_game_nodes": game.num_nodes, "bundle_nbytes": bundle.nbytes()}
    for pl in (1, 2):
        proc = bundle.procs[pl - 1]
        info[f"p{pl}"] = {"num_nodes": proc.num_nodes, "num_decisions": proc.num_decisions,
                          "num_seqs": proc.num_seqs, "height": proc.height,
                          "degree": proc.degree,
                          "digests": {f: digest(getattr(proc, f)) for f in PROC_FIELDS}}
    for tag, m in (("U", bundle.payoff), ("UT", bundle.payoff_t)):
        info[tag] = {"rows": m.rows, "cols": m.cols, "nnz": m.nnz,
                     "digests": {"indptr": digest(m.indptr), "indices": digest(m.indices),
                                 "data": digest(m.data)}}
    meta["structure"]["goof5"] = info
    save(meta)
    print("structure digests written", flush=True)

    if not args.skip_lockstep:
        lockstep(bundle, be, "pcfr+", "alt", {1, 2, 10, 30, 50}, {30, 50}, meta)
        lockstep(bundle, be, "cfr", "sim", {10}, {10}, meta)

    if args.target:
        T = args.target
        t0 = time.time()
        res = solvers.run(bundle, SolverConfig(variant="pcfr+"), iterations=T,
                          checkpoints=[T - 1, T], backend=be)
        meta["target"][f"goof5.pcfr+.alt.{T}"] = {
            "iters": T, "threshold": 1e-4,
            "records": [{"iteration": r.iteration, "exploitability": r.exploitability,
                         "current_exploitability": r.current_exploitability,
                         "work": r.work} for r in res.records],
            "digests": {"avg1": digest(res.average[0]), "avg2": digest(res.average[1])}}
        save(meta)
        print(f"target run {T}: {time.time() - t0:.1f}s "
              f"{[r.exploitability for r in res.records]}", flush=True)


if __name__ == "__main__":
    main()
