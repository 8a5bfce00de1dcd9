#!/usr/bin/env python
"""Generate tests/golden/ fixtures by running the REFERENCE seqcfr package.

Run in the build container (the reference exists only here):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src:. \
        python scripts/make_golden.py

Everything written is produced by reference code paths:
  * game text digests        — seqcfr.games.save_game          (pkg/games.py:558)
  * structure arrays         — DecisionProcess / build_payoff_matrix
                               (pkg/decision_process.py:76-242, pkg/operators.py:164-180)
  * lockstep iterates        — seqcfr.solvers._step + RegretState (pkg/solvers.py:351-372)
  * checkpoint records       — seqcfr.solvers.run                (pkg/solvers.py:375-438)
  * exploitability / BR      — seqcfr.metrics                    (pkg/metrics.py:59-75)

Small games keep full arrays (bit-exact comparison); large ones keep SHA-256
digests of the little-endian bytes plus scalar summaries.  The fixtures are
consumed by tests/ both here (CPU: oracle + compiler) and on the GPU box
(CUDA path), where /root/reference does not exist.
"""

from __future__ import annotations

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
from seqcfr import metrics, solvers  # noqa: E402
from seqcfr.solvers import RegretState, SolverConfig, _step  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")
sys.path.insert(0, os.path.dirname(HERE))
import paper_2605_14277_b200.games as MG  # noqa: E402  (only for liars/goofspiel trees)


def digest(a) -> str:
    a = np.asarray(a)
    if a.dtype.kind in "iub":
        a = a.astype("<i8")
    else:
        a = a.astype("<f8")
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def to_ref_game(game):
    """Our generators emit identical text; reload it as a reference Game."""
    return G.load_game(MG.save_game(game))


GAMES = {
    "kuhn": (lambda: G.kuhn_poker(), True),
    "leduc": (lambda: G.leduc_poker(), True),
    "mp": (lambda: G.matching_pennies(), True),
    "rps": (lambda: G.rock_paper_scissors(), True),
    "random6": (lambda: G.random_game(6, 3, 0.5, 1), True),
    "random7": (lambda: G.random_game(7, 3, 0.3, 7), True),
    "liars3": (lambda: to_ref_game(MG.liars_dice(3)), True),
    "goof3": (lambda: to_ref_game(MG.goofspiel(3)), True),
    "liars6": (lambda: to_ref_game(MG.liars_dice(6)), False),
    "goof4": (lambda: to_ref_game(MG.goofspiel(4)), False),
}

PROC_FIELDS = ("kind", "depth", "parent", "node_seq", "seq_node", "dp_node",
               "dp_first_seq", "dp_num_actions", "dp_parent_seq",
               "level_starts", "game_seq")


def structure(name, game, full, arrays, meta):
    bundle = solvers.GameBundle(game)
    info = {"game_text_sha256": hashlib.sha256(G.save_game(game).encode()).hexdigest(),
            "num_game_nodes": game.num_nodes}
    for pl in (1, 2):
        proc = bundle.procs[pl - 1]
        info[f"p{pl}"] = {"num_nodes": proc.num_nodes, "num_decisions": proc.num_decisions,
                          "num_seqs": proc.num_seqs, "height": proc.height,
                          "degree": proc.degree,
                          "digests": {f: digest(getattr(proc, f)) for f in PROC_FIELDS}}
        if full:
            for f in PROC_FIELDS:
                arrays[f"{name}.p{pl}.{f}"] = np.asarray(getattr(proc, f))
    for tag, m in (("U", bundle.payoff), ("UT", bundle.payoff_t)):
        info[tag] = {"rows": m.rows, "cols": m.cols, "nnz": m.nnz,
                     "digests": {"indptr": digest(m.indptr), "indices": digest(m.indices),
                                 "data": digest(m.data)}}
        if full:
            arrays[f"{name}.{tag}.indptr"] = m.indptr
            arrays[f"{name}.{tag}.indices"] = m.indices
            arrays[f"{name}.{tag}.data"] = m.data
    info["bundle_nbytes"] = bundle.nbytes()
    meta["structure"][name] = info
    return bundle


def lockstep(name, bundle, variant, mode, iters, full, arrays, meta, alpha=1.5, beta=0.0,
             gamma=None):
    """Drive reference _step exactly like run() and keep the state."""
    cfg = SolverConfig(variant=variant, mode=mode, alpha=alpha, beta=beta, gamma=gamma)
    be = solvers.serial_backend()
    s1 = RegretState(bundle.ops[0], cfg.gamma)
    s2 = RegretState(bundle.ops[1], cfg.gamma)
    p1 = p2 = None
    x1 = x2 = None
    for _ in range(iters):
        x1, x2, p1, p2 = _step(bundle, cfg, be, s1, s2, p1, p2)
    avg1, avg2 = s1.average_strategy(), s2.average_strategy()
    br_avg = metrics.best_response_values(bundle, avg1, avg2)
    br_cur = metrics.best_response_values(bundle, x1, x2)
    key = f"{name}.{variant}.{cfg.mode}.{iters}"
    if alpha != 1.5 or beta != 0.0 or gamma is not None:
        key += f".a{alpha}.b{beta}.g{cfg.gamma}"
    rec = {"game": name, "variant": variant, "mode": cfg.mode, "iters": iters,
           "alpha": alpha, "beta": beta, "gamma": cfg.gamma,
           "expl": (br_avg[0] + br_avg[1]) / 2.0, "br_avg": list(br_avg),
           "expl_current": (br_cur[0] + br_cur[1]) / 2.0, "br_cur": list(br_cur),
           "avg_weight": [s1.avg_weight, s2.avg_weight],
           "work_per_iter": be.work // iters,
           "value": metrics.expected_value(bundle.payoff, avg1, avg2),
           "digests": {"avg1": digest(avg1), "avg2": digest(avg2), "x1": digest(x1),
                       "x2": digest(x2), "r1": digest(s1.regrets), "r2": digest(s2.regrets),
                       "acc1": digest(s1.avg_accum), "acc2": digest(s2.avg_accum),
                       "u1": digest(p1), "u2": digest(p2)}}
    if full:
        for tag, arr in (("avg1", avg1), ("avg2", avg2), ("x1", x1), ("x2", x2),
                         ("r1", s1.regrets), ("r2", s2.regrets), ("u1", p1), ("u2", p2)):
            arrays[f"{key}.{tag}"] = np.asarray(arr)
    meta["lockstep"][key] = rec
    return rec


def main():
    os.makedirs(OUT, exist_ok=True)
    arrays: dict[str, np.ndarray] = {}
    meta = {"generator": "scripts/make_golden.py (reference seqcfr at /root/reference/pkg/src)",
            "structure": {}, "lockstep": {}, "runs": {}, "br": {}}
    bundles = {}
    for name, (make, full) in GAMES.items():
        t0 = time.time()
        game = make()
        bundles[name] = structure(name, game, full, arrays, meta)
        print(f"structure {name}: {time.time() - t0:.1f}s", flush=True)

    # Lockstep: every variant x mode (SPEC.md:554's acceptance matrix) on the
    # small games; full arrays.
    for name, iters in (("kuhn", 200), ("random6", 200), ("leduc", 100), ("mp", 50),
                        ("rps", 50), ("liars3", 60), ("goof3", 60), ("random7", 40)):
        for variant in solvers.VARIANTS:
            for mode in ("sim", "alt"):
                lockstep(name, bundles[name], variant, mode, iters,
                         GAMES[name][1], arrays, meta)
        print(f"lockstep {name} done", flush=True)
    # Variant defaults at 1000 iterations on Kuhn (SURVEY.md §8(c) known answers).
    for variant in solvers.VARIANTS:
        lockstep("kuhn", bundles["kuhn"], variant, None, 1000, True, arrays, meta)
    # DCFR parameter grid points on Leduc (config 5's batched sweep cases).
    for (a, b, g) in ((0.5, -1.0, 0.0), (1.0, -0.5, 1.0), (1.5, 0.0, 2.0), (2.0, 0.5, 3.0),
                      (3.0, 0.0, 1.0), (5.0, -1.0, 2.0), (4.0, 0.5, 0.0), (1.5, -0.5, 3.0)):
        lockstep("leduc", bundles["leduc"], "dcfr", "alt", 200, True, arrays, meta,
                 alpha=a, beta=b, gamma=g)
    # Larger games: digests only.
    lockstep("liars6", bundles["liars6"], "dcfr", "alt", 30, False, arrays, meta, gamma=2.0)
    lockstep("goof4", bundles["goof4"], "pcfr+", "alt", 10, False, arrays, meta)
    lockstep("goof4", bundles["goof4"], "cfr", "sim", 10, False, arrays, meta)
    print("lockstep large done", flush=True)

    # Checkpointed runs through the public run() (records / CSV schema).
    for name, variant, iters, cps in (("kuhn", "cfr", 1000, [1, 10, 100, 1000]),
                                       ("kuhn", "cfr+", 300, [1, 2, 50, 300]),
                                       ("leduc", "cfr+", 1592, [1, 100, 1000, 1591, 1592]),
                                       ("leduc", "dcfr", 1000, [1000]),
                                       ("liars6", "dcfr", 940, [300, 930, 940]),
                                       ("random6", "pcfr+", 120, [1, 60, 120])):
        t0 = time.time()
        res = solvers.run(bundles[name], SolverConfig(variant=variant), iterations=iters,
                          checkpoints=cps)
        meta["runs"][f"{name}.{variant}.{iters}"] = {
            "game": name, "variant": variant, "iters": iters, "checkpoints": cps,
            "records": [{"iteration": r.iteration, "exploitability": r.exploitability,
                         "current_exploitability": r.current_exploitability,
                         "work": r.work, "peak_bytes": r.peak_bytes} for r in res.records],
            "digests": {"avg1": digest(res.average[0]), "avg2": digest(res.average[1])},
            "value": metrics.expected_value(res.bundle.payoff, *res.average)}
        print(f"run {name} {variant} {iters}: {time.time() - t0:.1f}s "
              f"expl={res.records[-1].exploitability:.6e}", flush=True)

    # Best response on fixed profiles (uniform and a seeded random polytope point).
    from seqcfr.solvers import uniform_sequence_strategy
    for name in ("kuhn", "leduc", "random6", "liars3", "goof3"):
        b = bundles[name]
        be = solvers.serial_backend()
        x1 = uniform_sequence_strategy(b.ops[0], be)
        x2 = uniform_sequence_strategy(b.ops[1], be)
        br = metrics.best_response_values(b, x1, x2)
        meta["br"][name] = {"uniform": list(br), "expl": (br[0] + br[1]) / 2.0}
        arrays[f"{name}.uniform.x1"] = x1
        arrays[f"{name}.uniform.x2"] = x2

    np.savez_compressed(os.path.join(OUT, "reference_arrays.npz"), **arrays)
    with open(os.path.join(OUT, "reference_meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
