"""A level-engine switch on vs off on one GPU: same iterates bit for bit
(regrets, behaviour, accumulators, utilities, average and current strategies)
across games, variants, modes, batches and dtypes; prints launches per
iteration.  The switch is an environment variable read at creation:
SCFR_NO_TOP (default), SCFR_NO_LEAF_FUSE, SCFR_NO_PIPE, SCFR_NO_GROUP,
SCFR_PAIR, ... (SCFR_NO_* switches off the optimisation, other names on).

    python scripts/mode_check.py [--quick] [--env SCFR_NO_TOP|SCFR_NO_LEAF_FUSE|...]
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, flat_goofspiel  # noqa: E402
from paper_2605_14277_b200 import games as G  # noqa: E402


ENV = "SCFR_NO_TOP"


def run(b, cfg, n, on, batch=None, dtype="f64"):
    # on: the optimised path (SCFR_NO_X=0 / SCFR_X=1)
    os.environ[ENV] = ("0" if on else "1") if ENV.startswith("SCFR_NO") else ("1" if on else "0")
    s = Solver(b, cfg, engine="levels", batch_params=batch, dtype=dtype)
    s.step(n)
    s.synchronize()
    per_iter = s.launch_count() / n
    out = {}
    for k in range(len(batch) if batch else 1):
        for pl in (1, 2):
            for w in ("regrets", "behavior", "accum", "utility"):
                out[(k, pl, w)] = s.state(pl, w, k)
            out[(k, pl, "average")] = s.average(pl, k)
            out[(k, pl, "current")] = s.current(pl, k)
    s.close()
    return out, per_iter


def main():
    global ENV
    quick = "--quick" in sys.argv
    if "--env" in sys.argv:
        ENV = sys.argv[sys.argv.index("--env") + 1]
    games = [("goof3", lambda: G.goofspiel(3)), ("goof4", lambda: flat_goofspiel(4)),
             ("random7", lambda: G.random_game(7, 3, 0.3, 7)), ("liars3", lambda: G.liars_dice(3))]
    for depth, br, merge, seed in [(6, 3, 0.0, 3), (8, 2, 0.2, 5), (5, 4, 0.5, 11), (9, 2, 0.0, 2)]:
        games.append((f"rand{depth}_{br}_{merge}_{seed}",
                       lambda d=depth, b=br, m=merge, s=seed: G.random_game(d, b, m, s)))
    if not quick:
        games.append(("goof5", lambda: flat_goofspiel(5)))
    fails = 0
    for name, mk in games:
        b = GameBundle(mk())
        n = 3 if name == "goof5" else 9
        for variant in ("cfr", "cfr+", "dcfr", "pcfr", "pcfr+"):
            for mode in ("alt", "sim"):
                if name == "goof5" and (variant, mode) not in (("pcfr+", "alt"), ("cfr", "sim")):
                    continue
                cfg = SolverConfig(variant, mode=mode)
                for batch in (None, [(1.5, 0.0, 2.0), (1.0, 0.5, 1.0), (2.0, -0.5, 0.0)]):
                    if batch and name == "goof5":
                        continue
                    for dtype in ("f64", "f32"):
                        if dtype == "f32" and batch:
                            continue
                        t0 = time.time()
                        a, la = run(b, cfg, n, True, batch, dtype)
                        z, lz = run(b, cfg, n, False, batch, dtype)
                        bad = [k for k in a if not np.array_equal(a[k], z[k])]
                        tag = f"{name:>22} {variant:>5} {mode} B={len(batch) if batch else 1} {dtype}"
                        if bad:
                            fails += 1
                            k = bad[0]
                            d = np.flatnonzero(a[k] != z[k])
                            print(f"FAIL {tag}: {len(bad)} arrays differ, first {k} at {d[:5]} "
                                  f"({a[k][d[0]]!r} vs {z[k][d[0]]!r}); launches {la} vs {lz}", flush=True)
                        else:
                            print(f"ok   {tag}: launches/iter on {la:.0f} off {lz:.0f} "
                                  f"({time.time() - t0:.1f}s)", flush=True)
    print("FAILURES", fails)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
