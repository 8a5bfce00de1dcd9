"""A/B of SMEM-engine switches on Kuhn / Leduc: us/iter per configuration,
alternating over 3 rounds in one process (switches are read at creation).

usage: python scripts/micro/small_ab.py "" "SCFR_SMALL_OOL=1" "SCFR_SMALL_OOL=1,SCFR_SMALL_MAXA=3"
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, kuhn_poker, leduc_poker  # noqa: E402

configs = sys.argv[1:] or [""]
games = {"kuhn": GameBundle(kuhn_poker()), "leduc": GameBundle(leduc_poker())}
cases = (("kuhn", "cfr", "sim"), ("leduc", "cfr+", "alt"), ("leduc", "pcfr+", "alt"), ("leduc", "dcfr", "alt"))
keys = {kv.split("=")[0] for c in configs for kv in c.split(",") if kv}
res = {(c, k): [] for c in configs for k in cases}
for rnd in range(3):
    for case in cases:
        name, variant, mode = case
        for c in configs:
            for k in keys:
                os.environ.pop(k, None)
            for kv in filter(None, c.split(",")):
                k, v = kv.split("=", 1)
                os.environ[k] = v
            s = Solver(games[name], SolverConfig(variant, mode=mode))
            s.step(200)
            s.synchronize()
            s.step(2000)
            s.synchronize()
            res[(c, case)].append(s.last_step_ms() * 1e3 / 2000)
            s.close()
for case in cases:
    print(" ".join(case), " | ".join(f"{c or 'default'}: {statistics.median(res[(c, case)]):.2f}" for c in configs))
