"""A/B of level-engine switches on Goofspiel-5 PCFR+ alternating (fp64):
us/iter of each configuration, alternating over rounds, one process.

usage: python scripts/micro/goof5_ab.py "" "SCFR_TOP_DPS=30000" "SCFR_NO_OVERLAP=1,SCFR_NO_PIPE=1"
(an empty string = the defaults; switches are read at solver creation)"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, flat_goofspiel  # noqa: E402

configs = sys.argv[1:] or [""]
b = GameBundle(flat_goofspiel(int(os.environ.get("AB_CARDS", "5"))))
cfg = SolverConfig(os.environ.get("AB_VARIANT", "pcfr+"), mode=os.environ.get("AB_MODE", "alt"))
res = {c: [] for c in configs}
keys = {k.split("=")[0] for c in configs for k in c.split(",") if k}
for rnd in range(int(os.environ.get("AB_ROUNDS", "3"))):
    for c in configs:
        for k in keys:
            os.environ.pop(k, None)
        for kv in filter(None, c.split(",")):
            k, v = kv.split("=", 1)
            os.environ[k] = v
        s = Solver(b, cfg)
        s.step(30)
        s.synchronize()
        s.step(300)
        s.synchronize()
        res[c].append(s.last_step_ms() * 1e3 / 300)
        s.close()
for c in configs:
    print(f"{c or 'default':60s} median {statistics.median(res[c]):7.2f} us/iter  {['%.2f' % v for v in res[c]]}")
