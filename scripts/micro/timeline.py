"""In-graph per-launch timeline of one iteration (scfr_timeline):
python scripts/micro/timeline.py [goof5|goof4|liars6] [n] [variant]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, flat_goofspiel, flat_liars_dice  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "goof5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
variant = sys.argv[3] if len(sys.argv) > 3 else ("dcfr" if name.startswith("liars") else "pcfr+")
game = flat_liars_dice(int(name[-1])) if name.startswith("liars") else flat_goofspiel(int(name[-1]))
s = Solver(GameBundle(game), SolverConfig(variant), engine="levels")
s.step(5)
s.synchronize()
tl = s.timeline(n)
s.step(20)
s.synchronize()
end = max(e["end_us"] for e in tl)
print(f"graph step {s.last_step_ms() / 20 * 1e3:.1f} us; timeline end {end:.1f} us; launches {len(tl)}")
for k, e in enumerate(tl):
    gbs = e["bytes"] / (e["own_us"] * 1e3) if e["own_us"] > 0 else 0
    print(f"{k:3d} s{e['stream']} {e['kind']:>8} start {e['start_us']:7.1f} end {e['end_us']:7.1f} "
          f"own {e['own_us']:6.1f} excl {e['excl_us']:6.1f} us {e['bytes'] / 1e6:7.2f} MB {gbs:7.1f} GB/s")
