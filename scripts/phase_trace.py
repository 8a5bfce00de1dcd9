"""Per-phase cycle counts of the SMEM engine (SCFR_PHASE_TRACE=1 debug path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SCFR_PHASE_TRACE"] = "1"
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, kuhn_poker, leduc_poker  # noqa

for name, game, variant in (("kuhn", kuhn_poker(), "cfr"), ("leduc", leduc_poker(), "cfr+"), ("leduc", leduc_poker(), "pcfr+")):
    s = Solver(GameBundle(game), SolverConfig(variant), engine="persistent")
    s.step(5)
    s.synchronize()
    print(f"== {name} {variant}: 200 iterations", file=sys.stderr, flush=True)
    s.step(200)
    s.synchronize()
    print(f"   {s.last_step_ms() * 1e3 / 200:.2f} us/iter", file=sys.stderr, flush=True)
