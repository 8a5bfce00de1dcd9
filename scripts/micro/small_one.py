"""One SMEM-engine launch of Leduc CFR+ alternating (2000 iterations) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, leduc_poker  # noqa: E402

s = Solver(GameBundle(leduc_poker()), SolverConfig(sys.argv[1] if len(sys.argv) > 1 else "cfr+", mode="alt"))
s.step(2000)
s.synchronize()
print(f"{s.last_step_ms() * 1e3 / 2000:.2f} us/iter")
