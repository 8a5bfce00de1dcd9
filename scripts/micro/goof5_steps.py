"""Goofspiel-5 PCFR+ alternating: create, then N iterations (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, flat_goofspiel  # noqa: E402

s = Solver(GameBundle(flat_goofspiel(5)), SolverConfig("pcfr+", mode="alt"))
s.step(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
s.synchronize()
print("ok")
