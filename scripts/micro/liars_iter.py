"""A few eager Liar's dice DCFR alt iterations (level engine) for ncu."""
import sys
sys.path.insert(0, ".")
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, flat_liars_dice
s = Solver(GameBundle(flat_liars_dice(6)), SolverConfig("dcfr", gamma=2.0), engine="levels")
s.step(10)
s.synchronize()
