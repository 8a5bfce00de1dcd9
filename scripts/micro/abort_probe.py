import faulthandler, sys
faulthandler.enable()
sys.path.insert(0, '.')
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, kuhn_poker
b = GameBundle(kuhn_poker())
s = Solver(b, SolverConfig("cfr"), device=0)
s.step(10)
print("ok", s.engine, s.exploitability()[0])
