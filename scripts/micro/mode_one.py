"""One level-engine solve (debug aid): python scripts/micro/mode_one.py goof3 cfr alt 1"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, flat_goofspiel
from paper_2605_14277_b200 import games as G
name, variant, mode, n = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
mk = {"goof3": lambda: G.goofspiel(3), "goof4": lambda: flat_goofspiel(4), "goof5": lambda: flat_goofspiel(5),
      "random7": lambda: G.random_game(7, 3, 0.3, 7)}[name]
s = Solver(GameBundle(mk()), SolverConfig(variant, mode=mode), engine="levels")
s.step(n)
s.synchronize()
print("ok", s.launch_count() / n, s.regrets(1)[:4])
