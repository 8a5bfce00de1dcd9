"""Readback probe: wall time of Solver.average() on Goofspiel-5 against a
bare pinned D2H of the same bytes and a first-touch fill of a fresh array."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, flat_goofspiel  # noqa: E402

b = GameBundle(flat_goofspiel(5))
s = Solver(b, SolverConfig("pcfr+"))
s.step(10)
s.synchronize()
S = b.procs[0].num_seqs
for _ in range(3):
    t0 = time.perf_counter(); a1 = s.average(1); t1 = time.perf_counter(); a2 = s.average(2); t2 = time.perf_counter()
    print(f"average(1) {1e3*(t1-t0):.3f} ms  average(2) {1e3*(t2-t1):.3f} ms", file=sys.stderr)
d = torch.empty(S, dtype=torch.float64, device="cuda")
h = torch.empty(S, dtype=torch.float64, pin_memory=True)
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); h.copy_(d); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"pinned D2H {S*8/1e6:.1f} MB {1e3*(t1-t0):.3f} ms", file=sys.stderr)
for _ in range(3):
    t0 = time.perf_counter(); x = np.empty(S); x.fill(0.0); t1 = time.perf_counter()
    print(f"fresh np.empty + fill {1e3*(t1-t0):.3f} ms", file=sys.stderr)
    del x
