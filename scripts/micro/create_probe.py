"""Create-time probe: wall time of Solver() for Goofspiel-5 vs the native
SCFR_TRACE stage sum (run with SCFR_TRACE=1)."""
import sys, time
sys.path.insert(0, ".")
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, flat_goofspiel
b = GameBundle(flat_goofspiel(5))
cfg = SolverConfig("pcfr+")
for i in range(8):
    t0 = time.perf_counter()
    s = Solver(b, cfg)
    t1 = time.perf_counter()
    s.step(50); s.synchronize()
    t2 = time.perf_counter()
    a = (s.average(1), s.average(2))
    t3 = time.perf_counter()
    s.close()
    t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):7.2f} steps {1e3*(t2-t1):7.2f} read {1e3*(t3-t2):6.2f} close {1e3*(t4-t3):6.2f} ms", file=sys.stderr, flush=True)
