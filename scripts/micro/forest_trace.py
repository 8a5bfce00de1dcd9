"""Phase trace of one forest-mode iteration (CTA 0 of every launch; clock64
cycles).  python scripts/micro/forest_trace.py [goof5|goof4] [variant] [mode]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, flat_goofspiel  # noqa: E402
from paper_2605_14277_b200 import native as N  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "goof5"
variant = sys.argv[2] if len(sys.argv) > 2 else "pcfr+"
mode = sys.argv[3] if len(sys.argv) > 3 else "alt"
b = GameBundle(flat_goofspiel(int(name[-1])))
s = Solver(b, SolverConfig(variant, mode=mode), engine="levels")
s.step(5)
s.synchronize()
lib = N.lib()
lib.scfr_trace_start.argtypes = [C.c_int]
lib.scfr_trace_read.argtypes = [C.POINTER(C.c_int64), C.c_int, C.POINTER(C.c_int)]
cap = 1 << 16
N.check(lib.scfr_trace_start(cap))
s.step(1)
s.synchronize()
out = np.zeros(cap, dtype=np.int64)
n = C.c_int()
N.check(lib.scfr_trace_read(out.ctypes.data_as(C.POINTER(C.c_int64)), cap, C.byref(n)))
ev = out[: n.value]
tags = ev & 0xFF
clk = ev >> 8
# per launch (tag 1 starts one): items, issue->ready, ready->done cycles
launches = []
for t, c in zip(tags, clk):
    if t == 1:
        launches.append({"start": c, "ev": []})
    elif launches:
        launches[-1]["ev"].append((int(t), int(c)))
for k, L in enumerate(launches):
    ev = L["ev"]
    wait = [c1 - c0 for (t0, c0), (t1, c1) in zip(ev, ev[1:]) if t0 == 2 and t1 == 3]
    comp = [c1 - c0 for (t0, c0), (t1, c1) in zip(ev, ev[1:]) if t0 == 3 and t1 == 4]
    first = ev[0][1] - L["start"] if ev else 0
    end = ev[-1][1] - L["start"] if ev else 0
    print(f"launch {k}: items {len(comp)}, first issue+ {first} cyc, wait med {int(np.median(wait)) if wait else 0}, "
          f"compute med {int(np.median(comp)) if comp else 0} max {max(comp) if comp else 0}, span {end} cyc")
print("step ms", s.last_step_ms())
lib.scfr_trace_start(0)
# raw dump of the first 200 events of launch 0 with deltas
ev0 = [(int(t), int(c)) for t, c in zip(tags, clk)][:200]
prev = ev0[0][1] if ev0 else 0
for t, c in ev0:
    print(f"  tag {t:3d} +{c - prev}")
    prev = c
