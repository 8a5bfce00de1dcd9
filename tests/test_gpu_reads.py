"""scfr_read_averages (both players in one pipelined read) returns exactly
what two scfr_read_average calls return, on the level engine (with forced
leaf expansion), the SMEM engine and a batch."""

import numpy as np
import pytest

from conftest import bundle
from paper_2605_14277_b200 import Solver, SolverConfig

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,variant,engine,batch", [
    ("goof4", "pcfr+", "levels", 1),
    ("leduc", "cfr+", "persistent", 1),
    ("leduc", "dcfr", "persistent", 3),
])
def test_averages_match_single_reads(gpu, name, variant, engine, batch):
    b = bundle(name)
    cfg = SolverConfig(variant)
    kw = {"batch_params": [(1.5, 0.0, 2.0), (1.0, -0.5, 1.0), (2.0, 0.5, 3.0)][:batch]} if batch > 1 else {}
    s = Solver(b, cfg, device=gpu, engine=engine, **kw)
    s.step(9)
    for solve in range(batch):
        a1, a2 = s.averages(solve)
        assert np.array_equal(a1.view(np.uint64), s.average(1, solve).view(np.uint64))
        assert np.array_equal(a2.view(np.uint64), s.average(2, solve).view(np.uint64))
    s.close()
