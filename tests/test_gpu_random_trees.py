"""Parity sweep over generated game trees: the CUDA path against the C oracle
(itself pinned bit-exact to the reference by tests/test_oracle.py), for many
random shapes.  The trees vary depth, branching and infoset merge rate
(pkg/games.py:470-548).  That exercises non-layered decision processes,
observation points with many children, wide and single-action levels, and
the affine-shape detection.  Bar: bit-exact regrets, averages, utilities and
exploitability, on every engine that takes the tree."""

import numpy as np
import pytest

from oracle import tree
from oracle.oracle import OracleSolver
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig
from paper_2605_14277_b200 import games as G

pytestmark = pytest.mark.gpu

SHAPES = [(4, 2, 0.0, 3), (5, 3, 0.5, 11), (6, 2, 0.3, 5), (7, 2, 0.8, 2), (5, 4, 0.2, 9),
          (8, 2, 0.5, 17), (3, 6, 0.7, 4), (6, 3, 0.0, 23), (9, 2, 0.25, 31), (4, 5, 0.4, 8),
          (11, 2, 0.3, 7), (7, 3, 0.4, 13), (13, 2, 0.2, 19), (8, 3, 0.6, 3)]
VARIANTS = [("cfr", "sim"), ("cfr+", "alt"), ("dcfr", "alt"), ("pcfr", "sim"), ("pcfr+", "alt")]


def _bundles(shape):
    g = G.random_game(*shape)
    return GameBundle(g), tree.compile_flat(g.flatten())


@pytest.mark.parametrize("shape", SHAPES)
def test_random_trees_group_mode(gpu, shape, monkeypatch):
    """Group mode forced onto every eligible level, against the oracle."""
    monkeypatch.setenv("SCFR_GROUP_NJ", "0")
    b, ob = _bundles(shape)
    for k, (variant, mode) in enumerate(VARIANTS):
        iters = 20 + 5 * k
        o = OracleSolver(ob, variant, mode)
        o.step(iters)
        s = Solver(b, SolverConfig(variant, mode=mode), device=gpu, engine="levels")
        s.step(iters)
        for pl in (1, 2):
            np.testing.assert_array_equal(s.regrets(pl), o.regrets(pl), err_msg=f"{shape} {variant}")
            np.testing.assert_array_equal(s.average(pl), o.average(pl))
            np.testing.assert_array_equal(s.state(pl, "utility"), o.utility(pl))
        s.close()


@pytest.mark.parametrize("shape", SHAPES)
def test_random_trees_bit_exact(gpu, shape):
    b, ob = _bundles(shape)
    for k, (variant, mode) in enumerate(VARIANTS):
        iters = 25 + 7 * k
        o = OracleSolver(ob, variant, mode)
        o.step(iters)
        for engine in ("auto", "levels", "persistent", "tiled"):
            try:
                s = Solver(b, SolverConfig(variant, mode=mode), device=gpu, engine=engine)
            except ValueError:  # no tile plan for this tree
                assert engine == "tiled"
                continue
            s.step(iters)
            for pl in (1, 2):
                np.testing.assert_array_equal(s.regrets(pl), o.regrets(pl), err_msg=f"{shape} {variant} {engine}")
                np.testing.assert_array_equal(s.average(pl), o.average(pl))
                np.testing.assert_array_equal(s.state(pl, "utility"), o.utility(pl))
            e, _ = s.exploitability("average")
            assert e == o.exploitability(o.average(1), o.average(2))[0], (shape, variant, engine)
            s.close()
