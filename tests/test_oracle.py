"""Pins the oracle (oracle/seqcfr_oracle.c) to the reference: every lockstep
golden case (5 variants x 2 modes x 8 games, variant defaults on Kuhn @1000,
the Leduc DCFR grid, Liar's dice / Goofspiel-4 digests) must match BIT FOR
BIT — regrets, behaviours, averages, utilities, last iterates and
exploitability.  Also the spec's toy examples."""

import math

import numpy as np
import pytest

from conftest import digest, golden_arrays, golden_meta, oracle_bundle
from oracle.oracle import OracleSolver
from paper_2605_14277_b200 import games as G

CASES = sorted(golden_meta()["lockstep"])


def _run(rec, threads=1):
    s = OracleSolver(oracle_bundle(rec["game"]), rec["variant"], rec["mode"], rec["alpha"],
                     rec["beta"], rec["gamma"], threads=threads)
    s.step(rec["iters"])
    return s


@pytest.mark.parametrize("key", CASES)
def test_oracle_lockstep_bit_exact(key):
    rec = golden_meta()["lockstep"][key]
    s = _run(rec)
    got = {"avg1": s.average(1), "avg2": s.average(2), "x1": s.current(1), "x2": s.current(2),
           "r1": s.regrets(1), "r2": s.regrets(2), "acc1": s.avg_accum(1),
           "acc2": s.avg_accum(2), "u1": s.utility(1), "u2": s.utility(2)}
    for k, v in got.items():
        assert digest(v) == rec["digests"][k], (key, k)
    e, br = s.exploitability(s.average(1), s.average(2))
    assert e == rec["expl"] and list(br) == rec["br_avg"]
    ec, _ = s.exploitability(s.current(1), s.current(2))
    assert ec == rec["expl_current"]


def test_oracle_thread_count_invariance():
    rec = golden_meta()["lockstep"]["goof4.pcfr+.alt.10"]
    s = _run(rec, threads=4)
    assert digest(s.average(1)) == rec["digests"]["avg1"]
    assert digest(s.regrets(2)) == rec["digests"]["r2"]


@pytest.mark.parametrize("run_key", ["kuhn.cfr.1000", "leduc.cfr+.1592", "leduc.dcfr.1000"])
def test_oracle_checkpoint_exploitability(run_key):
    run = golden_meta()["runs"][run_key]
    s = OracleSolver(oracle_bundle(run["game"]), run["variant"])
    t = 0
    for rec in run["records"]:
        s.step(rec["iteration"] - t)
        t = rec["iteration"]
        e, _ = s.exploitability(s.average(1), s.average(2))
        assert e == rec["exploitability"]
        ec, _ = s.exploitability(s.current(1), s.current(2))
        assert ec == rec["current_exploitability"]


def test_known_answers():
    """Kuhn CFR@1000 = 7.269e-3; Leduc CFR+ first <= 1e-4 at 1592."""
    runs = golden_meta()["runs"]
    assert abs(runs["kuhn.cfr.1000"]["records"][-1]["exploitability"] - 0.0072691064085643325) < 1e-15
    leduc = {r["iteration"]: r["exploitability"] for r in runs["leduc.cfr+.1592"]["records"]}
    assert leduc[1592] <= 1e-4 < leduc[1591]


def test_best_response_uniform():
    arr = golden_arrays()
    for name, rec in golden_meta()["br"].items():
        s = OracleSolver(oracle_bundle(name), "cfr")
        x1, x2 = arr[f"{name}.uniform.x1"], arr[f"{name}.uniform.x2"]
        b1, b2 = s.best_response(1, x2), s.best_response(2, x1)
        assert [b1, b2] == rec["uniform"]


def _single_dp_game():
    b = G.GameBuilder("single")
    d = b.decision(None, None, 1, "p1")
    for a, pay in (("a", 0.0), ("b", 4.0)):
        b.terminal(d, a, pay)
    return b.build()


def test_spec_toy_examples():
    from oracle import tree
    ob = tree.compile_flat(_single_dp_game().flatten())
    s = OracleSolver(ob, "cfr", "sim")
    s.step(1)  # uniform b = [.5,.5], u = [0, 0, 4] -> r = [-2, 2]
    np.testing.assert_array_equal(s.regrets(1), [-2.0, 2.0])
    s.step(1)  # b = [0, 1]; u = [0, 0, 4] -> r += [-4, 0]
    np.testing.assert_array_equal(s.current(1), [1.0, 0.0, 1.0])
    np.testing.assert_array_equal(s.regrets(1), [-6.0, 2.0])
