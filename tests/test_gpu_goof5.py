"""The bench configuration itself (BASELINE.json configs[3]: Goofspiel-5,
PCFR+ alternating, fp64) against the REFERENCE: digests of the reference's
own iterates at iterations 1, 2, 10, 30 and 50 and its exploitability at 30
and 50 (tests/golden/goof5_meta.json, written by
scripts/make_golden_goof5.py running pkg/solvers.py:351-372), plus CFR sim
@10.  The bench times 20-50 iterations of exactly this solve, and CFR
iterates are chaotic at the ULP level, so bit-equality here
at 50 iterations is what pins the measured workload."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, digest
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, flat_goofspiel

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _meta():
    with open(os.path.join(GOLDEN, "goof5_meta.json")) as fh:
        return json.load(fh)


_B = {}


def _bundle():
    if "b" not in _B:
        _B["b"] = GameBundle(flat_goofspiel(5))
    return _B["b"]


def _check(s, rec, key, behavior):
    got = {"avg1": s.average(1), "avg2": s.average(2), "x1": s.current(1), "x2": s.current(2),
           "r1": s.regrets(1), "r2": s.regrets(2), "acc1": s.state(1, "accum"),
           "acc2": s.state(2, "accum"), "u1": s.state(1, "utility"), "u2": s.state(2, "utility")}
    if behavior:
        got["b1"] = s.state(1, "behavior")
        got["b2"] = s.state(2, "behavior")
    for k, v in got.items():
        assert digest(v) == rec["digests"][k], (key, k)
    assert s.avg_weight() == rec["avg_weight"][0]
    if "expl" in rec:
        e, br = s.exploitability("average")
        assert e == rec["expl"] and list(br) == rec["br_avg"], key
        assert s.exploitability("current")[0] == rec["expl_current"], key


@pytest.mark.parametrize("engine", ["auto", "levels"])
def test_goofspiel5_pcfr_plus_alt_matches_reference(gpu, engine):
    meta = _meta()["lockstep"]
    marks = sorted(int(k.rsplit(".", 1)[1]) for k in meta if k.startswith("goof5.pcfr+.alt."))
    assert marks == [1, 2, 10, 30, 50]
    s = Solver(_bundle(), SolverConfig("pcfr+"), device=gpu, engine=engine)
    done = 0
    for m in marks:
        s.step(m - done)
        done = m
        _check(s, meta[f"goof5.pcfr+.alt.{m}"], m, behavior=True)
    s.check_finite()


def test_goofspiel5_cfr_sim_matches_reference(gpu):
    rec = _meta()["lockstep"]["goof5.cfr.sim.10"]
    s = Solver(_bundle(), SolverConfig("cfr", mode="sim"), device=gpu)
    s.step(10)
    _check(s, rec, "cfr.sim.10", behavior=False)


def test_goofspiel5_fp32_mode_tracks_fp32_oracle(gpu):
    """The optional fp32 mode at the bench size, 10 iterations, against the
    fp32 restatement (relative 1e-5 bar; bit equality is what is observed)."""
    from oracle import tree
    from oracle.oracle import OracleSolver
    ob = tree.native_bundle("goofspiel", 5)
    s = Solver(_bundle(), SolverConfig("pcfr+"), device=gpu, dtype="f32")
    s.step(10)
    o = OracleSolver(ob, "pcfr+", threads=os.cpu_count() or 1, dtype="f32")
    o.step(10)
    for pl in (1, 2):
        np.testing.assert_allclose(s.average(pl), o.average(pl), rtol=1e-5, atol=0)
        np.testing.assert_array_equal(s.regrets(pl), o.regrets(pl))


def test_goofspiel5_target_iteration_matches_reference(gpu):
    """Time-to-target of the bench config: the first iteration with
    exploitability <= 1e-4, found on the device, equals the reference's
    (recorded by scripts/make_golden_goof5.py --target T)."""
    tgt = _meta().get("target", {})
    if not tgt:
        pytest.skip("no reference target run recorded")
    from paper_2605_14277_b200 import solve_to_target
    rec = next(iter(tgt.values()))
    T = rec["iters"]
    before, at = rec["records"]
    assert before["exploitability"] > 1e-4 >= at["exploitability"]
    r = solve_to_target(_bundle(), SolverConfig("pcfr+"), 1e-4, check_every=1, device=gpu)
    assert r.reached and r.iterations == T
    assert r.exploitability == at["exploitability"]
