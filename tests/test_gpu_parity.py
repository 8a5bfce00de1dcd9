"""CUDA path parity through the C-ABI (scfr_create / scfr_step / ...).

Bar: bit-exact fp64 against the reference (golden digests produced by the
reference itself) on every lockstep case, checkpoint record and best
response; at full Goofspiel-5 size, bit-exact against the oracle after a few
iterations plus size-independent properties (sequence-form polytope,
determinism)."""

import numpy as np
import pytest

from conftest import bundle, digest, golden_arrays, golden_meta
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, flat_goofspiel, metrics, run

pytestmark = pytest.mark.gpu
CASES = sorted(golden_meta()["lockstep"])


def _cfg(rec):
    return SolverConfig(rec["variant"], alpha=rec["alpha"], beta=rec["beta"], gamma=rec["gamma"],
                        mode=rec["mode"])


def _state(s, solve=0):
    return {"avg1": s.average(1, solve), "avg2": s.average(2, solve),
            "x1": s.current(1, solve), "x2": s.current(2, solve),
            "r1": s.regrets(1, solve), "r2": s.regrets(2, solve),
            "acc1": s.state(1, "accum", solve), "acc2": s.state(2, "accum", solve),
            "u1": s.state(1, "utility", solve), "u2": s.state(2, "utility", solve)}


@pytest.mark.parametrize("key", CASES)
def test_lockstep_bit_exact(gpu, key):
    rec = golden_meta()["lockstep"][key]
    s = Solver(bundle(rec["game"]), _cfg(rec), device=gpu)
    s.step(rec["iters"])
    for k, v in _state(s).items():
        assert digest(v) == rec["digests"][k], (key, k)
    e, br = s.exploitability("average")
    assert e == rec["expl"] and list(br) == rec["br_avg"]
    assert s.exploitability("current")[0] == rec["expl_current"]
    assert s.avg_weight() == rec["avg_weight"][0]
    s.check_finite()


@pytest.mark.parametrize("key", ["kuhn.cfr.sim.200", "leduc.pcfr+.alt.100", "random6.dcfr.alt.200"])
def test_lockstep_full_arrays(gpu, key):
    rec = golden_meta()["lockstep"][key]
    arr = golden_arrays()
    s = Solver(bundle(rec["game"]), _cfg(rec), device=gpu)
    s.step(rec["iters"])
    st = _state(s)
    for k in ("avg1", "avg2", "x1", "x2", "r1", "r2", "u1", "u2"):
        np.testing.assert_array_equal(st[k], arr[f"{key}.{k}"])


@pytest.mark.parametrize("run_key", sorted(golden_meta()["runs"]))
def test_run_records_match_reference(gpu, run_key):
    want = golden_meta()["runs"][run_key]
    res = run(bundle(want["game"]), SolverConfig(want["variant"]), iterations=want["iters"],
              checkpoints=want["checkpoints"], device=gpu)
    assert res.iterations == want["iters"]
    assert [r.iteration for r in res.records] == [r["iteration"] for r in want["records"]]
    for got, ref in zip(res.records, want["records"]):
        assert got.exploitability == ref["exploitability"]
        assert got.current_exploitability == ref["current_exploitability"]
        assert got.work == ref["work"] and got.peak_bytes == ref["peak_bytes"]
    assert digest(res.average[0]) == want["digests"]["avg1"]
    assert digest(res.average[1]) == want["digests"]["avg2"]
    assert metrics.expected_value(res.bundle, *res.average) == want["value"]


def test_batched_dcfr_sweep_matches_individual_solves(gpu):
    recs = [r for k, r in sorted(golden_meta()["lockstep"].items())
            if k.startswith("leduc.dcfr.alt.200.")]
    assert len(recs) == 8
    params = [(r["alpha"], r["beta"], r["gamma"]) for r in recs]
    s = Solver(bundle("leduc"), SolverConfig("dcfr"), device=gpu, batch_params=params)
    s.step(200)
    for k, rec in enumerate(recs):
        st = _state(s, k)
        for name in ("avg1", "avg2", "r1", "r2", "x1", "x2"):
            assert digest(st[name]) == rec["digests"][name], (k, name)
        assert s.exploitability("average", k)[0] == rec["expl"]


def test_best_response_uniform(gpu):
    arr = golden_arrays()
    for name, rec in golden_meta()["br"].items():
        b = bundle(name)
        got = metrics.best_response_values(b, arr[f"{name}.uniform.x1"], arr[f"{name}.uniform.x2"])
        assert list(got) == rec["uniform"], name


def test_deterministic_and_graph_free_path_agree(gpu, monkeypatch):
    rec = golden_meta()["lockstep"]["liars3.pcfr+.alt.60"]
    a = Solver(bundle("liars3"), _cfg(rec), device=gpu)
    a.step(rec["iters"])
    monkeypatch.setenv("SCFR_NO_GRAPH", "1")
    b = Solver(bundle("liars3"), _cfg(rec), device=gpu)
    b.step(rec["iters"])
    for k in ("avg1", "r2", "u1"):
        np.testing.assert_array_equal(_state(a)[k], _state(b)[k])


def test_nonfinite_regrets_raise(gpu):
    from paper_2605_14277_b200 import games as G
    g = G.GameBuilder("huge")
    top = g.decision(None, None, 1, "p1")
    for a in ("H", "T"):
        sub = g.decision(top, a, 2, "p2")
        for b_ in ("H", "T"):
            g.terminal(sub, b_, 1.7e308 if a == b_ else -1.7e308)
    s = Solver(GameBundle(g.build()), SolverConfig("cfr"), device=gpu)
    s.step(4)
    with pytest.raises(FloatingPointError):
        s.check_finite()


@pytest.mark.slow
def test_goofspiel5_full_size_against_oracle(gpu):
    """Largest config at full size: 2 PCFR+ iterations bit-exact vs the C oracle,
    then sequence-form polytope membership of the average."""
    from oracle.oracle import OracleSolver
    b = GameBundle(flat_goofspiel(5))
    s = Solver(b, SolverConfig("pcfr+"), device=gpu)
    s.step(2)
    o = OracleSolver(b, "pcfr+", threads=8)
    o.step(2)
    for pl in (1, 2):
        np.testing.assert_array_equal(s.regrets(pl), o.regrets(pl))
        np.testing.assert_array_equal(s.average(pl), o.average(pl))
        np.testing.assert_array_equal(s.state(pl, "utility"), o.utility(pl))
    for pl in (1, 2):
        p = b.procs[pl - 1]
        x = s.average(pl)
        assert x[0] == 1.0
        sums = np.add.reduceat(x[1:], p.dp_first_seq - 1)
        np.testing.assert_allclose(sums, x[p.dp_parent_seq], rtol=0, atol=1e-11)
