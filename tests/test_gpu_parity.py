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


@pytest.mark.parametrize("key", CASES)
def test_group_mode_bit_exact(gpu, key, monkeypatch):
    """Level engine with group mode (G = 32/n DPs per warp) forced onto every
    eligible level (uniform 2..16 actions, below level 0) of the lockstep cases."""
    monkeypatch.setenv("SCFR_GROUP_NJ", "0")
    rec = golden_meta()["lockstep"][key]
    s = Solver(bundle(rec["game"]), _cfg(rec), device=gpu, engine="levels")
    s.step(rec["iters"])
    for k, v in _state(s).items():
        assert digest(v) == rec["digests"][k], (key, k)
    e, br = s.exploitability("average")
    assert e == rec["expl"] and list(br) == rec["br_avg"]


# Level-engine modes forced onto every eligible level, each checked against
# the reference digests: the cp.async-pipelined group kernels (all pass
# kinds), parent pairs, the plain launches without the top recompute /
# fused leaf rows, and alt iterations without the two-stream overlap.
MODES = {
    "pipelined": {"SCFR_GROUP_NJ": "0", "SCFR_PIPE_NJ": "0", "SCFR_PIPE_KINDS": "31"},
    "pairs": {"SCFR_GROUP_NJ": "0", "SCFR_PAIR": "1"},
    "unfused": {"SCFR_NO_TOP": "1", "SCFR_NO_LEAF_FUSE": "1"},
    "sequential": {"SCFR_NO_OVERLAP": "1"},
    "obs_side": {"SCFR_OBS_SIDE": "1"},  # (predictive alt cases: OBS2's top levels on a third stream)
    "cur_top": {"SCFR_CUR_TOP": "1"},  # (alt cases: player 1's current strategy from a deeper top)
}


@pytest.mark.parametrize("mode", sorted(MODES))
@pytest.mark.parametrize("key", [k for k in CASES if k.split(".")[0] in ("goof4", "liars6", "random7", "leduc")])
def test_level_engine_modes_bit_exact(gpu, key, mode, monkeypatch):
    for name, value in MODES[mode].items():
        monkeypatch.setenv(name, value)
    rec = golden_meta()["lockstep"][key]
    s = Solver(bundle(rec["game"]), _cfg(rec), device=gpu, engine="levels")
    s.step(rec["iters"])
    for k, v in _state(s).items():
        assert digest(v) == rec["digests"][k], (key, mode, k)
    e, br = s.exploitability("average")
    assert e == rec["expl"] and list(br) == rec["br_avg"]


def test_deterministic_and_graph_free_path_agree(gpu, monkeypatch):
    """The level engine with and without CUDA-graph replay."""
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
    # H always pays +1.7e308, T -1.7e308: after one iteration r_T = -1.7e308,
    # the next update adds (-E) + q = -3.4e308 -> -inf (the reference raises
    # FloatingPointError at the following next_strategy, pkg/solvers.py:154).
    g = G.GameBuilder("huge")
    top = g.decision(None, None, 1, "p1")
    for a in ("H", "T"):
        sub = g.decision(top, a, 2, "p2")
        for b_ in ("H", "T"):
            g.terminal(sub, b_, 1.7e308 if a == "H" else -1.7e308)
    s = Solver(GameBundle(g.build()), SolverConfig("cfr"), device=gpu)
    s.step(1)
    s.check_finite()
    s.step(3)
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


ENGINES = ["levels", "persistent", "persistent_grid", "persistent_cluster"]
ENGINE_CASES = ["kuhn.cfr.sim.200", "leduc.cfr+.alt.100", "leduc.pcfr+.alt.100",
                "random6.dcfr.sim.200", "random7.pcfr.alt.40", "liars3.dcfr.alt.60",
                "goof3.pcfr+.sim.60", "mp.cfr+.alt.50", "liars6.dcfr.alt.30.a1.5.b0.0.g2.0"]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("key", ENGINE_CASES)
def test_engines_bit_exact(gpu, engine, key):
    """Every engine reproduces the reference bit for bit (same per-DP code)."""
    rec = golden_meta()["lockstep"][key]
    s = Solver(bundle(rec["game"]), _cfg(rec), device=gpu, engine=engine)
    assert s.engine == engine
    # uneven step sizes exercise the iteration counter / schedule indexing
    done = 0
    for chunk in (1, 2, 7):
        if done + chunk <= rec["iters"]:
            s.step(chunk)
            done += chunk
    s.step(rec["iters"] - done)
    st = _state(s)
    for k in ("avg1", "avg2", "r1", "r2", "x1", "x2", "u1", "u2"):
        assert digest(st[k]) == rec["digests"][k], (key, engine, k)
    assert s.exploitability("average")[0] == rec["expl"]


def test_batched_persistent_sweep(gpu):
    """Config 5 shape: 256 Leduc DCFR solves in one handle, one CTA each; the
    8 golden parameter points are embedded in the batch and must match."""
    recs = [r for k, r in sorted(golden_meta()["lockstep"].items())
            if k.startswith("leduc.dcfr.alt.200.")]
    grid = [(a, b, g) for a in (0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 5.0, 8.0)
            for b in (-1.0, -0.5, 0.0, 0.5) for g in (0.0, 1.0, 2.0, 3.0)] * 2
    for k, r in enumerate(recs):
        grid[k * 31] = (r["alpha"], r["beta"], r["gamma"])
    s = Solver(bundle("leduc"), SolverConfig("dcfr"), device=gpu, batch_params=grid,
               engine="auto")
    assert s.engine == "persistent" and s.batch == 256
    s.step(200)
    for k, rec in enumerate(recs):
        assert digest(s.average(1, k * 31)) == rec["digests"]["avg1"]
        assert digest(s.regrets(2, k * 31)) == rec["digests"]["r2"]
        assert s.exploitability("average", k * 31)[0] == rec["expl"]


@pytest.mark.parametrize("key", ["leduc.pcfr+.alt.100", "liars3.dcfr.sim.60", "random6.cfr.alt.200",
                                 "goof3.cfr+.alt.60"])
def test_row_sharded_mode_world1_bit_exact(gpu, key):
    """The NCCL row-sharded path (scfr_create_sharded) on a 1-rank
    communicator: SpMV slices + in-place all-gather inside the iteration graph
    must leave every iterate bit-identical to the reference."""
    from paper_2605_14277_b200.distributed import nccl_unique_id
    rec = golden_meta()["lockstep"][key]
    s = Solver(bundle(rec["game"]), _cfg(rec), device=gpu, engine="levels",
               shard=(nccl_unique_id(), 0, 1))
    s.step(rec["iters"])
    st = _state(s)
    for k in ("avg1", "avg2", "r1", "r2", "u1", "u2"):
        assert digest(st[k]) == rec["digests"][k], (key, k)
    assert s.exploitability("average")[0] == rec["expl"]


def _tiled_or_skip(b, cfg, gpu, **kw):
    try:
        return Solver(b, cfg, device=gpu, engine="tiled", **kw)
    except ValueError as e:  # the tree has no tile plan (e.g. a one-level player)
        if "tile" in str(e):
            pytest.skip(str(e))
        raise


@pytest.mark.parametrize("key", CASES)
def test_tiled_engine_bit_exact(gpu, key):
    """The tile engine (renumbered subtrees, one launch per pass) against the
    reference on every lockstep case whose trees tile; reads come back in the
    reference's order."""
    rec = golden_meta()["lockstep"][key]
    s = _tiled_or_skip(bundle(rec["game"]), _cfg(rec), gpu)
    assert s.engine == "tiled"
    done = 0
    for chunk in (1, 3):
        if done + chunk <= rec["iters"]:
            s.step(chunk)
            done += chunk
    s.step(rec["iters"] - done)
    for k, v in _state(s).items():
        assert digest(v) == rec["digests"][k], (key, k)
    e, br = s.exploitability("average")
    assert e == rec["expl"] and list(br) == rec["br_avg"]
    assert s.exploitability("current")[0] == rec["expl_current"]
    s.check_finite()


def test_tiled_graph_free_and_profiled_paths_agree(gpu, monkeypatch):
    rec = golden_meta()["lockstep"]["goof4.pcfr+.alt.10"]
    a = _tiled_or_skip(bundle(rec["game"]), _cfg(rec), gpu)
    a.step(rec["iters"])
    monkeypatch.setenv("SCFR_NO_GRAPH", "1")
    b = _tiled_or_skip(bundle(rec["game"]), _cfg(rec), gpu)
    b.step(rec["iters"] - 2)
    prof = b.profile(2)
    assert set(prof) >= {"td_avg", "tick"}
    for k in ("avg1", "avg2", "r1", "u2"):
        np.testing.assert_array_equal(_state(a)[k], _state(b)[k])


def test_solve_to_target_coarse_to_fine_is_exact(gpu):
    """Snapshot / replay search finds the same first iteration <= 1e-4 as a
    check after every iteration: Leduc CFR+ @1592 (reference golden run)."""
    from paper_2605_14277_b200 import solve_to_target
    want = golden_meta()["runs"]["leduc.cfr+.1592"]["records"][-1]
    r = solve_to_target(bundle("leduc"), SolverConfig("cfr+"), 1e-4, check_every=1, stride=16)
    assert r.reached and r.iterations == 1592 and r.exploitability == want["exploitability"]
    assert r.checks < 1592 // 4
    r1 = solve_to_target(bundle("leduc"), SolverConfig("cfr+"), 1e-4, check_every=1, stride=1)
    assert (r1.iterations, r1.exploitability) == (r.iterations, r.exploitability)


@pytest.mark.parametrize("engine", ["levels", "persistent", "tiled"])
def test_snapshot_restore_replays_bit_exact(gpu, engine):
    rec = golden_meta()["lockstep"]["goof3.pcfr+.alt.60"]
    s = Solver(bundle(rec["game"]), _cfg(rec), device=gpu, engine=engine)
    s.step(20)
    s.snapshot()
    s.step(rec["iters"] - 20)
    first = _state(s)
    s.snapshot(restore=True)
    assert s.iterations == 20
    s.step(rec["iters"] - 20)
    for k, v in _state(s).items():
        np.testing.assert_array_equal(v, first[k])
        assert digest(v) == rec["digests"][k], k


@pytest.mark.parametrize("engine", ["levels", "persistent"])
def test_set_schedule_reproduces_other_parameters(gpu, engine):
    """scfr_set_schedule: a DCFR solve given the weights and factors of
    other (alpha, beta, gamma) equals the solve created with them, bit for
    bit (state and the host-side average weight)."""
    from paper_2605_14277_b200.solvers import discount_factors
    n = 60
    target = SolverConfig("dcfr", alpha=2.5, beta=-0.5, gamma=3.0)
    ref = Solver(bundle("leduc"), target, device=gpu, engine=engine)
    ref.step(n)
    s = Solver(bundle("leduc"), SolverConfig("dcfr", alpha=1.5, beta=0.0, gamma=2.0), device=gpu, engine=engine)
    ts = range(1, n + 1)
    s.set_schedule(w=[float(t) ** 3.0 for t in ts], pos_factor=[discount_factors(t, 2.5, -0.5)[0] for t in ts],
                   neg_factor=[discount_factors(t, 2.5, -0.5)[1] for t in ts])
    s.step(n)
    for k, v in _state(ref).items():
        np.testing.assert_array_equal(_state(s)[k], v, err_msg=k)
    assert s.avg_weight() == ref.avg_weight()
    with pytest.raises(ValueError):
        s.set_schedule(w=[float("inf")])
