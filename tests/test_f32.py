"""The optional fp32 mode (north star: "an optional fp32 mode within 1e-5").

fp32 iterates cannot track the fp64 reference: CFR is chaotic at the ULP
level.  The checker is therefore a float32 restatement of
the same operation order: the C oracle built with -DREAL=float
(oracle/seqcfr_oracle.c).  The bar written in the tests:

* iterates (regrets, behaviours, average accumulators, utilities, strategies)
  within 1e-5 relative of the fp32 oracle; the kernels reproduce its
  operation order, so they are in fact equal bit for bit, and that is
  asserted too;
* exploitability: fp64 best response on the widened average, equal to the
  fp64 oracle's best response on the fp32 oracle's average.

CPU tests pin the fp32 oracle itself: float-representable state, thread-count
determinism, and closeness to the fp64 reference where CFR is not chaotic
(Kuhn CFR: the SURVEY chaos table gives 1e-15 for a reordered fp64 sum there).
"""

import numpy as np
import pytest

from conftest import bundle, golden_meta, oracle_bundle
from oracle.oracle import OracleSolver

F32_TOL = 1e-5  # relative; the north-star bound for the fp32 mode


def _f32_oracle(name, variant, mode=None, gamma=None, alpha=1.5, beta=0.0, iters=50, threads=1):
    o = OracleSolver(oracle_bundle(name), variant, mode, alpha, beta, gamma, threads=threads, dtype="f32")
    o.step(iters)
    return o


def _representable_f32(a):
    a = np.asarray(a)
    return np.array_equal(a.astype(np.float32).astype(np.float64), a)


def test_f32_oracle_state_is_float32():
    o = _f32_oracle("leduc", "cfr+", iters=30)
    for pl in (1, 2):
        for v in (o.regrets(pl), o.behavior(pl), o.avg_accum(pl), o.utility(pl), o.current(pl)):
            assert _representable_f32(v)


def test_f32_oracle_deterministic_across_threads():
    a = _f32_oracle("liars3", "dcfr", iters=40, threads=1)
    b = _f32_oracle("liars3", "dcfr", iters=40, threads=4)
    for pl in (1, 2):
        np.testing.assert_array_equal(a.avg_accum(pl), b.avg_accum(pl))
        np.testing.assert_array_equal(a.regrets(pl), b.regrets(pl))


def test_f32_oracle_tracks_fp64_on_kuhn_cfr():
    """Kuhn CFR @1000 is not chaotic: fp32 lands within fp32 rounding of the
    reference's exploitability 7.2691064e-3 (golden) and value -1/18."""
    want = golden_meta()["runs"]["kuhn.cfr.1000"]["records"][-1]["exploitability"]
    o32 = _f32_oracle("kuhn", "cfr", iters=1000)
    o64 = OracleSolver(oracle_bundle("kuhn"), "cfr")  # fp64 best response as the metric
    e, _ = o64.exploitability(o32.average(1), o32.average(2))
    assert abs(e - want) <= 1e-4 * abs(want) + 1e-7


# --- GPU: the fp32 kernels against the fp32 oracle -------------------------

CASES = [("kuhn", "cfr", "sim", 200), ("leduc", "cfr+", "alt", 100), ("leduc", "pcfr+", "alt", 100),
         ("leduc", "pcfr", "sim", 60), ("random6", "dcfr", "sim", 120), ("liars3", "dcfr", "alt", 60),
         ("goof3", "pcfr+", "sim", 60), ("goof4", "pcfr+", "alt", 10), ("liars6", "dcfr", "alt", 20),
         ("random7", "cfr", "alt", 40)]


def _rm_f32(proc, regrets):
    """Regret matching of the regrets in float32, op for op (pkg/solvers.py:156-160):
    the behaviour the next iteration plays."""
    r = np.concatenate([[0.0], regrets]).astype(np.float32)
    b = np.zeros_like(r)
    for j in range(proc.num_decisions):
        s0, n = int(proc.dp_first_seq[j]), int(proc.dp_num_actions[j])
        S = np.float32(0.0)
        for a in range(n):
            S = np.float32(S + max(r[s0 + a], np.float32(0.0)))
        for a in range(n):
            p = max(r[s0 + a], np.float32(0.0))
            b[s0 + a] = np.float32(p / S) if S != 0 else np.float32(np.float32(1.0) / np.float32(n))
    return b[1:].astype(np.float64)


def _close(got, want, what):
    got, want = np.asarray(got), np.asarray(want)
    scale = np.maximum(np.abs(want), 1e-30)
    assert np.all(np.abs(got - want) <= F32_TOL * scale + 1e-30), what
    np.testing.assert_array_equal(got, want, err_msg=what)  # op-for-op restatement: exact


@pytest.mark.gpu
@pytest.mark.parametrize("game,variant,mode,iters", CASES)
def test_f32_kernels_match_f32_oracle(gpu, game, variant, mode, iters):
    from paper_2605_14277_b200 import Solver, SolverConfig
    s = Solver(bundle(game), SolverConfig(variant, mode=mode), device=gpu, dtype="f32")
    assert s.dtype == "f32" and s.engine == "levels"
    s.step(iters)
    o = _f32_oracle(game, variant, mode=mode, iters=iters)
    predictive = variant in ("pcfr", "pcfr+")
    for pl in (1, 2):
        _close(s.regrets(pl), o.regrets(pl), (game, pl, "regrets"))
        # non-predictive variants regret-match inside the observe pass, so the
        # stored behaviour is the one the NEXT iteration plays: RM(regrets)
        want_b = o.behavior(pl) if predictive else _rm_f32(bundle(game).procs[pl - 1], o.regrets(pl))
        _close(s.state(pl, "behavior"), want_b, (game, pl, "behavior"))
        _close(s.state(pl, "accum"), o.avg_accum(pl), (game, pl, "accum"))
        _close(s.state(pl, "utility"), o.utility(pl), (game, pl, "utility"))
        _close(s.current(pl), o.current(pl), (game, pl, "current"))
        _close(s.average(pl), o.average(pl), (game, pl, "average"))
    o64 = OracleSolver(oracle_bundle(game), variant, mode)
    want, wbr = o64.exploitability(o.average(1), o.average(2))
    got, gbr = s.exploitability("average")
    assert got == want and list(gbr) == list(wbr)
    s.check_finite()


@pytest.mark.gpu
def test_f32_rejects_other_engines(gpu):
    from paper_2605_14277_b200 import Solver, SolverConfig
    with pytest.raises(ValueError):
        Solver(bundle("kuhn"), SolverConfig("cfr"), device=gpu, dtype="f32", engine="persistent")


def test_unknown_dtype_rejected():
    from paper_2605_14277_b200 import Solver, SolverConfig
    with pytest.raises(ValueError):
        Solver(bundle("kuhn"), SolverConfig("cfr"), dtype="f16")


@pytest.mark.gpu
@pytest.mark.slow
def test_f32_goofspiel5_full_size(gpu):
    """The largest config in fp32: 2 PCFR+ iterations against the fp32 oracle."""
    from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, flat_goofspiel
    b = GameBundle(flat_goofspiel(5))
    s = Solver(b, SolverConfig("pcfr+"), device=gpu, dtype="f32")
    s.step(2)
    o = OracleSolver(b, "pcfr+", threads=8, dtype="f32")
    o.step(2)
    for pl in (1, 2):
        np.testing.assert_array_equal(s.regrets(pl), o.regrets(pl))
        np.testing.assert_array_equal(s.average(pl), o.average(pl))
