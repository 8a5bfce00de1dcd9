"""Launch structure of the level engine: merged levels, exact shortcuts and
group mode change how many kernels one iteration runs, never the results.
The counts come from scfr_profile_step (CUDA events around every launch)
and guard against silently losing an optimisation."""

import numpy as np
import pytest

from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, flat_liars_dice

pytestmark = pytest.mark.gpu


def _launches(b, cfg):
    s = Solver(b, cfg, engine="levels")
    s.step(3)
    prof = s.profile(1)
    r = s.regrets(1)
    s.close()
    return {k: v["launches"] for k, v in prof.items()}, r


def test_liars_dice_merged_levels(gpu, monkeypatch):
    # the level engine's launched levels (the top recompute and the fused
    # leaf rows change the count; test_top_and_leaf_fusion covers those)
    monkeypatch.setenv("SCFR_NO_TOP", "1")
    monkeypatch.setenv("SCFR_NO_LEAF_FUSE", "1")
    b = GameBundle(flat_liars_dice(6))
    cfg = SolverConfig("dcfr", gamma=2.0)
    merged, r_merged = _launches(b, cfg)
    # 7 / 6 merged levels: TD+avg over max(7, 6), CUR-as-TD over player 1's 7
    # minus its forced leaf level, OBS over 7 + 6, one tick
    assert merged == {"td_avg": 6, "td": 6, "obs_rm": 13, "tick": 1}, merged
    monkeypatch.setenv("SCFR_NO_LEVEL_MERGE", "1")
    node_depth, r_nd = _launches(b, cfg)
    assert node_depth["obs_rm"] == 23 and node_depth["td_avg"] == 11, node_depth
    np.testing.assert_array_equal(r_merged, r_nd)


def test_group_mode_same_launches_same_bits(gpu, monkeypatch):
    """Group mode swaps kernels on big uniform levels; the launch count and the
    iterates are unchanged."""
    from conftest import bundle
    b = bundle("goof4")
    cfg = SolverConfig("pcfr+")
    monkeypatch.setenv("SCFR_GROUP_NJ", "0")
    monkeypatch.setenv("SCFR_NO_SMALL_WARP", "1")  # Goofspiel-4's levels are small
    monkeypatch.setenv("SCFR_NO_LEAF_FUSE", "1")  # (needs group mode: would change the count)
    grouped, r_g = _launches(b, cfg)
    monkeypatch.setenv("SCFR_NO_GROUP", "1")
    plain, r_p = _launches(b, cfg)
    assert grouped == plain
    np.testing.assert_array_equal(r_g, r_p)


def test_batched_level_engine_group_and_bcur(gpu, monkeypatch):
    """A batch of PCFR+ alt solves on the level engine, group mode forced onto
    every eligible level: each solve equals the same solve run alone (the
    batch offsets of the group kernels and of bcur)."""
    from conftest import bundle
    monkeypatch.setenv("SCFR_GROUP_NJ", "0")
    monkeypatch.setenv("SCFR_NO_SMALL_WARP", "1")
    b = bundle("goof4")
    params = [(1.5, 0.0, 2.0), (1.5, 0.0, 1.0), (1.5, 0.0, 0.0)]
    s = Solver(b, SolverConfig("pcfr+"), engine="levels", batch_params=params)
    s.step(7)
    for k, (a, be, g) in enumerate(params):
        one = Solver(b, SolverConfig("pcfr+", alpha=a, beta=be, gamma=g), engine="levels")
        one.step(7)
        for pl in (1, 2):
            np.testing.assert_array_equal(s.regrets(pl, k), one.regrets(pl))
            np.testing.assert_array_equal(s.average(pl, k), one.average(pl))
        one.close()
    s.close()


def test_top_and_leaf_fusion(gpu, monkeypatch):
    """Top-down passes skip the top's launches (ancestor-chain x) and OBS
    computes the forced leaf level inside the level above: fewer launches,
    the same iterates bit for bit."""
    from conftest import bundle
    b = bundle("goof4")
    cfg = SolverConfig("pcfr+")
    monkeypatch.setenv("SCFR_GROUP_NJ", "0")
    monkeypatch.setenv("SCFR_NO_SMALL_WARP", "1")
    fused, r_f = _launches(b, cfg)
    monkeypatch.setenv("SCFR_NO_TOP", "1")
    monkeypatch.setenv("SCFR_NO_LEAF_FUSE", "1")
    plain, r_p = _launches(b, cfg)
    assert fused["td_avg"] < plain["td_avg"] and fused["cur"] < plain["cur"], (fused, plain)
    assert fused["obs"] == plain["obs"] - 2, (fused, plain)  # one leaf launch per observe pass
    assert fused["pred"] == plain["pred"]
    np.testing.assert_array_equal(r_f, r_p)
