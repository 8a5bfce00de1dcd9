"""Tree compiler: the native compiler (csrc/compiler.cpp through
scfr_compile) and the oracle's Python restatement (oracle/tree.py) both
reproduce the reference DecisionProcess / payoff CSR arrays bit for bit
(golden digests and full arrays from the reference), and agree with each
other on games outside the golden set."""

import numpy as np
import pytest

from conftest import bundle, digest, golden_arrays, golden_meta, make_game, oracle_bundle
from paper_2605_14277_b200 import games as G
from paper_2605_14277_b200.compiler import GameBundle, flat_goofspiel, flat_liars_dice

NAMES = ["kuhn", "leduc", "mp", "rps", "random6", "random7", "liars3", "goof3", "liars6", "goof4"]
PROC = ("kind", "depth", "parent", "node_seq", "seq_node", "dp_node", "dp_first_seq",
        "dp_num_actions", "dp_parent_seq", "level_starts", "game_seq")


def _check_structure(name, b):
    info = golden_meta()["structure"][name]
    for pl in (1, 2):
        p = b.procs[pl - 1]
        meta = info[f"p{pl}"]
        for key in ("num_nodes", "num_decisions", "num_seqs", "height", "degree"):
            assert getattr(p, key) == meta[key], (name, pl, key)
        for f, d in meta["digests"].items():
            assert digest(getattr(p, f)) == d, (name, pl, f)
    for tag, m in (("U", b.payoff), ("UT", b.payoff_t)):
        meta = info[tag]
        assert (m.rows, m.cols, m.nnz) == (meta["rows"], meta["cols"], meta["nnz"])
        for f, d in meta["digests"].items():
            assert digest(getattr(m, f)) == d, (name, tag, f)


@pytest.mark.parametrize("name", NAMES)
def test_native_compiler_matches_reference(name):
    b = bundle(name)
    _check_structure(name, b)
    assert b.reference_nbytes() == golden_meta()["structure"][name]["bundle_nbytes"]


@pytest.mark.parametrize("name", ["kuhn", "leduc", "random6", "goof3"])
def test_native_compiler_full_arrays(name):
    arr = golden_arrays()
    b = bundle(name)
    for pl in (1, 2):
        for f in PROC:
            np.testing.assert_array_equal(getattr(b.procs[pl - 1], f), arr[f"{name}.p{pl}.{f}"])
    np.testing.assert_array_equal(b.payoff.data, arr[f"{name}.U.data"])
    np.testing.assert_array_equal(b.payoff_t.indices, arr[f"{name}.UT.indices"])


@pytest.mark.parametrize("name", ["kuhn", "leduc", "random6", "random7", "liars3", "goof3"])
def test_oracle_compiler_matches_reference(name):
    _check_structure(name, oracle_bundle(name))


@pytest.mark.parametrize("args", [(5, 2, 0.0, 3), (6, 3, 0.7, 11), (8, 2, 0.5, 5), (3, 5, 1.0, 2)])
def test_native_vs_oracle_compiler_random(args):
    g = G.random_game(*args)
    nb = GameBundle(g)
    from oracle import tree
    ob = tree.compile_flat(g.flatten())
    for pl in (0, 1):
        for f in PROC:
            np.testing.assert_array_equal(getattr(nb.procs[pl], f), getattr(ob.procs[pl], f))
    for m, o in ((nb.payoff, ob.payoff), (nb.payoff_t, ob.payoff_t)):
        np.testing.assert_array_equal(m.indptr, o.indptr)
        np.testing.assert_array_equal(m.indices, o.indices)
        np.testing.assert_array_equal(m.data, o.data)


@pytest.mark.parametrize("size", [1, 2, 3, 4])
def test_native_generators_match_python(size):
    for native, py in ((flat_liars_dice, G.liars_dice), (flat_goofspiel, G.goofspiel)):
        a, b = native(size), py(size).flatten().canonical()
        for f in ("kind", "parent", "child_ptr", "child_idx", "player", "infoset"):
            np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
        np.testing.assert_array_equal(a.prob, b.prob)
        np.testing.assert_array_equal(a.payoff, b.payoff)


def test_goofspiel5_matches_reference():
    """The bench workload: every structure array of the native compile equals
    the reference's own GameBundle (digests by scripts/make_golden_goof5.py)."""
    import json
    import os
    from conftest import GOLDEN
    with open(os.path.join(GOLDEN, "goof5_meta.json")) as fh:
        info = json.load(fh)["structure"]["goof5"]
    flat = flat_goofspiel(5)
    assert flat.num_nodes == info["num_game_nodes"] == 8_530_656
    b = GameBundle(flat)
    for p in b.procs:
        assert (p.num_nodes, p.num_seqs, p.num_decisions) == (4_850_531, 2_666_026, 2_184_505)
    assert b.payoff.nnz == 1_728_000
    for pl in (1, 2):
        for f, d in info[f"p{pl}"]["digests"].items():
            assert digest(getattr(b.procs[pl - 1], f)) == d, (pl, f)
    for tag, m in (("U", b.payoff), ("UT", b.payoff_t)):
        for f, d in info[tag]["digests"].items():
            assert digest(getattr(m, f)) == d, (tag, f)
    assert b.reference_nbytes() == info["bundle_nbytes"]


def test_perfect_recall_violation_is_rejected():
    b = G.GameBuilder("forget")
    d = b.decision(None, None, 1, "x")
    for a in ("l", "r"):
        d2 = b.decision(d, a, 1, "y")
        b.terminal(d2, "u", 1.0)
        b.terminal(d2, "v", 0.0)
    with pytest.raises(G.GameValidationError):
        GameBundle(b.build(), validate=False)


def test_labels_and_dump():
    b = bundle("kuhn")
    p = b.procs[0]
    assert p.seq_label(0) == ""
    assert p.seq_label(1) == f"{p.dp_label[0]}/{p.dp_action_labels[0][0]}"
    assert p.dump().count("\n") == p.num_nodes - 1
    np.testing.assert_array_equal(p.uniform_behavior(), np.repeat(1.0 / p.dp_num_actions,
                                                                  p.dp_num_actions))
