"""The oracle's C compile step and fixture generators (oracle/seqcfr_tree.c)
against the reference: structure digests written by scripts/make_golden.py
and scripts/make_golden_goof5.py (both ran the reference), and the product's
Python generators on small sizes.  This is what lets bench.py's reference arm
build Goofspiel-5 without the product library."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, digest, golden_meta, make_game
from oracle import tree

PROC = ("kind", "depth", "parent", "node_seq", "seq_node", "dp_node", "dp_first_seq",
        "dp_num_actions", "dp_parent_seq", "level_starts", "game_seq")


def goof5_meta():
    with open(os.path.join(GOLDEN, "goof5_meta.json")) as fh:
        return json.load(fh)


def check_structure(info, b):
    for pl in (1, 2):
        p, meta = b.procs[pl - 1], info[f"p{pl}"]
        for key in ("num_nodes", "num_decisions", "num_seqs", "height", "degree"):
            assert getattr(p, key) == meta[key], (pl, key)
        for f, d in meta["digests"].items():
            assert digest(getattr(p, f)) == d, (pl, f)
    for tag, m in (("U", b.payoff), ("UT", b.payoff_t)):
        meta = info[tag]
        assert (m.rows, m.cols, m.nnz) == (meta["rows"], meta["cols"], meta["nnz"])
        for f, d in meta["digests"].items():
            assert digest(getattr(m, f)) == d, (tag, f)


@pytest.mark.parametrize("name", ["kuhn", "leduc", "mp", "rps", "random6", "random7", "liars3",
                                  "goof3", "liars6", "goof4"])
def test_oracle_c_compile_matches_reference(name):
    g = make_game(name)
    flat = g if hasattr(g, "child_ptr") else g.flatten()
    check_structure(golden_meta()["structure"][name], tree.compile_native(flat))


@pytest.mark.parametrize("name,size", [("liars_dice", 6), ("goofspiel", 4)])
def test_oracle_generators_match_reference(name, size):
    key = {"liars_dice": "liars", "goofspiel": "goof"}[name] + str(size)
    check_structure(golden_meta()["structure"][key], tree.native_bundle(name, size))


def test_oracle_goofspiel5_matches_reference():
    """The bench workload, built product-free, equals the reference's bundle."""
    check_structure(goof5_meta()["structure"]["goof5"], tree.native_bundle("goofspiel", 5))


@pytest.mark.parametrize("name,size", [("goofspiel", 1), ("goofspiel", 2), ("goofspiel", 3),
                                       ("liars_dice", 2), ("liars_dice", 3)])
def test_oracle_generators_match_python(name, size):
    from paper_2605_14277_b200 import games as G
    a = tree.native_game(name, size)
    b = getattr(G, name)(size).flatten().canonical()
    for f in ("kind", "parent", "child_ptr", "child_idx", "player", "infoset"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    np.testing.assert_array_equal(a.prob, b.prob)
    np.testing.assert_array_equal(a.payoff, b.payoff)


@pytest.mark.parametrize("args", [(5, 2, 0.0, 3), (6, 3, 0.7, 11), (3, 5, 1.0, 2)])
def test_oracle_c_and_python_compile_agree(args):
    from paper_2605_14277_b200 import games as G
    flat = G.random_game(*args).flatten()
    a, b = tree.compile_native(flat), tree.compile_flat(flat)
    for pl in (0, 1):
        for f in PROC:
            np.testing.assert_array_equal(getattr(a.procs[pl], f), getattr(b.procs[pl], f))
    for m, o in ((a.payoff, b.payoff), (a.payoff_t, b.payoff_t)):
        for f in ("indptr", "indices", "data"):
            np.testing.assert_array_equal(getattr(m, f), getattr(o, f))


def test_oracle_compile_rejects_perfect_recall_violation():
    from paper_2605_14277_b200 import games as G
    b = G.GameBuilder("forget")
    d = b.decision(None, None, 1, "x")
    for a in ("l", "r"):
        d2 = b.decision(d, a, 1, "y")
        b.terminal(d2, "u", 1.0)
        b.terminal(d2, "v", 0.0)
    with pytest.raises(ValueError):
        tree.compile_native(b.build().flatten())
