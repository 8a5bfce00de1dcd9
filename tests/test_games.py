"""Game model: generators emit the reference's exact trees (golden text
digests from scripts/make_golden.py), the JSON-lines format round-trips, and
validation rejects broken trees (reference pkg/games.py)."""

import hashlib

import numpy as np
import pytest

from conftest import golden_meta, make_game
from paper_2605_14277_b200 import games as G


@pytest.mark.parametrize("name", ["kuhn", "leduc", "mp", "rps", "random6", "random7",
                                  "liars3", "goof3"])
def test_generator_text_matches_reference(name):
    text = G.save_game(make_game(name))
    want = golden_meta()["structure"][name]["game_text_sha256"]
    assert hashlib.sha256(text.encode()).hexdigest() == want


def test_known_sizes():
    # SPEC.md:51-52 (Kuhn), PAPER.md:484-487 (Leduc, Liar's dice)
    k = G.kuhn_poker()
    assert k.num_nodes == 58 and len(k.terminal_ids()) == 30
    assert G.leduc_poker().num_nodes == 9457
    ld = G.liars_dice(6)
    assert ld.num_nodes == 294883 and len(ld.terminal_ids()) == 147420


def test_roundtrip_and_validation():
    g = G.leduc_poker()
    again = G.load_game(G.save_game(g))
    assert G.save_game(again) == G.save_game(g)
    assert G.validate_game(g).ok


def test_flatten_matches_game():
    g = G.kuhn_poker()
    f = g.flatten()
    assert f.num_nodes == g.num_nodes
    np.testing.assert_array_equal(f.chance_reach(), g.chance_reach())
    for i, nd in enumerate(g.nodes):
        kids = f.child_idx[f.child_ptr[i]:f.child_ptr[i + 1]].tolist()
        assert kids == nd.children


def test_validation_errors():
    b = G.GameBuilder("bad")
    root = b.chance()
    b.terminal(root, "a", 1.0, prob=0.5)
    b.terminal(root, "b", 1.0, prob=0.25)
    rep = G.validate_game(b.build())
    assert not rep.ok and "sum to" in rep.message
    # perfect recall: P1 forgets its own first action
    b = G.GameBuilder("forget")
    d = b.decision(None, None, 1, "x")
    for a in ("l", "r"):
        d2 = b.decision(d, a, 1, "y")
        b.terminal(d2, "u", 1.0)
        b.terminal(d2, "v", 0.0)
    rep = G.validate_game(b.build())
    assert not rep.ok and "perfect recall" in rep.message


def test_parse_errors():
    with pytest.raises(G.GameParseError):
        G.load_game("")
    with pytest.raises(G.GameParseError):
        G.load_game('{"players": 3, "name": "x"}\n')
    with pytest.raises(G.GameParseError):
        G.load_game('{"players": 2, "name": "x"}\n{"id": 0, "kind": "nope", "parent": null, '
                    '"label_from_parent": null}\n')


def test_random_game_budget():
    with pytest.raises(G.GameSizeError):
        G.random_game(30, 3)
