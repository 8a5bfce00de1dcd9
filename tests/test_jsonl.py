"""Native JSON-lines game reader (csrc/jsonl.cpp) against the
Python path games.load_game + FlatGame.from_game: the same flat arrays and
labels, the same compiled structure, and the same errors (class, message,
line / node) on corrupted files.  Host-only: runs without a GPU."""

import json

import numpy as np
import pytest

from conftest import digest
from paper_2605_14277_b200 import games as G
from paper_2605_14277_b200.compiler import GameBundle, load_game_flat

GAMES = {
    "kuhn": G.kuhn_poker, "leduc": G.leduc_poker, "mp": G.matching_pennies, "rps": G.rock_paper_scissors,
    "random7": lambda: G.random_game(7, 3, 0.3, 7), "random6": lambda: G.random_game(6, 3, 0.5, 1),
    "liars3": lambda: G.liars_dice(3), "goof3": lambda: G.goofspiel(3),
}


@pytest.mark.parametrize("name", sorted(GAMES))
def test_native_reader_matches_python_path(name):
    text = G.save_game(GAMES[name]())
    want = G.FlatGame.from_game(G.load_game(text))
    got = load_game_flat(text)
    assert got.name == want.name
    for f in ("kind", "parent", "child_ptr", "child_idx", "player", "infoset", "prob", "payoff"):
        np.testing.assert_array_equal(getattr(got, f), getattr(want, f), err_msg=f)
    assert got.infoset_labels == want.infoset_labels
    assert got.action_labels == want.action_labels


@pytest.mark.parametrize("name", ["kuhn", "leduc", "random6", "liars3"])
def test_native_reader_compiles_to_the_same_structure(name):
    text = G.save_game(GAMES[name]())
    a = GameBundle(G.load_game(text))
    b = GameBundle(load_game_flat(text))
    for pa, pb in zip(a.procs, b.procs):
        for f in ("dp_first_seq", "dp_num_actions", "dp_parent_seq", "level_starts", "game_seq"):
            assert digest(getattr(pa, f)) == digest(getattr(pb, f)), f
    for ma, mb in ((a.payoff, b.payoff), (a.payoff_t, b.payoff_t)):
        for f in ("indptr", "indices", "data"):
            assert digest(getattr(ma, f)) == digest(getattr(mb, f)), f
    assert a.procs[0].seq_label(3) == b.procs[0].seq_label(3)


def _kuhn_lines():
    return G.save_game(G.kuhn_poker()).splitlines()


def _edit(fn):
    lines = _kuhn_lines()
    fn(lines)
    return "\n".join(lines) + "\n"


def _set(i, **kw):
    def fn(lines):
        obj = json.loads(lines[i])
        for k, v in kw.items():
            if v is _DEL:
                obj.pop(k, None)
            else:
                obj[k] = v
        lines[i] = json.dumps(obj)
    return fn


_DEL = object()

CORRUPT = {
    "empty": lambda: "",
    "not_object": lambda: _edit(lambda ls: ls.__setitem__(3, "[1, 2]")),
    "bad_header": lambda: _edit(lambda ls: ls.__setitem__(0, json.dumps({"players": 2}))),
    "three_players": lambda: _edit(lambda ls: ls.__setitem__(0, json.dumps({"players": 3, "name": "x"}))),
    "unknown_field": lambda: _edit(_set(5, color="red")),
    "missing_field": lambda: _edit(_set(5, kind=_DEL)),
    "bad_id": lambda: _edit(_set(5, id=-3)),
    "duplicate_id": lambda: _edit(_set(6, id=4)),
    "sparse_ids": lambda: _edit(lambda ls: ls.pop(7)),
    "unknown_kind": lambda: _edit(_set(5, kind="oracle")),
    "root_parent": lambda: _edit(_set(1, parent=3)),
    "parent_type": lambda: _edit(_set(5, parent="3")),
    "parent_range": lambda: _edit(_set(5, parent=999)),
    "field_type": lambda: _edit(_set(5, infoset=7)),
    "self_parent": lambda: _edit(_set(5, parent=4)),
    "cycle": lambda: _edit(lambda ls: (_set(5, parent=6)(ls), _set(6, parent=5)(ls))),
    "dup_labels": lambda: _edit(_set(6, label_from_parent=json.loads(_kuhn_lines()[5])["label_from_parent"])),
    "terminal_no_payoff": lambda: _edit(_set(next(i for i, l in enumerate(_kuhn_lines()) if '"terminal"' in l),
                                           payoff=_DEL)),
    "chance_sum": lambda: _edit(_set(2, prob=0.5)),
    "prob_on_decision_child": lambda: _edit(_set(next(i for i, l in enumerate(_kuhn_lines()) if '"terminal"' in l),
                                               prob=0.3)),
    "decision_player": lambda: _edit(_set(next(i for i, l in enumerate(_kuhn_lines()) if '"decision"' in l),
                                        player=5)),
    "infoset_two_players": lambda: _edit(_set(next(i for i, l in enumerate(_kuhn_lines())
                                                   if '"player": 2' in l), infoset="0|")),
    "invalid_json": lambda: _edit(lambda ls: ls.__setitem__(4, ls[4][:-1])),
}


@pytest.mark.parametrize("case", sorted(CORRUPT))
def test_native_reader_errors_match_python_path(case):
    text = CORRUPT[case]()
    with pytest.raises(G.GameError) as py:
        G.load_game(text)
    with pytest.raises(G.GameError) as nat:
        load_game_flat(text)
    assert type(nat.value) is type(py.value), (case, py.value, nat.value)
    if isinstance(py.value, G.GameParseError):
        assert nat.value.line == py.value.line, (case, py.value, nat.value)
        if "invalid JSON" not in str(py.value):  # (the JSON decoder's own wording differs)
            assert str(nat.value) == str(py.value), case
    else:
        assert nat.value.node_id == py.value.node_id and str(nat.value) == str(py.value), (case, py.value, nat.value)
