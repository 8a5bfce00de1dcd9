"""CLI drop-in (pkg/cli.py): parser, exit codes, checkpoint defaults and the
strategy-file writer on CPU; a full `solve` through the GPU against the
reference's own convergence records."""

import csv
import io
import json

import numpy as np
import pytest

from conftest import golden_meta
from paper_2605_14277_b200 import cli
from paper_2605_14277_b200.compiler import GameBundle
from paper_2605_14277_b200.games import kuhn_poker


def test_checkpoint_defaults():
    # np.geomspace(1, n, 12) truncated and uniqued, as pkg/cli.py:80-82
    assert cli.parse_checkpoints(None, 1000) == [1, 3, 6, 12, 23, 43, 81, 151, 284, 533, 1000]
    assert cli.parse_checkpoints("30, 10,10", 5) == [10, 30]
    assert cli.parse_checkpoints(None, None)[:3] == [1, 2, 4]
    with pytest.raises(cli.UsageError):
        cli.parse_checkpoints("0,3", None)
    with pytest.raises(cli.UsageError):
        cli.parse_checkpoints("a", None)


def test_exit_codes(capsys):
    assert cli.main(["info", "--game", "no_such_game"]) == cli.EXIT_DATA
    assert cli.main(["solve", "--game", "kuhn"]) == cli.EXIT_USAGE          # no budget
    assert cli.main(["solve", "--game", "kuhn", "--iters", "0"]) == cli.EXIT_USAGE
    assert cli.main(["solve", "--game", "kuhn", "--backend", "serial", "--iters", "3"]) == cli.EXIT_USAGE
    assert cli.main(["bench", "--sizes", "100", "--backends", "parallel"]) == cli.EXIT_USAGE
    assert cli.main(["bench", "--sizes", "100", "--measure", "3"]) == cli.EXIT_USAGE
    assert cli.main(["info", "--game", "random:depth=3"]) == cli.EXIT_USAGE  # spec misses branching
    assert cli.main(["--help"]) == cli.EXIT_OK
    capsys.readouterr()


def test_info_kuhn(capsys):
    assert cli.main(["info", "--game", "kuhn"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[1:] == ["game tree nodes: 58", "terminal nodes: 30",
                       "player 1: nodes=16 decision_points=6 sequences=13 height=3 degree=3",
                       "player 2: nodes=19 decision_points=6 sequences=13 height=2 degree=6"]


def test_strategy_lines_uniform_fallback():
    b = GameBundle(kuhn_poker())
    p = b.procs[0]
    x = np.zeros(p.num_seqs)
    x[0] = 1.0
    lines = [json.loads(s) for s in cli.behavioral_lines(p, x, 1)]
    assert len(lines) == p.num_seqs - 1
    # the root DPs have parent mass 1 and x = 0 -> prob 0; unreached DPs are uniform
    for j in range(p.num_decisions):
        first, n = int(p.dp_first_seq[j]), int(p.dp_num_actions[j])
        probs = [lines[first - 1 + a]["prob"] for a in range(n)]
        if int(p.dp_parent_seq[j]) == 0:
            assert probs == [0.0] * n
        else:
            assert probs == [1.0 / n] * n
    assert all(rec["player"] == 1 and rec["sequence"] for rec in lines)


@pytest.mark.gpu
def test_solve_matches_reference_records(gpu, tmp_path, capsys):
    want = golden_meta()["runs"]["kuhn.cfr.1000"]
    out = tmp_path / "solve.csv"
    rc = cli.main(["solve", "--game", "kuhn", "--variant", "cfr", "--iters", "1000",
                   "--checkpoints", ",".join(map(str, want["checkpoints"])), "--out", str(out)])
    assert rc == 0
    rows = list(csv.DictReader(io.StringIO(out.read_text())))
    assert [int(r["iteration"]) for r in rows] == want["checkpoints"]
    for r, w in zip(rows, want["records"]):
        assert float(r["exploitability"]) == w["exploitability"]
        assert float(r["current_exploitability"]) == w["current_exploitability"]
        assert int(r["work"]) == w["work"] and int(r["peak_bytes"]) == w["peak_bytes"]
    strat = [json.loads(s) for s in (tmp_path / "solve.strategy.jsonl").read_text().splitlines()]
    assert len(strat) == 24
    assert "exploitability=7.269106e-03" in capsys.readouterr().out


def test_info_from_a_game_file_matches_builtin(tmp_path, capsys):
    """A JSON-lines file goes through the native reader (csrc/jsonl.cpp)."""
    from paper_2605_14277_b200.games import save_game
    path = tmp_path / "kuhn.jsonl"
    path.write_text(save_game(kuhn_poker()))
    assert cli.main(["info", "--game", "kuhn"]) == 0
    want = capsys.readouterr().out
    assert cli.main(["info", "--game", str(path)]) == 0
    assert capsys.readouterr().out == want
    bad = tmp_path / "bad.jsonl"
    bad.write_text(path.read_text().replace('"prob": 0.5', '"prob": 0.25', 1))
    assert cli.main(["info", "--game", str(bad)]) == cli.EXIT_DATA
