"""bench.py's SURVEY §8(d) byte model against the survey's own table of
fp64 bytes per iteration."""

import pytest

import bench
from paper_2605_14277_b200 import SolverConfig


@pytest.mark.parametrize("kind,cfg,expected", [
    ("kuhn", SolverConfig("cfr"), 3_616),
    ("leduc", SolverConfig("cfr+"), 404_040),
    ("liars", SolverConfig("dcfr", gamma=2.0), 9_779_208),
    ("goof", SolverConfig("pcfr+"), 1_041_361_716),
    ("goof", SolverConfig("cfr", mode="sim"), 714_485_432),
])
def test_survey_bytes_per_iteration(kind, cfg, expected):
    assert bench.survey_step_bytes(bench.make_bundle(kind), cfg) == expected
