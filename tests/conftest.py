"""Shared fixtures: golden reference data, game makers, GPU gating."""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100) device")
    config.addinivalue_line("markers", "slow: long-running case")


def digest(a) -> str:
    """Same digest as scripts/make_golden.py."""
    a = np.asarray(a)
    a = a.astype("<i8") if a.dtype.kind in "iub" else a.astype("<f8")
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


_META = None
_ARR = None


def golden_meta() -> dict:
    global _META
    if _META is None:
        with open(os.path.join(GOLDEN, "reference_meta.json")) as fh:
            _META = json.load(fh)
    return _META


def golden_arrays():
    global _ARR
    if _ARR is None:
        _ARR = np.load(os.path.join(GOLDEN, "reference_arrays.npz"))
    return _ARR


def make_game(name: str):
    """Fixture games by golden name (Game objects, or FlatGame for the big ones)."""
    from paper_2605_14277_b200 import games as G
    from paper_2605_14277_b200.compiler import flat_goofspiel, flat_liars_dice
    table = {
        "kuhn": G.kuhn_poker, "leduc": G.leduc_poker, "mp": G.matching_pennies,
        "rps": G.rock_paper_scissors, "random6": lambda: G.random_game(6, 3, 0.5, 1),
        "random7": lambda: G.random_game(7, 3, 0.3, 7), "liars3": lambda: G.liars_dice(3),
        "goof3": lambda: G.goofspiel(3), "liars6": lambda: flat_liars_dice(6),
        "goof4": lambda: flat_goofspiel(4),
    }
    return table[name]()


_BUNDLES: dict = {}


def bundle(name: str):
    from paper_2605_14277_b200.compiler import GameBundle
    if name not in _BUNDLES:
        _BUNDLES[name] = GameBundle(make_game(name))
    return _BUNDLES[name]


_OBUNDLES: dict = {}


def oracle_bundle(name: str):
    """Bundle compiled by the oracle's own Python restatement."""
    from oracle import tree
    from paper_2605_14277_b200.games import FlatGame
    if name not in _OBUNDLES:
        g = make_game(name)
        flat = g if isinstance(g, FlatGame) else g.flatten()
        _OBUNDLES[name] = tree.compile_flat(flat)
    return _OBUNDLES[name]


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def gpu():
    if not cuda_available():
        pytest.skip("no CUDA device")
    from paper_2605_14277_b200 import native
    native.lib()
    return 0
