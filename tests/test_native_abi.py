"""The C-ABI library loads on CPU and exports every entry point declared in
include/seqcfr_b200.h; host-only logic (schedules, work counter, peak bytes)
matches the reference."""

import ctypes
import math
import os
import re

import pytest

from conftest import ROOT, bundle, cuda_available, golden_meta
from paper_2605_14277_b200 import native
from paper_2605_14277_b200.solvers import SolverConfig, discount_factors, work_per_iteration


def _declared():
    text = open(os.path.join(ROOT, "include", "seqcfr_b200.h")).read()
    return sorted(set(re.findall(r"\b(scfr_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(native.LIB_PATH)
    names = _declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert set(native.EXPORTED) <= set(names)
    assert native.lib().scfr_abi_version() == 1


@pytest.mark.skipif(cuda_available(), reason="checks the no-device error path")
def test_create_fails_loudly_without_device():
    from paper_2605_14277_b200.solvers import Solver
    with pytest.raises(native.CudaError):
        Solver(bundle("kuhn"), SolverConfig("cfr"))


def test_work_per_iteration_matches_reference():
    for key, rec in golden_meta()["lockstep"].items():
        cfg = SolverConfig(rec["variant"], alpha=rec["alpha"], beta=rec["beta"],
                           gamma=rec["gamma"], mode=rec["mode"])
        assert work_per_iteration(bundle(rec["game"]), cfg) == rec["work_per_iter"], key
    run = golden_meta()["runs"]["kuhn.cfr.1000"]
    assert run["records"][0]["work"] == 657


def test_peak_bytes_matches_reference():
    for key, run in golden_meta()["runs"].items():
        b = bundle(run["game"])
        assert b.reference_nbytes() + b.reference_state_bytes() == run["records"][0]["peak_bytes"]


def test_discount_factors_reference_semantics():
    # t=1, alpha=1.5, beta=0 -> both factors 0.5
    assert discount_factors(1, 1.5, 0.0) == (0.5, 0.5)
    pf, nf = discount_factors(10, 1.5, 0.0)
    assert pf == 10.0 ** 1.5 / (10.0 ** 1.5 + 1.0) and nf == 0.5


def test_config_validation():
    with pytest.raises(ValueError):
        SolverConfig("nope")
    with pytest.raises(ValueError):
        SolverConfig("dcfr", alpha=math.inf)
    with pytest.raises(ValueError):
        SolverConfig("cfr", gamma=-1.0)
    assert SolverConfig("pcfr+").gamma == 2.0 and SolverConfig("pcfr+").mode == "alt"
