"""Convergence records and profile metrics (reference pkg/metrics.py).

``exploitability`` / ``best_response_values`` / ``expected_value`` take host
profiles like the reference's and evaluate them on the device through the
bundle's cached evaluator handle (best response = the bottom-up pass with a
max, csrc/kernels.cuh:br_dp), bit-identical to pkg/metrics.py:50-75.
"""

from __future__ import annotations

import csv
import io
from dataclasses import dataclass

CSV_HEADER = ("iteration", "seconds", "exploitability", "current_exploitability", "work",
              "peak_bytes")


@dataclass
class ConvergenceRecord:
    iteration: int
    seconds: float
    exploitability: float
    current_exploitability: float
    work: int
    peak_bytes: int

    def row(self) -> list:
        return [self.iteration, repr(self.seconds), repr(self.exploitability),
                repr(self.current_exploitability), self.work, self.peak_bytes]


def records_to_csv(records) -> str:
    out = io.StringIO()
    w = csv.writer(out, lineterminator="\n")
    w.writerow(CSV_HEADER)
    for rec in records:
        w.writerow(rec.row())
    return out.getvalue()


def best_response_values(bundle, x1, x2, backend=None) -> tuple[float, float]:
    from .solvers import evaluator
    del backend
    return evaluator(bundle).best_response_values(x1, x2)


def exploitability(bundle, x1, x2, backend=None) -> float:
    b1, b2 = best_response_values(bundle, x1, x2)
    return (b1 + b2) / 2.0


def expected_value(bundle, x1, x2, backend=None) -> float:
    """x1 . (U x2).  Takes the bundle (the device evaluator needs it); the
    reference takes the payoff matrix (pkg/metrics.py:50-56)."""
    from .solvers import evaluator
    del backend
    if len(x1) != bundle.payoff.rows:
        raise ValueError("dimension mismatch: x1 does not match the payoff rows")
    return evaluator(bundle).expected_value_of(x1, x2)
