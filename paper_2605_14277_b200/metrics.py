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


def expected_value(payoff, x1, x2, backend=None) -> float:
    """x1 . (U x2) (pkg/metrics.py:50-56).  ``payoff`` is the bundle's payoff
    matrix, as in the reference, or the bundle itself; the product runs on the
    device evaluator of the bundle that owns the matrix."""
    from .compiler import CsrMatrix
    from .solvers import evaluator
    del backend
    bundle = payoff
    if isinstance(payoff, CsrMatrix):
        bundle = payoff._bundle() if payoff._bundle is not None else None
        if bundle is None or bundle.payoff is not payoff:
            raise ValueError("expected_value needs the payoff matrix of a live GameBundle")
    if len(x1) != bundle.payoff.rows:
        raise ValueError("dimension mismatch: x1 does not match the payoff rows")
    return evaluator(bundle).expected_value_of(x1, x2)
