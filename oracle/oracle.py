"""ctypes wrapper of the C oracle (TEST INFRASTRUCTURE — see seqcfr_oracle.c).

``OracleSolver`` runs the reference iteration (pkg/solvers.py:351-372) on the
CPU over reference-layout arrays (a compiled bundle from ``oracle.tree`` or
any object exposing ``procs`` with DecisionProcess fields and
``payoff``/``payoff_t`` CSR).  Vectors come back in the reference layout:
regrets/behaviour over Σ+ (``num_seqs-1``), strategies/averages over Σ.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libseqcfr_oracle.so")
LIB_PATH_F32 = os.path.join(HERE, "_build", "libseqcfr_oracle_f32.so")  # -DREAL=float build
VARIANTS = {"cfr": 0, "cfr+": 1, "dcfr": 2, "pcfr": 3, "pcfr+": 4}
_libs = {}


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib(dtype: str = "f64"):
    """The fp64 restatement, or (dtype "f32") the same source built with
    float state: the checker of the fp32 mode."""
    path = LIB_PATH_F32 if dtype in ("f32", "float32") else LIB_PATH
    if path not in _libs:
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        P = C.POINTER
        i64p = P(C.c_int64)
        f64p = P(C.c_double)
        L.oc_create.restype = C.c_void_p
        L.oc_create.argtypes = [i64p, i64p, i64p, P(i64p), P(i64p), P(i64p), P(i64p), P(i64p),
                                C.c_int64, i64p, i64p, f64p, i64p, i64p, f64p, C.c_int, C.c_int,
                                C.c_double, C.c_double, C.c_double, C.c_int]
        L.oc_step.argtypes = [C.c_void_p, C.c_int64]
        L.oc_read.argtypes = [C.c_void_p, C.c_int, C.c_int, f64p]
        L.oc_read.restype = C.c_double
        L.oc_t.argtypes = [C.c_void_p]
        L.oc_t.restype = C.c_int64
        L.oc_best_response.argtypes = [C.c_void_p, C.c_int, f64p]
        L.oc_best_response.restype = C.c_double
        L.oc_spmv.argtypes = [C.c_void_p, C.c_int, f64p, f64p, C.c_int]
        L.oc_free.argtypes = [C.c_void_p]
        _libs[path] = L
    return _libs[path]


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class OracleSolver:
    def __init__(self, bundle, variant="cfr", mode=None, alpha=1.5, beta=0.0, gamma=None,
                 threads: int = 1, dtype: str = "f64"):
        defaults = {"cfr": (0.0, "sim"), "cfr+": (1.0, "alt"), "dcfr": (2.0, "alt"),
                    "pcfr": (0.0, "sim"), "pcfr+": (2.0, "alt")}
        g0, m0 = defaults[variant]
        self.gamma = float(g0 if gamma is None else gamma)
        self.mode = m0 if mode is None else mode
        self.variant = variant
        self.threads = threads
        self.dtype = dtype
        L = self._L = lib(dtype)
        p1, p2 = bundle.procs
        keep = []
        arr = lambda *xs: (C.POINTER(C.c_int64) * 2)(*[_ptr(x, C.c_int64) for x in xs])  # noqa: E731
        fields = {}
        for f in ("depth", "dp_node", "dp_first_seq", "dp_num_actions", "dp_parent_seq"):
            a, b = _i64(getattr(p1, f)), _i64(getattr(p2, f))
            keep += [a, b]
            fields[f] = arr(a, b)
        nn = _i64([p1.num_nodes, p2.num_nodes])
        ns = _i64([p1.num_seqs, p2.num_seqs])
        nj = _i64([p1.num_decisions, p2.num_decisions])
        U, UT = bundle.payoff, bundle.payoff_t
        ui, ux, ud = _i64(U.indptr), _i64(U.indices), np.ascontiguousarray(U.data, np.float64)
        ti, tx, td = _i64(UT.indptr), _i64(UT.indices), np.ascontiguousarray(UT.data, np.float64)
        keep += [nn, ns, nj, ui, ux, ud, ti, tx, td]
        self._st = L.oc_create(
            _ptr(nn, C.c_int64), _ptr(ns, C.c_int64), _ptr(nj, C.c_int64), fields["depth"],
            fields["dp_node"], fields["dp_first_seq"], fields["dp_num_actions"],
            fields["dp_parent_seq"], len(ud), _ptr(ui, C.c_int64), _ptr(ux, C.c_int64),
            _ptr(ud, C.c_double), _ptr(ti, C.c_int64), _ptr(tx, C.c_int64), _ptr(td, C.c_double),
            VARIANTS[variant], 0 if self.mode == "sim" else 1, float(alpha), float(beta),
            self.gamma, int(threads))
        if not self._st:
            raise ValueError("oracle: decision-process arrays are not level-ordered")
        self.sizes = (p1.num_seqs, p2.num_seqs)

    def step(self, n: int = 1) -> None:
        self._L.oc_step(self._st, int(n))

    @property
    def t(self) -> int:
        return int(self._L.oc_t(self._st))

    def _read(self, player, which):
        out = np.empty(self.sizes[player - 1])
        w = self._L.oc_read(self._st, player, which, _ptr(out, C.c_double))
        return out, w

    def regrets(self, player):
        return self._read(player, 0)[0][1:]

    def behavior(self, player):
        return self._read(player, 1)[0][1:]

    def avg_accum(self, player):
        return self._read(player, 2)[0]

    def utility(self, player):
        return self._read(player, 3)[0]

    def current(self, player):
        return self._read(player, 4)[0]

    def average(self, player):
        acc, w = self._read(player, 2)
        return acc / w

    def best_response(self, player, x_opp):
        x = np.ascontiguousarray(x_opp, dtype=np.float64)
        return float(self._L.oc_best_response(self._st, player, _ptr(x, C.c_double)))

    def exploitability(self, x1, x2):
        b1 = self.best_response(1, x2)
        b2 = self.best_response(2, x1)
        return (b1 + b2) / 2.0, (b1, b2)

    def __del__(self):
        if getattr(self, "_st", None):
            self._L.oc_free(self._st)
            self._st = None
