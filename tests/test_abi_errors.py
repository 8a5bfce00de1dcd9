"""Error behaviour of the C-ABI through the host mirror: the reference's
exception classes (ValueError for bad arguments, FloatingPointError for
non-finite values; pkg/solvers.py:62-75, :154-155) and loud failures instead
of silent fallbacks."""

import ctypes as C

import numpy as np
import pytest

from conftest import bundle
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, native

pytestmark = pytest.mark.gpu


def _raw_create(b, cfg, p1=None, p2=None, U=None, UT=None):
    L = native.lib()
    c1, c2, cu, cut = b._c
    h = C.c_void_p()
    return L.scfr_create(C.byref(p1 or c1), C.byref(p2 or c2), C.byref(U or cu), C.byref(UT or cut),
                         C.byref(cfg), 0, C.byref(h)), h


def _cfg(**kw):
    cfg = native.Config()
    cfg.variant, cfg.mode, cfg.batch = 0, 0, 1
    cfg.alpha, cfg.beta, cfg.gamma = 1.5, 0.0, 0.0
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


def test_bad_config_values(gpu):
    b = bundle("kuhn")
    for kw in ({"variant": 9}, {"mode": 3}, {"batch": 0}, {"engine": 42}, {"dtype": 7}, {"gamma": -1.0},
               {"alpha": float("nan")}):
        rc, _ = _raw_create(b, _cfg(**kw))
        assert rc == native.EINVAL, kw
        assert native.lib().scfr_last_error()


def test_dimension_mismatch(gpu):
    kuhn, leduc = bundle("kuhn"), bundle("leduc")
    rc, _ = _raw_create(kuhn, _cfg(), U=leduc._c[2])
    assert rc == native.EINVAL
    assert b"dimension" in native.lib().scfr_last_error()


def test_corrupt_decision_process_rejected(gpu):
    b = bundle("leduc")
    p = b.procs[0]
    bad = np.array(p.dp_first_seq, dtype=np.int64)
    bad[5] += 1  # not contiguous in j
    t = p.as_c()
    t.dp_first_seq = bad.ctypes.data_as(C.POINTER(C.c_int64))
    rc, _ = _raw_create(b, _cfg(), p1=t)
    assert rc == native.EINVAL
    assert b"contiguous" in native.lib().scfr_last_error()
    par = np.array(p.dp_parent_seq, dtype=np.int64)
    par[7] = p.num_seqs + 3  # parent after its decision point
    t = p.as_c()
    t.dp_parent_seq = par.ctypes.data_as(C.POINTER(C.c_int64))
    rc, _ = _raw_create(b, _cfg(), p1=t)
    assert rc == native.EINVAL


def test_depth_order_and_child_groups_rejected(gpu):
    """The fused validation pass (upload_player): DPs out of depth order, and
    a parent sequence whose child DPs do not form one contiguous group."""
    b = bundle("leduc")
    p = b.procs[0]
    dpn = np.asarray(p.dp_node)
    depth = np.array(p.depth, dtype=np.int64)
    dd = depth[dpn]
    j = int(np.flatnonzero(np.diff(dd) > 0)[-1]) + 1  # first DP of the deepest level
    depth[dpn[j]] = 10_000  # deeper than the DPs after it
    t = p.as_c()
    t.depth = depth.ctypes.data_as(C.POINTER(C.c_int64))
    rc, _ = _raw_create(b, _cfg(), p1=t)
    assert rc == native.EINVAL
    assert b"ordered by depth" in native.lib().scfr_last_error()
    par = np.array(p.dp_parent_seq, dtype=np.int64)
    # DPs a, b, c where a and c share a parent and b's differs: give c a's parent
    ps = par.tolist()
    k = next(i for i in range(2, len(ps)) if ps[i - 2] != ps[i - 1] and ps[i - 1] != ps[i] and ps[i - 2] < ps[i])
    par[k] = par[k - 2]
    t = p.as_c()
    t.dp_parent_seq = par.ctypes.data_as(C.POINTER(C.c_int64))
    rc, _ = _raw_create(b, _cfg(), p1=t)
    assert rc == native.EINVAL
    assert b"not contiguous" in native.lib().scfr_last_error()


def test_bad_column_index_rejected(gpu):
    b = bundle("kuhn")
    U = b.payoff
    ix = np.array(U.indices, dtype=np.int64)
    ix[0] = U.cols + 5
    cu = U.as_c()
    cu.indices = ix.ctypes.data_as(C.POINTER(C.c_int64))
    rc, _ = _raw_create(b, _cfg(), U=cu)
    assert rc == native.EINVAL
    assert b"column" in native.lib().scfr_last_error()


def test_engine_constraints(gpu):
    b = bundle("leduc")
    with pytest.raises(ValueError):
        Solver(b, SolverConfig("cfr"), device=gpu, batch_params=[(1.5, 0, 2)] * 2, engine="persistent_grid")
    with pytest.raises(ValueError):
        Solver(bundle("kuhn"), SolverConfig("cfr"), device=gpu, engine="tiled")  # player 2 has one level
    with pytest.raises(ValueError):
        Solver(b, SolverConfig("cfr"), device=10_000)


def test_read_arguments(gpu):
    s = Solver(bundle("kuhn"), SolverConfig("cfr"), device=gpu)
    with pytest.raises(ValueError):
        s.average(1)  # nothing accumulated yet (the reference divides by zero weight)
    s.step(3)
    with pytest.raises(ValueError):
        s.average(3)
    with pytest.raises(ValueError):
        s.average(1, solve=1)
    with pytest.raises(ValueError):
        s.best_response_values(np.zeros(4), np.zeros(13))
    with pytest.raises(ValueError):
        s.snapshot(restore=True)  # none saved
    assert s.exploitability()[0] > 0


def test_nonfinite_payoffs_raise_floating_point_error(gpu):
    from paper_2605_14277_b200 import games as G
    g = G.GameBuilder("inf")
    top = g.decision(None, None, 1, "p1")
    for a in ("H", "T"):
        sub = g.decision(top, a, 2, "p2")
        for b_ in ("H", "T"):
            g.terminal(sub, b_, 1.7e308 if a == "H" else -1.7e308)
    for dtype in ("f64", "f32"):  # fp32 overflows at once: the payoffs round to inf
        s = Solver(GameBundle(g.build()), SolverConfig("cfr"), device=gpu, dtype=dtype)
        s.step(8)
        with pytest.raises(FloatingPointError):
            s.check_finite()


def test_transposed_payoff_checked(gpu):
    """Uᵀ is derived on the device from U (transpose.cu); a caller's Uᵀ that
    is not U's transpose is rejected, not silently replaced."""
    b = bundle("leduc")
    UT = b._c[3]
    data = np.ctypeslib.as_array(UT.data, shape=(UT.nnz,)).copy()
    data[0] += 1.0  # one entry off (entry 0 is always probed)
    bad = native.Csr()
    C.memmove(C.byref(bad), C.byref(UT), C.sizeof(native.Csr))
    bad.data = data.ctypes.data_as(C.POINTER(C.c_double))
    rc, _ = _raw_create(b, _cfg(), UT=bad)
    assert rc == native.EINVAL
    assert b"transpose" in native.lib().scfr_last_error()


def test_device_transpose_matches_host_upload(gpu, monkeypatch):
    """Same iterates with the device-derived Uᵀ and with the caller's Uᵀ
    uploaded (SCFR_HOST_UT=1), on a game with duplicate payoff cells."""
    for name, variant in (("random6", "cfr"), ("liars3", "dcfr"), ("leduc", "pcfr+")):
        b = bundle(name)
        out = []
        for env in ("0", "1"):
            monkeypatch.setenv("SCFR_HOST_UT", env)
            s = Solver(b, SolverConfig(variant), engine="levels")
            s.step(7)
            out.append((s.average(1), s.average(2), s.current(1), s.current(2)))
            s.close()
        for a, c in zip(*out):
            assert np.array_equal(a.view(np.uint64), c.view(np.uint64)), name
