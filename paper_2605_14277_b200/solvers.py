"""Solver API mirroring the reference (pkg/solvers.py), executed on the GPU.

Drop-in surface for the hot path:

* ``SolverConfig`` / ``VARIANTS`` / ``discount_factors``  pkg/solvers.py:35-94
* ``run(game|bundle, config, iterations, seconds, checkpoints, ...)``
                                                       pkg/solvers.py:375-438
* ``RunResult`` / ``IterationBenchmark`` / ``benchmark_iterations``
                                                       pkg/solvers.py:339-492
* ``Solver`` — the device handle behind them (``scfr_create`` / ``scfr_step``
  / ``scfr_exploitability`` …); one handle can carry a batch of independent
  solves that share the game (hyper-parameter sweeps).

Every iteration runs inside the native library as sm_100a kernels; this
module only schedules steps between checkpoints and rebuilds the reference's
records.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass

import numpy as np

from . import native as N
from .compiler import GameBundle, build_bundle
from .games import FlatGame, Game
from .metrics import ConvergenceRecord

VARIANTS = ("cfr", "cfr+", "dcfr", "pcfr", "pcfr+")
_VARIANT_DEFAULTS = {"cfr": (0.0, "sim"), "cfr+": (1.0, "alt"), "dcfr": (2.0, "alt"),
                     "pcfr": (0.0, "sim"), "pcfr+": (2.0, "alt")}


@dataclass
class SolverConfig:
    """Variant and parameters; gamma/mode default per variant
    (reference pkg/solvers.py:47-79)."""

    variant: str = "cfr"
    alpha: float = 1.5
    beta: float = 0.0
    gamma: float | None = None
    mode: str | None = None

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}")
        if not (math.isfinite(self.alpha) and math.isfinite(self.beta)):
            raise ValueError("alpha and beta must be finite")
        g0, m0 = _VARIANT_DEFAULTS[self.variant]
        if self.gamma is None:
            self.gamma = g0
        if self.gamma < 0:
            raise ValueError("gamma must be >= 0")
        if self.mode is None:
            self.mode = m0
        if self.mode not in ("sim", "alt"):
            raise ValueError("mode must be 'sim' or 'alt'")

    @property
    def predictive(self) -> bool:
        return self.variant in ("pcfr", "pcfr+")


def discount_factors(t: int, alpha: float, beta: float) -> tuple[float, float]:
    """t^e/(t^e+1) per sign; infinite powers give 1 (pkg/solvers.py:82-94).
    The device schedule is built from the same libm pow in the native code."""
    def f(e):
        p = float(t) ** e
        return 1.0 if math.isinf(p) else p / (p + 1.0)
    return f(alpha), f(beta)


def work_per_iteration(bundle: GameBundle, config: SolverConfig) -> int:
    """The reference Backend work counter's per-iteration delta (exact by
    construction, pkg/kernels.py:10-13), from the structure sizes."""
    def parts(p):
        Nn, Sg, Sp = p.num_nodes, p.num_seqs, p.num_seqs - 1
        nxt = 4 * Sp + 3 * (Nn - 1) + 2 * Sg
        obs = 4 * (Nn - 1) + Sg + Nn + 6 * Sp
        cur = 4 * Sp + 3 * (Nn - 1) + Sg
        return nxt, obs, cur, Sp
    z = bundle.payoff.nnz
    total = z + z + bundle.procs[1].num_seqs
    for k, p in enumerate(bundle.procs):
        nxt, obs, cur, Sp = parts(p)
        post = Sp if config.variant in ("cfr+", "pcfr+", "dcfr") else 0
        total += obs + post
        if config.predictive:
            total += obs + (Sp if config.variant == "pcfr+" else 0) + nxt
        else:
            total += nxt
        if k == 0 and config.mode == "alt":
            total += cur
    return total


class Solver:
    """A device-resident solve (or a batch of solves sharing one game).

    ``batch_params`` is an optional sequence of (alpha, beta, gamma) tuples,
    one per solve; the variant and mode are common to the batch.
    """

    def __init__(self, bundle: GameBundle, config: SolverConfig, device: int = 0,
                 batch_params=None, engine: str = "auto", shard=None, dtype: str = "f64",
                 subtree: bool = False):
        """``shard=(nccl_unique_id, rank, world)`` selects a multi-GPU mode:
        the row-sharded payoff (distributed.sharded_solver) or, with
        ``subtree=True``, the subtree-sharded tree passes
        (distributed.subtree_solver).  ``dtype="f32"``
        runs the iteration in fp32 (same operation order, fp32 rounding;
        level engine); reads and exploitability stay fp64."""
        if dtype not in N.DTYPE_CODE:
            raise ValueError(f"unknown dtype {dtype!r}")
        self.bundle = bundle
        self.config = config
        L = N.lib()
        cfg = N.Config()
        cfg.variant = N.VARIANT_CODE[config.variant]
        cfg.mode = N.MODE_CODE[config.mode]
        cfg.alpha, cfg.beta, cfg.gamma = float(config.alpha), float(config.beta), float(config.gamma)
        self._keep = []
        if batch_params:
            bp = np.asarray(batch_params, dtype=np.float64).reshape(-1, 3)
            for k in range(bp.shape[0]):
                a, b, g = bp[k]
                if not (math.isfinite(a) and math.isfinite(b)):
                    raise ValueError("alpha and beta must be finite")
                if g < 0:
                    raise ValueError("gamma must be >= 0")
            cols = [np.ascontiguousarray(bp[:, i]) for i in range(3)]
            self._keep += cols
            cfg.batch = bp.shape[0]
            cfg.batch_alpha, cfg.batch_beta, cfg.batch_gamma = (N.ptr(c, C.c_double) for c in cols)
            self.batch_params = [tuple(map(float, row)) for row in bp]
        else:
            cfg.batch = 1
            self.batch_params = [(float(config.alpha), float(config.beta), float(config.gamma))]
        cfg.engine = N.ENGINE_CODE[engine]
        cfg.dtype = N.DTYPE_CODE[dtype]
        self.dtype = "f32" if cfg.dtype == 1 else "f64"
        self.batch = int(cfg.batch)
        self.device = device
        h = C.c_void_p()
        p1, p2, U, UT = bundle._c
        self.shard = None
        self.subtree = bool(subtree)
        if subtree and shard is None:
            raise ValueError("subtree=True needs shard=(nccl_unique_id, rank, world)")
        if shard is not None:
            uid, rank, world = shard
            if len(uid) != 128:
                raise ValueError("NCCL unique id must be 128 bytes")
            self.shard = (int(rank), int(world))
            create = L.scfr_create_subtree if subtree else L.scfr_create_sharded
            N.check(create(C.byref(p1), C.byref(p2), C.byref(U), C.byref(UT),
                           C.byref(cfg), int(device), uid, int(rank), int(world), C.byref(h)))
        else:
            N.check(L.scfr_create(C.byref(p1), C.byref(p2), C.byref(U), C.byref(UT),
                                  C.byref(cfg), int(device), C.byref(h)))
        self._h = h

    # -- iteration -----------------------------------------------------------
    def step(self, n: int = 1) -> None:
        N.check(N.lib().scfr_step(self._h, int(n)))

    def set_schedule(self, w=None, pos_factor=None, neg_factor=None, solve: int = -1) -> None:
        """Caller-computed scalars for the next len(...) iterations: averaging
        weights w_t (float(t)**gamma in the reference) and DCFR factors for
        positive / negative regrets.  None keeps the library's libm values."""
        arrs = [None if a is None else np.ascontiguousarray(a, dtype=np.float64) for a in (w, pos_factor, neg_factor)]
        sizes = {a.shape[0] for a in arrs if a is not None}
        if len(sizes) > 1:
            raise ValueError("schedule arrays must have one length")
        n = sizes.pop() if sizes else 0
        ptrs = [None if a is None else N.ptr(a, C.c_double) for a in arrs]
        N.check(N.lib().scfr_set_schedule(self._h, int(solve), *ptrs, n))

    def synchronize(self) -> None:
        N.check(N.lib().scfr_synchronize(self._h))

    def snapshot(self, restore: bool = False) -> None:
        """Save (or restore) the whole iteration state in device memory."""
        N.check(N.lib().scfr_snapshot(self._h, 1 if restore else 0))

    @property
    def iterations(self) -> int:
        v = C.c_int64()
        N.check(N.lib().scfr_iterations(self._h, C.byref(v)))
        return int(v.value)

    def check_finite(self) -> None:
        flag = C.c_int()
        N.check(N.lib().scfr_status(self._h, C.byref(flag)))
        if flag.value:
            raise FloatingPointError("non-finite regrets or utilities")

    @property
    def engine(self) -> str:
        """Engine the handle runs: levels / persistent / persistent_grid."""
        v = C.c_int()
        N.check(N.lib().scfr_engine(self._h, C.byref(v)))
        return N.ENGINE_NAME[int(v.value)]

    def last_step_ms(self) -> float:
        v = C.c_double()
        N.check(N.lib().scfr_last_step_ms(self._h, C.byref(v)))
        return float(v.value)

    def launch_count(self) -> int:
        v = C.c_int64()
        N.check(N.lib().scfr_launch_count(self._h, C.byref(v)))
        return int(v.value)

    def device_bytes(self) -> int:
        v = C.c_int64()
        N.check(N.lib().scfr_device_bytes(self._h, C.byref(v)))
        return int(v.value)

    def profile(self, n: int = 1) -> dict:
        """Run n real iterations with CUDA events around every launch;
        returns {kind: {"launches", "ms", "bytes"}} (algorithmic bytes)."""
        stats = (N.KernelStat * 16)()
        cnt = C.c_int()
        N.check(N.lib().scfr_profile_step(self._h, int(n), stats, 16, C.byref(cnt)))
        return {stats[k].name.decode(): {"launches": int(stats[k].launches), "ms": float(stats[k].ms),
                                         "bytes": float(stats[k].bytes)}
                for k in range(cnt.value) if stats[k].launches}

    def timeline(self, n: int = 3) -> list[dict]:
        """Run n real iterations through a recording copy of the iteration
        graph (the overlapped two-stream body when the handle overlaps alt
        iterations); one entry per launch: kind, stream, algorithmic bytes,
        mean start / end (us from the iteration's first start, %globaltimer),
        own duration, and the exclusive span: launches ordered by end time
        partition the step, each instant belonging to the launch that
        finishes next."""
        spans = (N.KernelSpan * 4096)()
        cnt = C.c_int()
        N.check(N.lib().scfr_timeline(self._h, int(n), spans, 4096, C.byref(cnt)))
        out = [{"kind": spans[k].name.decode(), "stream": int(spans[k].stream), "bytes": float(spans[k].bytes),
                "start_us": float(spans[k].start_us), "end_us": float(spans[k].end_us)} for k in range(cnt.value)]
        prev = 0.0
        for e in sorted(out, key=lambda e: e["end_us"]):
            e["own_us"] = e["end_us"] - e["start_us"]
            e["excl_us"] = max(0.0, e["end_us"] - prev)
            prev = max(prev, e["end_us"])
        return out

    # -- reads -----------------------------------------------------------------
    def _nseq(self, player: int) -> int:
        if player not in (1, 2):
            raise ValueError("player must be 1 or 2")
        return self.bundle.procs[player - 1].num_seqs

    def average(self, player: int, solve: int = 0) -> np.ndarray:
        out = np.empty(self._nseq(player))
        N.check(N.lib().scfr_read_average(self._h, player, solve, N.ptr(out, C.c_double)))
        return out

    def averages(self, solve: int = 0) -> tuple[np.ndarray, np.ndarray]:
        """Both players' average strategies (one pipelined read)."""
        o1, o2 = np.empty(self._nseq(1)), np.empty(self._nseq(2))
        N.check(N.lib().scfr_read_averages(self._h, solve, N.ptr(o1, C.c_double), N.ptr(o2, C.c_double)))
        return o1, o2

    def current(self, player: int, solve: int = 0) -> np.ndarray:
        out = np.empty(self._nseq(player))
        N.check(N.lib().scfr_read_current(self._h, player, solve, N.ptr(out, C.c_double)))
        return out

    def state(self, player: int, which: str, solve: int = 0) -> np.ndarray:
        n = self._nseq(player) - (1 if which in ("regrets", "behavior") else 0)
        out = np.empty(n)
        N.check(N.lib().scfr_read_state(self._h, player, solve, N.STATE_CODE[which],
                                        N.ptr(out, C.c_double)))
        return out

    def regrets(self, player: int, solve: int = 0) -> np.ndarray:
        return self.state(player, "regrets", solve)

    def avg_weight(self, solve: int = 0) -> float:
        v = C.c_double()
        N.check(N.lib().scfr_avg_weight(self._h, 1, solve, C.byref(v)))
        return float(v.value)

    def exploitability(self, which: str = "average", solve: int = 0):
        """NashConv/2 of the average or current profile; returns
        (exploitability, (br1, br2))."""
        e, b1, b2 = C.c_double(), C.c_double(), C.c_double()
        N.check(N.lib().scfr_exploitability(self._h, solve, 0 if which == "average" else 1,
                                            C.byref(e), C.byref(b1), C.byref(b2)))
        return float(e.value), (float(b1.value), float(b2.value))

    def expected_value(self, solve: int = 0) -> float:
        v = C.c_double()
        N.check(N.lib().scfr_expected_value(self._h, solve, C.byref(v)))
        return float(v.value)

    def best_response_values(self, x1, x2) -> tuple[float, float]:
        a = np.ascontiguousarray(x1, dtype=np.float64)
        b = np.ascontiguousarray(x2, dtype=np.float64)
        if a.shape[0] != self._nseq(1) or b.shape[0] != self._nseq(2):
            raise ValueError("dimension mismatch: profile does not match the game")
        b1, b2 = C.c_double(), C.c_double()
        N.check(N.lib().scfr_best_response_values(self._h, N.ptr(a, C.c_double), N.ptr(b, C.c_double),
                                                  C.byref(b1), C.byref(b2)))
        return float(b1.value), float(b2.value)

    def expected_value_of(self, x1, x2) -> float:
        a = np.ascontiguousarray(x1, dtype=np.float64)
        b = np.ascontiguousarray(x2, dtype=np.float64)
        if a.shape[0] != self._nseq(1) or b.shape[0] != self._nseq(2):
            raise ValueError("dimension mismatch: profile does not match the game")
        v = C.c_double()
        N.check(N.lib().scfr_expected_value_of(self._h, N.ptr(a, C.c_double), N.ptr(b, C.c_double),
                                               C.byref(v)))
        return float(v.value)

    def close(self) -> None:
        if getattr(self, "_h", None):
            N.lib().scfr_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def evaluator(bundle: GameBundle, device: int = 0) -> Solver:
    """A cached batch-1 handle used for metrics on arbitrary profiles."""
    if bundle._evaluator is None:
        bundle._evaluator = Solver(bundle, SolverConfig("cfr"), device=device, engine="levels")
    return bundle._evaluator


@dataclass
class RunResult:
    bundle: GameBundle
    config: SolverConfig
    average: tuple[np.ndarray, np.ndarray]
    last_iterates: tuple[np.ndarray, np.ndarray]
    records: list[ConvergenceRecord]
    iterations: int


def _as_bundle(game) -> GameBundle:
    if isinstance(game, GameBundle):
        return game
    if isinstance(game, (Game, FlatGame)):
        return GameBundle(game)
    raise TypeError("run needs a Game, FlatGame or GameBundle")


def run(game, config: SolverConfig, iterations: int | None = None,
        seconds: float | None = None, checkpoints=None, backend=None,
        record_current: bool = True, device: int = 0, engine: str = "auto",
        dtype: str = "f64") -> RunResult:
    """Solve and record convergence (reference pkg/solvers.py:375-438).

    Iterates are bit-identical to the reference's.  Iterations between
    checkpoints run as one device batch; a ``seconds`` budget is checked
    between batches of at most 64 iterations.  ``backend`` is accepted for
    signature compatibility and ignored (the device is the backend).
    """
    if iterations is None and seconds is None:
        raise ValueError("budget must be positive: give iterations and/or seconds")
    if iterations is not None and iterations <= 0:
        raise ValueError("budget must be positive: iterations <= 0")
    if seconds is not None and seconds <= 0:
        raise ValueError("budget must be positive: seconds <= 0")
    del backend
    bundle = _as_bundle(game)
    solver = Solver(bundle, config, device=device, engine=engine, dtype=dtype)
    schedule = sorted(set(int(c) for c in checkpoints)) if checkpoints else []
    wpi = work_per_iteration(bundle, config)
    peak = bundle.reference_nbytes() + bundle.reference_state_bytes()
    records: list[ConvergenceRecord] = []
    start = time.perf_counter()

    def record(t: int) -> None:
        expl = solver.exploitability("average")[0]
        cur = solver.exploitability("current")[0] if record_current else math.nan
        records.append(ConvergenceRecord(iteration=t, seconds=time.perf_counter() - start,
                                         exploitability=expl, current_exploitability=cur,
                                         work=wpi * t, peak_bytes=peak))

    t = 0
    while True:
        nxt = [c for c in schedule if c > t]
        target = nxt[0] if nxt else None
        if iterations is not None:
            target = iterations if target is None else min(target, iterations)
        chunk = (target - t) if target is not None else 64
        if seconds is not None:
            chunk = min(chunk, 64)
        solver.step(chunk)
        if seconds is not None:
            solver.synchronize()
        t += chunk
        done = (iterations is not None and t >= iterations) or \
            (seconds is not None and time.perf_counter() - start >= seconds)
        if t in schedule or done:
            solver.check_finite()
            record(t)
        if done:
            break
    solver.check_finite()
    result = RunResult(bundle=bundle, config=config,
                       average=solver.averages(),
                       last_iterates=(solver.current(1), solver.current(2)),
                       records=records, iterations=t)
    solver.close()
    return result


@dataclass
class TargetResult:
    """Outcome of ``solve_to_target``: the first checked iteration whose
    average-profile exploitability is <= target."""

    reached: bool
    iterations: int
    exploitability: float
    seconds: float          # wall clock, iterations + exploitability checks
    solve_seconds: float    # device time of the iterations alone (CUDA events)
    checks: int


def solve_to_target(game, config: SolverConfig, target: float = 1e-4, check_every: int = 1,
                    max_iterations: int = 1_000_000, device: int = 0,
                    engine: str = "auto", dtype: str = "f64", stride: int = 16) -> TargetResult:
    """Iterate until the average profile's exploitability is <= target,
    checking every ``check_every`` iterations on the device (time-to-target
    metric of BASELINE.json; the reference computes the same quantity with a
    checkpointed ``run``, pkg/solvers.py:406-432).

    With ``check_every=1`` the search is coarse-to-fine: the state is
    snapshotted on the device, ``stride`` iterations run, one exploitability
    check; on a hit the snapshot is restored and the last ``stride``
    iterations replay with a check after each.  The iterates are
    deterministic, so the result is the exact first iteration that meets
    the target, with about 1/stride of the best-response checks on the
    critical path."""
    if target <= 0 or check_every < 1 or stride < 1:
        raise ValueError("target must be > 0, check_every >= 1 and stride >= 1")
    bundle = _as_bundle(game)
    s = Solver(bundle, config, device=device, engine=engine, dtype=dtype)
    t0 = time.perf_counter()
    solve_ms = 0.0
    t = checks = 0
    e = math.inf

    def advance(n):
        nonlocal solve_ms, t, e, checks
        s.step(n)
        solve_ms += s.last_step_ms()
        t += n
        e = s.exploitability("average")[0]
        checks += 1

    coarse = check_every == 1 and stride > 1
    while t < max_iterations and e > target:
        if not coarse:
            advance(min(check_every, max_iterations - t))
            continue
        k = min(stride, max_iterations - t)
        s.snapshot()
        t_start = t
        advance(k)
        if e <= target and k > 1:  # the first hit lies in (t_start, t]: replay one by one
            s.snapshot(restore=True)
            t = t_start
            e = math.inf
            while e > target:
                advance(1)
    s.check_finite()
    out = TargetResult(e <= target, t, e, time.perf_counter() - t0, solve_ms / 1e3, checks)
    s.close()
    return out


@dataclass
class IterationBenchmark:
    proc_nodes: int
    backend_kind: str
    workers: int
    times: list[float]
    work_per_iteration: int
    state_bytes: int          # the reference's figure: bundle.nbytes() + both RegretState.state_bytes()
    device_bytes: int = 0     # what this handle holds in HBM (structure, state, schedules)

    @property
    def mean_seconds(self) -> float:
        return float(np.mean(self.times))

    @property
    def stderr_seconds(self) -> float:
        if len(self.times) < 2:
            return 0.0
        return float(np.std(self.times, ddof=1) / math.sqrt(len(self.times)))


def benchmark_iterations(bundle: GameBundle, config: SolverConfig, backend=None,
                         warmup: int = 2, measured: int = 8, device: int = 0,
                         engine: str = "auto", dtype: str = "f64") -> IterationBenchmark:
    """Per-iteration device time (CUDA events around each step)
    (reference pkg/solvers.py:463-492)."""
    if measured < 1:
        raise ValueError("measured iterations must be >= 1")
    del backend
    s = Solver(bundle, config, device=device, engine=engine, dtype=dtype)
    if warmup:
        s.step(warmup)
    s.synchronize()
    times = []
    for _ in range(measured):
        s.step(1)
        times.append(s.last_step_ms() / 1e3)
    out = IterationBenchmark(proc_nodes=bundle.num_proc_nodes, backend_kind="cuda", workers=1,
                             times=times, work_per_iteration=work_per_iteration(bundle, config),
                             state_bytes=bundle.reference_nbytes() + bundle.reference_state_bytes(),
                             device_bytes=s.device_bytes())
    s.close()
    return out


__all__ = ["VARIANTS", "SolverConfig", "discount_factors", "Solver", "RunResult", "run",
           "TargetResult", "solve_to_target",
           "IterationBenchmark", "benchmark_iterations", "work_per_iteration", "build_bundle",
           "GameBundle", "evaluator"]
