#!/usr/bin/env python
"""Benchmark: CFR iterations/sec on the largest single-GPU config.

Workload (default): Goofspiel-5 (bids revealed, random prize order, win/loss;
8 530 656 game nodes, |Σ| = 2 666 026 per player, nnz(U) = 1 728 000), PCFR+
alternating, gamma = 2, fp64 — BASELINE.json configs[3] on one GPU.  A step is
one full CFR iteration (reference ``_step``, pkg/solvers.py:351-372).  The
working set (~1 GB/iteration) is far above the 126 MB L2, so no L2 flush is
needed between iterations.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload ...]

N > 1 (torchrun, one rank per GPU): every rank runs an independent replica of
the solve (no collective on the data path; weak scaling), value = all ranks'
iterations / max-over-ranks device time.

``--impl reference`` times the reference algorithm's CPU implementation on the
host cores: the C oracle (a port of the reference's per-iteration path,
oracle/seqcfr_oracle.c, pinned bit-exact to the reference by tests/) with all
host threads; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

E2E_REPS = 3

WORKLOADS = {
    # name: (description, builder, variant)
    "goofspiel5": ("goofspiel-5 pcfr+ alt (bids revealed, random prize order, win/loss)", "goof", "pcfr+"),
    "liars_dice": ("liars-dice 1x1x6 dcfr(1.5,0,2) alt", "liars", "dcfr"),
    "leduc": ("leduc cfr+ alt", "leduc", "cfr+"),
    "kuhn": ("kuhn cfr sim", "kuhn", "cfr"),
}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def make_bundle(kind: str):
    from paper_2605_14277_b200 import GameBundle, flat_goofspiel, flat_liars_dice, kuhn_poker, leduc_poker
    if kind == "goof":
        return GameBundle(flat_goofspiel(5))
    if kind == "liars":
        return GameBundle(flat_liars_dice(6))
    if kind == "leduc":
        return GameBundle(leduc_poker())
    return GameBundle(kuhn_poker())


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self.window = None

    def start(self):
        def loop():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True,
                                         text=True, timeout=5).stdout.strip()
                    if out:
                        self.samples.append((time.time(), out.split(", ")))
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self, t0: float, t1: float) -> dict:
        rows = [s for (t, s) in self.samples if t0 <= t <= t1] or [s for (_, s) in self.samples]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def survey_step_bytes(bundle, cfg, v: int = 8) -> int:
    """SURVEY.md §8(d)'s fused compulsory bytes per iteration (8 B values,
    4 B indices): per player OBS = 8Σ+40S+20J, NEXT = 8S+12J+24Σ, PRED =
    8Σ+32S+20J (and OBS drops its b write, −8S), one SpMV each way
    4(R+1)+12Z+8C+8R, and alt adds NEXT_1 without avg (8S+12J+8Σ).
    Σ counts the empty sequence, S does not.  Scaled to v-byte values."""
    Z = bundle.payoff.nnz
    sig = [p.num_seqs for p in bundle.procs]
    tot = 0
    for p, sg in zip(bundle.procs, sig):
        S, J = sg - 1, p.num_decisions
        obs = v * sg + 5 * v * S + 20 * J
        nxt = v * S + 12 * J + 3 * v * sg
        if cfg.predictive:
            tot += (obs - v * S) + (v * sg + 4 * v * S + 20 * J) + nxt
        else:
            tot += obs + nxt
    spmv = lambda R, C_: 4 * (R + 1) + (4 + v) * Z + v * C_ + v * R
    tot += spmv(sig[0], sig[1]) + spmv(sig[1], sig[0])
    if cfg.mode == "alt":
        S, J = sig[0] - 1, bundle.procs[0].num_decisions
        tot += v * S + 12 * J + v * sig[0]
    return tot


def size_matched_copy(device: int, bytes_per_launch: float, achieved_gbs: float) -> dict:
    """What a bare fp64 device copy moving the dominant kernel's average
    bytes per launch achieves on this GPU (cold L2, CUDA events, best of 10):
    the attainable bandwidth at that launch size, reported beside the
    roofline.  Peak stays MEASURED_PEAKS' 1 GiB copy."""
    import torch
    n = max(1, int(bytes_per_launch / 16))  # read + write 8 B each
    src = torch.zeros(n, dtype=torch.float64, device=f"cuda:{device}")
    dst = torch.empty_like(src)
    flush = torch.empty(64 << 20, dtype=torch.float64, device=f"cuda:{device}")  # 512 MB > L2
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = float("inf")
    for _ in range(10):
        flush.fill_(1.0)
        e0.record()
        dst.copy_(src)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    gbs = 16.0 * n / (best / 1e3) / 1e9
    del src, dst, flush
    return {"bytes_per_launch": 16.0 * n, "gbs": gbs, "kernel_frac_of_copy": achieved_gbs / gbs,
            "how": "torch fp64 copy of the same bytes per launch, L2 flushed, best of 10"}


def cpu_oracle_rate(bundle, variant: str, steps: int, warmup: int, budget_s: float | None,
                    threads: int, dtype: str = "f64"):
    """The oracle port on the host cores: iterations/sec over a bounded sample."""
    from oracle.oracle import OracleSolver
    o = OracleSolver(bundle, variant, threads=threads, dtype=dtype)
    if warmup:
        o.step(warmup)
    if budget_s is not None:
        t0 = time.perf_counter()
        o.step(1)
        one = time.perf_counter() - t0
        steps = max(1, min(steps, int(budget_s / max(one, 1e-9))))
    t0 = time.perf_counter()
    o.step(steps)
    dt = time.perf_counter() - t0
    return steps / dt, steps, dt


def per_game_suite(device: int, cpu: bool) -> dict:
    """BASELINE.json configs on one GPU: iterations/s and time to
    exploitability 1e-4 (the exact first iteration, found by a coarse-to-fine
    search over device-side snapshots), the 256-solve Leduc DCFR sweep, and the CPU
    oracle on the same small configs for context."""
    from paper_2605_14277_b200 import Solver, SolverConfig, solve_to_target

    out = {}
    for name, kind, variant, check in (("kuhn_cfr", "kuhn", "cfr", None),
                                        ("leduc_cfr+", "leduc", "cfr+", 1),
                                        ("liars_dice_dcfr", "liars", "dcfr", 1)):
        b = make_bundle(kind)
        cfg = SolverConfig(variant)
        s = Solver(b, cfg, device=device)
        s.step(20)
        s.synchronize()
        s.step(500)
        rate = 500 / (s.last_step_ms() / 1e3)
        rec = {"engine": s.engine, "iterations_per_s": rate}
        s.close()
        if check:
            r = solve_to_target(b, cfg, 1e-4, check_every=check, device=device)
            rec.update({"target": 1e-4, "reached": r.reached, "iterations": r.iterations,
                        "exploitability": r.exploitability, "seconds_wall": r.seconds,
                        "seconds_solve_only": r.solve_seconds, "check_every": check,
                        "search": "coarse-to-fine: snapshot, 16 iterations, check; replay on a hit"})
        else:
            s = Solver(b, cfg, device=device)
            s.step(1000)
            rec["exploitability_at_1000"] = s.exploitability("average")[0]
            s.close()
        if cpu:
            threads = 1  # small trees: the port is latency-bound, one thread is fastest
            crate, _, _ = cpu_oracle_rate(b, variant, 200, 3, 5.0, threads)
            rec["cpu_oracle_iterations_per_s"] = crate
        out[name] = rec
    # config 5: 256 DCFR(alpha, beta, gamma) Leduc solves, one handle
    grid = [(a, bb, g) for a in (0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 5.0, 8.0)
            for bb in (-1.0, -0.5, 0.0, 0.5) for g in (0.0, 1.0, 2.0, 3.0)] * 2
    b = make_bundle("leduc")
    s = Solver(b, SolverConfig("dcfr"), device=device, batch_params=grid)
    s.step(5)
    s.synchronize()
    s.step(1000)
    ms = s.last_step_ms()
    out["leduc_dcfr_sweep_256"] = {"engine": s.engine, "solves": len(grid), "iterations": 1000,
                                   "seconds": ms / 1e3,
                                   "solve_iterations_per_s": len(grid) * 1000 / (ms / 1e3)}
    s.close()
    return out


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    desc, kind, variant = WORKLOADS[args.workload]
    bundle = make_bundle(kind)
    threads = os.cpu_count() or 1
    rate, steps, dt = cpu_oracle_rate(bundle, variant, args.steps, args.warmup, None, threads)
    line = {
        "impl": "reference", "metric": "cfr_iterations_per_sec", "value": rate,
        "unit": "iterations/s", "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (generated game tree)",
        "config": {"workload": desc, "variant": variant, "parallelism": "host threads"},
        "cpu_baseline": {"value": rate, "unit": "iterations/s", "cores": threads, "kind": "port",
                         "sample": f"{steps} {args.workload} iterations after {args.warmup} warm-up "
                                   f"(oracle/seqcfr_oracle.c, bit-exact port of the reference path)"},
        "e2e": {"value": rate, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    dist = None
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    device = local
    from paper_2605_14277_b200 import Solver, SolverConfig, native

    desc, kind, variant = WORKLOADS[args.workload]
    bundle = make_bundle(kind)
    cfg = SolverConfig(variant)
    sharded = args.mode == "sharded" and ws > 1

    def make_solver():
        if sharded:  # config 4: one solve, payoff SpMV rows split over the ranks
            from paper_2605_14277_b200.distributed import sharded_solver
            return sharded_solver(bundle, cfg, device=device)
        return Solver(bundle, cfg, device=device, dtype=args.dtype)

    # process-level warm-up (CUDA context, lazy module load) outside any timing
    torch.cuda.synchronize(device)
    warm = make_solver()
    warm.step(1)
    warm.synchronize()
    warm.close()
    h2d0, d2h0 = native.transfer_bytes()

    # --- end-to-end through the public API: upload (create) + K iterations +
    # read back both average strategies; wall clock, host buffers.  The median
    # of E2E_REPS full repetitions (host-side create time is noisy on a VM).
    runs = []
    for _ in range(E2E_REPS):
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        s = make_solver()
        t1 = time.perf_counter()
        s.step(args.steps)
        s.synchronize()
        t2 = time.perf_counter()
        avg = (s.average(1), s.average(2))
        t3 = time.perf_counter()
        runs.append((t3 - t0, {"create_s": t1 - t0, "steps_s": t2 - t1, "readback_s": t3 - t2}))
        del avg
        s.close()
    h2d1, d2h1 = native.transfer_bytes()
    runs.sort(key=lambda r: r[0])
    e2e_s, e2e_parts = runs[len(runs) // 2]
    e2e_parts = dict(e2e_parts, reps=E2E_REPS, all_s=[round(r[0], 6) for r in runs])

    # --- device-timed region
    s = make_solver()
    s.step(args.warmup)
    s.synchronize()
    sampler = ClockSampler(device)
    sampler.start()
    soak_end = time.time() + args.soak
    while time.time() < soak_end:  # keep the GPU loaded while the clock sampler warms up
        s.step(max(1, args.warmup))
        s.synchronize()
    launches0 = s.launch_count()
    if dist:
        dist.barrier()
    torch.cuda.synchronize(device)
    tw0 = time.time()
    s.step(args.steps)
    s.synchronize()
    tw1 = time.time()
    ms = s.last_step_ms()
    launches = s.launch_count() - launches0
    sampler.stop()
    clocks = sampler.summary(tw0 - args.soak, tw1)
    ms_max = ms
    e2e_max = e2e_s
    if dist:
        t = torch.tensor([ms, e2e_s], dtype=torch.float64, device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max, e2e_max = float(t[0]), float(t[1])

    # --- per-kernel roofline (CUDA events around every launch, same stream)
    prof = s.profile(args.profile_iters)
    peak, peak_kind = _peaks()
    dom = max(prof.items(), key=lambda kv: kv[1]["ms"])
    dname, d = dom
    achieved = d["bytes"] / (d["ms"] / 1e3) / 1e9
    step_bytes = sum(v["bytes"] for v in prof.values()) / args.profile_iters
    prof_ms = sum(v["ms"] for v in prof.values()) / args.profile_iters
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            with open(tfile) as fh:
                tj = json.load(fh)
            if args.workload in tj and dname in tj[args.workload]:
                traffic = tj[args.workload][dname]
        except Exception:
            traffic = None

    copy_ref = size_matched_copy(device, d["bytes"] / max(1, d["launches"]), achieved)
    survey_bytes = survey_step_bytes(bundle, cfg, 4 if args.dtype == "f32" else 8)
    survey_gbs = survey_bytes / (ms_max / args.steps / 1e3) / 1e9

    solves = 1 if sharded else ws  # sharded: all ranks advance ONE solve
    value = solves * args.steps / (ms_max / 1e3)
    line = {
        "metric": "cfr_iterations_per_sec", "value": value, "unit": "iterations/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (generated game tree)",
        "config": {"workload": desc, "variant": variant, "mode": cfg.mode, "gamma": cfg.gamma,
                   "seqs_per_player": [p.num_seqs for p in bundle.procs],
                   "nnz_U": bundle.payoff.nnz, "parallelism": (f"row-sharded payoff SpMV + NCCL all-gather x{ws}" if sharded
                                   else f"independent replicas x{ws}" if ws > 1 else "1 gpu"),
                   "l2": "working set > L2 (no flush needed)",
                   "engine": s.engine},
        "gpu_launches": launches,
        "clocks": clocks,
        "e2e": {"value": solves * args.steps / e2e_max, "unit": "iterations/s",
                "h2d_bytes_per_step": (h2d1 - h2d0) / E2E_REPS / args.steps,
                "d2h_bytes_per_step": (d2h1 - d2h0) / E2E_REPS / args.steps,
                "includes": "scfr_create upload + K iterations + average-strategy readback, wall clock; "
                            f"median of {E2E_REPS} repetitions",
                "parts": e2e_parts},
        "roofline": {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak,
                     "size_matched_copy": copy_ref,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_kind,
                     "step": {"algorithmic_bytes": step_bytes, "profiled_ms": prof_ms,
                              "achieved_gbs": step_bytes / (prof_ms / 1e3) / 1e9,
                              "frac": step_bytes / (prof_ms / 1e3) / 1e9 / peak},
                     "survey_8d": {"algorithmic_bytes_per_step": survey_bytes,
                                   "achieved_gbs": survey_gbs, "frac": survey_gbs / peak,
                                   "note": "SURVEY §8(d) fused compulsory bytes over the graph-timed step; "
                                           "the exact shortcuts (DESIGN §4) skip part of them, so this "
                                           "overstates bandwidth use: frac above uses the bytes the "
                                           "kernels load"},
                     "kernels": {k: {"launches": v["launches"] // args.profile_iters,
                                     "ms": v["ms"] / args.profile_iters,
                                     "gbs": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] else None}
                                 for k, v in prof.items()}},
    }
    if ws == 1 and rank == 0 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rate, steps, dt = cpu_oracle_rate(bundle, variant, 50, 1, args.cpu_budget, threads, args.dtype)
        line["cpu_baseline"] = {"value": rate, "unit": "iterations/s", "cores": threads,
                                "kind": "port",
                                "sample": f"{steps} {args.workload} iterations after 1 warm-up, "
                                          f"{dt:.1f}s (oracle/seqcfr_oracle.c)"}
    s.close()
    if rank == 0 and not args.no_suite:
        line["per_game"] = per_game_suite(device, ws == 1 and not args.no_cpu_baseline)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="goofspiel5")
    ap.add_argument("--dtype", choices=("f64", "f32"), default="f64",
                    help="f64 (default; bit-exact with the reference) or the optional fp32 mode")
    ap.add_argument("--profile-iters", type=int, default=3)
    ap.add_argument("--soak", type=float, default=1.0)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-suite", action="store_true", help="skip the per-game section")
    ap.add_argument("--mode", choices=("replicas", "sharded"), default="replicas",
                    help="N>1: independent replicas (weak) or one row-sharded solve (strong)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
