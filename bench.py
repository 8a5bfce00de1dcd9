#!/usr/bin/env python
"""Benchmark: CFR iterations/sec on the largest config (BASELINE.json configs[3]).

Workload (default): Goofspiel-5 (bids revealed, random prize order, win/loss;
8 530 656 game nodes, |Σ| = 2 666 026 per player, nnz(U) = 1 728 000), PCFR+
alternating, gamma = 2, fp64.  A step is one full CFR iteration (reference
``_step``, pkg/solvers.py:351-372).  The working set (~0.4 GB moved per
iteration) is far above the 126 MB L2, so no L2 flush is needed between
iterations.  Iterates at 1/2/10/30/50 iterations are bit-identical to the
reference's own (tests/test_gpu_goof5.py).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload ...]

N = 1: the Goofspiel-5 solve on one GPU.  N > 1 (torchrun, one rank per GPU):
the SAME single solve (strong scaling; value = that solve's iterations/s over
the max-over-ranks device time) with the tree passes subtree-sharded
(``--mode subtree``, default: each rank runs the trunk and its own subtrees,
NCCL broadcasts of the subtree roots' values) or with the
payoff SpMV row-sharded and u all-gathered (``--mode sharded``, config 4).
``--mode subtree|sharded`` at N = 1 runs that path over a 1-rank NCCL
communicator.  Every line
also carries ``sweep``: config 5, 256 distinct Leduc DCFR(alpha, beta, gamma)
solves split over the N ranks (no collective), in solve-iterations/s.

``--impl reference`` times the reference algorithm's CPU implementation on the
host cores: the C oracle (oracle/seqcfr_oracle.c, a port of the reference's
per-iteration path, pinned bit-exact to the reference by tests/) over a bundle
built by the oracle's own compile step (oracle/seqcfr_tree.c) — no product
code is loaded.  Serial and all-core runs are both timed and the better one
is reported; rank 0 only.
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


def oracle_bundle(kind: str):
    """The same game compiled by the oracle's C restatement of the reference
    compile step (oracle/seqcfr_tree.c): the CPU legs never load the product
    library.  Kuhn / Leduc trees come from the pure-Python game builders."""
    from oracle import tree
    if kind == "goof":
        return tree.native_bundle("goofspiel", 5)
    if kind == "liars":
        return tree.native_bundle("liars_dice", 6)
    from paper_2605_14277_b200 import games as G  # pure Python (no native code)
    g = G.leduc_poker() if kind == "leduc" else G.kuhn_poker()
    return tree.compile_native(g.flatten())


def loaded_native_libs() -> list:
    """Shared objects from this repo mapped into the process (self-check of
    which native code a leg actually ran)."""
    out = set()
    try:
        with open("/proc/self/maps") as fh:
            for line in fh:
                p = line.split()[-1]
                if p.endswith(".so") and p.startswith(ROOT):
                    out.add(os.path.relpath(p, ROOT))
    except OSError:
        pass
    return sorted(out)


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


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


def cpu_best_rate(bundle, variant: str, steps: int, warmup: int, budget_s: float | None,
                  dtype: str = "f64") -> dict:
    """Serial and all-core runs of the oracle port; the better is the
    baseline ('the better of serial and parallel[cores]')."""
    cores = os.cpu_count() or 1
    runs = {}
    for th in sorted({1, cores}):
        rate, n, dt = cpu_oracle_rate(bundle, variant, steps, warmup, budget_s, th, dtype)
        runs[th] = {"iterations_per_s": rate, "steps": n, "seconds": dt}
    best = max(runs, key=lambda k: runs[k]["iterations_per_s"])
    return {"value": runs[best]["iterations_per_s"], "cores": best, "runs": runs,
            "steps": runs[best]["steps"], "seconds": runs[best]["seconds"]}


def sweep_grid():
    """Config 5: 256 DISTINCT DCFR (alpha, beta, gamma) triples on a fixed
    grid (gamma refined to reach 256)."""
    return [(a, b, g) for a in (0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 5.0, 8.0)
            for b in (-1.0, -0.5, 0.0, 0.5) for g in (0.0, 0.5, 1.0, 1.5, 2.0, 2.5, 3.0, 4.0)]


def per_game_suite(device: int, cpu: bool) -> dict:
    """BASELINE.json configs on one GPU: iterations/s and time to
    exploitability 1e-4 (the exact first iteration, found by a coarse-to-fine
    search over device-side snapshots) for Leduc, Liar's dice and the bench
    config Goofspiel-5, Kuhn @1000, and the CPU oracle on the same small
    configs for context (built product-free)."""
    from paper_2605_14277_b200 import Solver, SolverConfig, solve_to_target

    out = {}
    for name, kind, variant, check in (("kuhn_cfr", "kuhn", "cfr", None),
                                        ("leduc_cfr+", "leduc", "cfr+", 1),
                                        ("liars_dice_dcfr", "liars", "dcfr", 1),
                                        ("goofspiel5_pcfr+", "goof", "pcfr+", 1)):
        b = make_bundle(kind)
        cfg = SolverConfig(variant)
        s = Solver(b, cfg, device=device)
        s.step(20)
        s.synchronize()
        n = 100 if kind == "goof" else 500
        s.step(n)
        rate = n / (s.last_step_ms() / 1e3)
        rec = {"engine": s.engine, "iterations_per_s": rate}
        s.close()
        if check:
            r = solve_to_target(b, cfg, 1e-4, check_every=check, device=device,
                                max_iterations=20000)
            rec.update({"target": 1e-4, "reached": r.reached, "iterations": r.iterations,
                        "exploitability": r.exploitability, "seconds_wall": r.seconds,
                        "seconds_solve_only": r.solve_seconds, "check_every": check,
                        "search": "coarse-to-fine: snapshot, 16 iterations, check; replay on a hit"})
        else:
            s = Solver(b, cfg, device=device)
            s.step(1000)
            rec["exploitability_at_1000"] = s.exploitability("average")[0]
            s.close()
        if cpu and kind != "goof":
            crate, _, _ = cpu_oracle_rate(oracle_bundle(kind), variant, 200, 3, 5.0, 1)
            rec["cpu_oracle_iterations_per_s"] = crate  # small trees: one thread is fastest
        out[name] = rec
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
    t0 = time.perf_counter()
    bundle = oracle_bundle(kind)
    build_s = time.perf_counter() - t0
    best = cpu_best_rate(bundle, variant, args.steps, args.warmup, None)
    rate = best["value"]
    line = {
        "impl": "reference", "metric": "cfr_iterations_per_sec", "value": rate,
        "unit": "iterations/s", "n_gpus": args.gpus, "steps": best["steps"], "warmup": args.warmup,
        "ms_per_step": 1e3 * best["seconds"] / best["steps"], "higher_is_better": True,
        "scaling": "strong" if args.gpus > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (generated game tree)",
        "config": {"workload": desc, "variant": variant, "parallelism": "host threads"},
        "cpu_baseline": {"value": rate, "unit": "iterations/s", "cores": best["cores"], "kind": "port",
                         "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
                         "serial_vs_parallel": {str(k): v["iterations_per_s"] for k, v in best["runs"].items()},
                         "sample": f"{best['steps']} {args.workload} iterations after {args.warmup} warm-up, "
                                   f"better of 1 and {os.cpu_count()} threads (oracle/seqcfr_oracle.c, "
                                   f"bit-exact port of the reference path; bundle by oracle/seqcfr_tree.c "
                                   f"in {build_s:.1f}s)"},
        "e2e": {"value": rate, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "native_so_loaded": loaded_native_libs(),
    }
    print(json.dumps(line), flush=True)


def sweep_measure(device: int, ws: int, rank: int, dist, iters: int) -> dict:
    """Config 5 over the ranks: rank k solves its contiguous slice of the
    256-point DCFR grid as one batched handle (no collective)."""
    import torch
    from paper_2605_14277_b200 import Solver, SolverConfig
    from paper_2605_14277_b200.distributed import sweep_slice
    grid = sweep_grid()
    mine, lo = sweep_slice(grid, ws, rank)
    b = make_bundle("leduc")
    s = Solver(b, SolverConfig("dcfr"), device=device, batch_params=mine)
    s.step(5)
    s.synchronize()
    if dist:
        dist.barrier()
    s.step(iters)
    ms = s.last_step_ms()
    eng = s.engine
    s.close()
    ms_max = ms
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t[0])
    return {"config": "256 distinct Leduc DCFR(alpha, beta, gamma) alt solves, "
                      f"{iters} iterations each, split over {ws} rank(s), no collective",
            "solves": len(grid), "solves_per_rank": len(mine), "engine": eng,
            "iterations": iters, "seconds": ms_max / 1e3,
            "solve_iterations_per_s": len(grid) * iters / (ms_max / 1e3)}


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    dist = None
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # comm_nranks in the log
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    device = local
    from paper_2605_14277_b200 import Solver, SolverConfig, native

    desc, kind, variant = WORKLOADS[args.workload]
    bundle = make_bundle(kind)
    cfg = SolverConfig(variant)
    mode = args.mode or ("subtree" if ws > 1 else "single")
    sharded = mode in ("sharded", "subtree")  # one solve over the ranks (strong scaling)

    def make_solver():
        if mode in ("sharded", "subtree"):
            from paper_2605_14277_b200.distributed import nccl_unique_id, sharded_solver, subtree_solver
            if dist is None:  # N = 1: a 1-rank NCCL communicator
                return Solver(bundle, cfg, device=device, engine="levels", subtree=mode == "subtree",
                              shard=(nccl_unique_id(), 0, 1))
            return (subtree_solver if mode == "subtree" else sharded_solver)(bundle, cfg, device=device)
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
        avg = s.averages()
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

    # --- per-kernel roofline, measured inside the timed configuration: a
    # recording copy of the iteration graph (scfr_timeline: every launch's
    # first-CTA start and last-CTA end, %globaltimer).  A launch's own
    # duration gives its achieved GB/s; exclusive spans (launches ordered by
    # end time, each instant belonging to the launch that finishes next)
    # partition the step, so the per-kind sums add up to the graph step.  With
    # overlapped alt iterations the recorded graph is the two-stream body.
    peak, peak_kind = _peaks()
    tl_n = max(3, 3 * args.profile_iters)
    if s.engine == "levels":
        timeline = s.timeline(tl_n)  # (overlapped body when the handle overlaps alt iterations)
        method = (f"in-graph timeline (scfr_timeline, {tl_n} iterations): the longest launch that ran "
                  "alone (no other-stream launch overlapping it); its algorithmic bytes over its own "
                  "first-CTA-start to last-CTA-end duration")
    else:
        # the persistent engines run whole iterations in one launch (no level
        # launches to record): that launch, timed with CUDA events, per iteration
        timeline = []
        for k, v in s.profile(tl_n).items():
            us = v["ms"] * 1e3 / tl_n
            timeline.append({"kind": k, "stream": 0, "bytes": v["bytes"] / tl_n, "start_us": 0.0,
                             "end_us": us, "own_us": us, "excl_us": us})
        method = (f"{s.engine} engine: one launch runs every iteration; its algorithmic bytes per "
                  f"iteration over its CUDA-event time per iteration ({tl_n} iterations; latency-bound, "
                  "state resident on chip)")
    kinds = {}
    for e in timeline:
        k = kinds.setdefault(e["kind"], {"launches": 0, "excl_us": 0.0, "own_us": 0.0, "bytes": 0.0})
        k["launches"] += 1
        k["excl_us"] += e["excl_us"]
        k["own_us"] += e["own_us"]
        k["bytes"] += e["bytes"]
    # the dominant launch: the longest one that ran alone (no launch of the
    # other stream overlapping it: an overlapped launch shares the SMs and
    # HBM with that stream's kernel, so its own duration understates the
    # kernel's bandwidth); the longest overall is reported beside it
    def _alone(e):
        return not any(o is not e and o["stream"] != e["stream"] and o["start_us"] < e["end_us"]
                       and e["start_us"] < o["end_us"] for o in timeline)
    longest = max(timeline, key=lambda e: e["end_us"] - e["start_us"])
    alone = [e for e in timeline if _alone(e)]
    top = max(alone, key=lambda e: e["end_us"] - e["start_us"]) if alone else longest
    dname = top["kind"]
    dur_us = top["end_us"] - top["start_us"]
    achieved = top["bytes"] / (max(dur_us, 1e-6) * 1e3)
    step_bytes = sum(e["bytes"] for e in timeline)
    tl_us = max(e["end_us"] for e in timeline)
    prof = s.profile(args.profile_iters)  # eager launches with CUDA events, for comparison
    d = {"bytes": top["bytes"], "launches": 1}
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            with open(tfile) as fh:
                tj = json.load(fh)
            tw = tj.get(args.workload, {})
            # the longest launch of the kind (ncu_summary.py "<kind>@top"), else the kind's mean
            traffic = tw.get(dname + "@top", tw.get(dname))
        except Exception:
            traffic = None

    copy_ref = size_matched_copy(device, d["bytes"] / max(1, d["launches"]), achieved)
    survey_bytes = survey_step_bytes(bundle, cfg, 4 if args.dtype == "f32" else 8)
    survey_gbs = survey_bytes / (ms_max / args.steps / 1e3) / 1e9

    value = args.steps / (ms_max / 1e3) * (1 if sharded else ws)
    line = {
        "metric": "cfr_iterations_per_sec", "value": value, "unit": "iterations/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (generated game tree)",
        "config": {"workload": desc, "variant": variant, "mode": cfg.mode, "gamma": cfg.gamma,
                   "seqs_per_player": [p.num_seqs for p in bundle.procs],
                   "nnz_U": bundle.payoff.nnz,
                   "parallelism": (f"subtree-sharded tree passes + NCCL root broadcasts x{ws}" if mode == "subtree"
                                   else f"row-sharded payoff SpMV + NCCL all-gather x{ws} (config 4)" if sharded
                                   else f"independent replicas x{ws}" if ws > 1 else "1 gpu"),
                   "l2": "working set > L2 (no flush needed)",
                   "engine": s.engine},
        "gpu_launches": launches,
        "clocks": clocks,
        "e2e": {"value": (1 if sharded else ws) * args.steps / e2e_max, "unit": "iterations/s",
                "h2d_bytes_per_step": (h2d1 - h2d0) / E2E_REPS / args.steps,
                "d2h_bytes_per_step": (d2h1 - d2h0) / E2E_REPS / args.steps,
                "includes": "scfr_create upload + K iterations + average-strategy readback, wall clock; "
                            f"median of {E2E_REPS} repetitions",
                "parts": e2e_parts},
        "roofline": {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak,
                     "size_matched_copy": copy_ref,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_kind,
                     "method": method,
                     "kernel_us": dur_us, "kernel_bytes": top["bytes"],
                     "kernel_alone": top is not longest or _alone(top),
                     "longest_launch": {"kind": longest["kind"], "stream": longest["stream"],
                                        "us": longest["end_us"] - longest["start_us"],
                                        "mb": longest["bytes"] / 1e6,
                                        "frac": longest["bytes"] / (max(longest["end_us"] - longest["start_us"],
                                                                        1e-6) * 1e3) / peak,
                                        "overlapped": not _alone(longest)},
                     "step": {"algorithmic_bytes": step_bytes, "timeline_us": tl_us,
                              "graph_ms_per_step": ms_max / args.steps,
                              "achieved_gbs": step_bytes / (tl_us * 1e3),
                              "frac": step_bytes / (tl_us * 1e3) / peak},
                     "survey_8d": {"algorithmic_bytes_per_step": survey_bytes,
                                   "achieved_gbs": survey_gbs, "frac": survey_gbs / peak,
                                   "note": "SURVEY §8(d) fused compulsory bytes over the graph-timed step; "
                                           "the exact shortcuts (DESIGN §4) skip part of them, so this "
                                           "overstates bandwidth use: frac above uses the bytes the "
                                           "kernels load"},
                     "kernels": {k: {"launches": v["launches"], "excl_us": v["excl_us"], "own_us": v["own_us"],
                                     "mb": v["bytes"] / 1e6,
                                     "gbs": v["bytes"] / (v["own_us"] * 1e3) if v["own_us"] else None}
                                 for k, v in kinds.items()},
                     "launches": [{"kind": e["kind"], "stream": e["stream"], "start_us": round(e["start_us"], 2),
                                   "end_us": round(e["end_us"], 2), "mb": round(e["bytes"] / 1e6, 3)}
                                  for e in timeline],
                     "eager_events": {k: {"launches": v["launches"] // args.profile_iters,
                                          "ms": v["ms"] / args.profile_iters}
                                      for k, v in prof.items()}},
    }
    s.close()
    if not args.no_sweep:
        line["sweep"] = sweep_measure(device, ws, rank, dist, args.sweep_iters)
    if ws == 1 and rank == 0 and not args.no_cpu_baseline:
        best = cpu_best_rate(oracle_bundle(kind), variant, 50, 1, args.cpu_budget, args.dtype)
        line["cpu_baseline"] = {"value": best["value"], "unit": "iterations/s", "cores": best["cores"],
                                "kind": "port", "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
                                "serial_vs_parallel": {str(k): v["iterations_per_s"]
                                                       for k, v in best["runs"].items()},
                                "sample": f"{best['steps']} {args.workload} iterations after 1 warm-up, "
                                          f"{best['seconds']:.1f}s, better of 1 and {os.cpu_count()} threads "
                                          f"(oracle/seqcfr_oracle.c over an oracle-compiled bundle)"}
    if rank == 0 and ws == 1 and not args.no_suite:
        line["per_game"] = per_game_suite(device, not args.no_cpu_baseline)
    if rank == 0:
        line["native_so_loaded"] = loaded_native_libs()
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
    ap.add_argument("--mode", choices=("subtree", "sharded", "replicas", "single"), default=None,
                    help="one solve with subtree-sharded tree passes (default for N>1), one row-sharded "
                         "solve (config 4), independent replicas, or a plain one-GPU handle (default for N=1)")
    ap.add_argument("--no-sweep", action="store_true", help="skip config 5 (the 256-solve sweep)")
    ap.add_argument("--sweep-iters", type=int, default=1000)
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
