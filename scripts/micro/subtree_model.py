"""Subtree-sharded mode on one B200: parity with the one-GPU handle at world 1
over real NCCL, and the per-rank iteration time of a W-rank plan measured by
launching exactly one rank's ranges (SCFR_SUBTREE_VIEW="W,r": timing only, no
exchange).  The projected N-GPU iteration is max_r(view time) + the NCCL root
exchanges.

usage: python scripts/micro/subtree_model.py [--game goof5] [--variant pcfr+] [--iters 200]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, flat_goofspiel  # noqa: E402
from paper_2605_14277_b200.distributed import nccl_unique_id, subtree_plan  # noqa: E402


def us_per_iter(make, iters, reps=5):
    s = make()
    s.step(20)
    s.synchronize()
    best = []
    for _ in range(reps):
        s.step(iters)
        s.synchronize()
        best.append(s.last_step_ms() * 1e3 / iters)
    return float(np.median(best)), s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cards", type=int, default=5)
    ap.add_argument("--variant", default="pcfr+")
    ap.add_argument("--mode", default="alt")
    ap.add_argument("--iters", type=int, default=200)
    a = ap.parse_args()
    b = GameBundle(flat_goofspiel(a.cards))
    cfg = SolverConfig(a.variant, mode=a.mode)
    out = {"game": f"goofspiel_{a.cards}", "variant": a.variant, "mode": a.mode}
    t1, s1 = us_per_iter(lambda: Solver(b, cfg), a.iters)
    out["one_gpu_us"] = t1
    os.environ["SCFR_NO_OVERLAP"] = "1"
    tseq, _ = us_per_iter(lambda: Solver(b, cfg), a.iters)
    del os.environ["SCFR_NO_OVERLAP"]
    out["one_gpu_sequential_us"] = tseq
    mk = lambda: Solver(b, cfg, engine="levels", subtree=True, shard=(nccl_unique_id(), 0, 1))  # noqa: E731
    tw1, sw = us_per_iter(mk, a.iters)
    out["subtree_world1_us"] = tw1
    # parity at world 1: same number of iterations on both handles
    s1.synchronize()
    n1 = s1.iterations
    ref = Solver(b, cfg)
    ref.step(n1)
    sw2 = mk()
    sw2.step(n1)
    same = all(np.array_equal(f(ref), f(sw2)) for f in (lambda s: s.regrets(1), lambda s: s.regrets(2),
                                                         lambda s: s.average(1), lambda s: s.average(2)))
    out["world1_bit_exact_vs_one_gpu"] = bool(same)
    out["views"] = {}
    for W in (2, 4, 8):
        plan = subtree_plan(b, W)
        seqs = [plan["seqs"][0][r] + plan["seqs"][1][r] for r in range(W)]
        per = []
        for r in range(W):
            os.environ["SCFR_SUBTREE_VIEW"] = f"{W},{r}"
            t, _ = us_per_iter(mk, a.iters, reps=3)
            per.append(t)
        del os.environ["SCFR_SUBTREE_VIEW"]
        out["views"][W] = {"per_rank_us": per, "max_us": max(per), "seq_share": max(seqs) / sum(seqs),
                           "cuts": plan["cuts"]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
