"""Small solves through every engine and level-engine mode, for
compute-sanitizer (memcheck / racecheck / synccheck): python
scripts/micro/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, flat_goofspiel, flat_liars_dice  # noqa: E402
from paper_2605_14277_b200 import games as G  # noqa: E402

leduc = GameBundle(G.leduc_poker())
goof3 = GameBundle(flat_goofspiel(3))
liars = GameBundle(flat_liars_dice(3))
cases = [
    ("levels overlapped pcfr+ alt", goof3, SolverConfig("pcfr+"), "levels", {}),
    ("levels sequential dcfr alt", goof3, SolverConfig("dcfr"), "levels", {"SCFR_NO_OVERLAP": "1"}),
    ("levels sim cfr", liars, SolverConfig("cfr", mode="sim"), "levels", {}),
    ("levels pipelined groups", goof3, SolverConfig("pcfr+"), "levels",
     {"SCFR_GROUP_NJ": "0", "SCFR_PIPE_NJ": "0", "SCFR_PIPE_KINDS": "31"}),
    ("persistent (SMEM, out-of-line phases, payoff in SMEM)", leduc, SolverConfig("cfr+"), "persistent", {}),
    ("persistent (SMEM, pcfr+)", leduc, SolverConfig("pcfr+"), "persistent", {}),
    ("persistent (SMEM, inlined, payoff from global)", leduc, SolverConfig("dcfr"), "persistent",
     {"SCFR_SMALL_OOL": "0", "SCFR_NO_SMEM_PAYOFF": "1"}),
    ("persistent grid barrier", leduc, SolverConfig("cfr+"), "persistent_grid", {}),
    ("persistent cluster barrier", leduc, SolverConfig("pcfr+"), "persistent_cluster", {}),
    ("tiled", goof3, SolverConfig("pcfr+"), "tiled", {}),
]
# subtree-sharded mode over a 1-rank NCCL communicator, and its range-restricted launches
from paper_2605_14277_b200.distributed import nccl_unique_id  # noqa: E402
cases += [
    ("subtree world 1", goof3, SolverConfig("pcfr+"), "subtree", {}),
    ("subtree simulated 3 ranks", goof3, SolverConfig("cfr", mode="sim"), "subtree", {"SCFR_SUBTREE_SIM": "3"}),
]
for name, b, cfg, engine, env in cases:
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    if engine == "subtree":
        s = Solver(b, cfg, engine="levels", subtree=True, shard=(nccl_unique_id(), 0, 1))
    else:
        s = Solver(b, cfg, engine=engine)
    s.step(4)
    e, _ = s.exploitability("average")
    s.synchronize()
    print(f"{name}: engine {s.engine} exploitability {e:.6e}", flush=True)
    s.close()
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k)
        else:
            os.environ[k] = v
