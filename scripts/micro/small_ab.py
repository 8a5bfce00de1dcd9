"""A/B of the SMEM engine on Kuhn / Leduc: us/iter with and without an env
switch (alternating, 3 rounds), e.g. SCFR_NO_SMEM_PAYOFF=1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_14277_b200 import GameBundle, Solver, SolverConfig, kuhn_poker, leduc_poker  # noqa: E402

switch = sys.argv[1] if len(sys.argv) > 1 else "SCFR_NO_SMEM_PAYOFF"
games = {"kuhn": GameBundle(kuhn_poker()), "leduc": GameBundle(leduc_poker())}
for rnd in range(3):
    for name, variant, mode in (("kuhn", "cfr", "sim"), ("leduc", "cfr+", "alt"), ("leduc", "pcfr+", "alt")):
        row = []
        for on in (False, True):
            if on:
                os.environ[switch] = "1"
            else:
                os.environ.pop(switch, None)
            s = Solver(games[name], SolverConfig(variant, mode=mode))
            s.step(200)
            s.synchronize()
            s.step(2000)
            s.synchronize()
            row.append(s.last_step_ms() * 1e3 / 2000)
            s.close()
        print(f"round {rnd} {name:5s} {variant:5s} {mode}: base {row[0]:7.2f}  {switch}=1 {row[1]:7.2f} us/iter", flush=True)
