"""B200-native sequence-form CFR (drop-in for the reference ``seqcfr`` hot path).

The public names mirror the reference package (pkg/__init__.py:11-65): game
model and generators, the compiled ``GameBundle`` / ``DecisionProcess`` /
``CsrMatrix``, ``SolverConfig`` / ``run`` / ``benchmark_iterations`` and the
metrics.  Iterations execute as hand-written sm_100a kernels in the in-tree
native library (``_lib/libseqcfr_b200.so``, C-ABI in
``include/seqcfr_b200.h``).
"""

from .games import (
    BUILTIN_GAMES,
    FlatGame,
    Game,
    GameBuilder,
    GameError,
    GameNode,
    GameParseError,
    GameSizeError,
    GameValidationError,
    goofspiel,
    kuhn_poker,
    leduc_poker,
    liars_dice,
    load_game,
    matching_pennies,
    random_game,
    rock_paper_scissors,
    save_game,
    validate_game,
)
from .compiler import (
    CsrMatrix,
    DecisionProcess,
    GameBundle,
    build_bundle,
    extract_decision_process,
    flat_goofspiel,
    flat_liars_dice,
)
from .metrics import ConvergenceRecord, best_response_values, exploitability, expected_value, records_to_csv
from .solvers import (
    VARIANTS,
    IterationBenchmark,
    RunResult,
    Solver,
    SolverConfig,
    TargetResult,
    benchmark_iterations,
    solve_to_target,
    discount_factors,
    run,
    work_per_iteration,
)

__version__ = "0.1.0"

__all__ = [
    "BUILTIN_GAMES", "ConvergenceRecord", "CsrMatrix", "DecisionProcess", "FlatGame", "Game",
    "GameBuilder", "GameBundle", "GameError", "GameNode", "GameParseError", "GameSizeError",
    "GameValidationError", "IterationBenchmark", "RunResult", "Solver", "SolverConfig",
    "VARIANTS", "benchmark_iterations", "best_response_values", "build_bundle",
    "discount_factors", "exploitability", "expected_value", "extract_decision_process",
    "flat_goofspiel", "flat_liars_dice", "goofspiel", "kuhn_poker", "leduc_poker",
    "liars_dice", "load_game", "matching_pennies", "random_game", "records_to_csv",
    "rock_paper_scissors", "run", "save_game", "solve_to_target", "TargetResult",
    "validate_game", "work_per_iteration",
]
