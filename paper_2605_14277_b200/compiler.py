"""Host side of the tree compiler: Game / FlatGame -> GameBundle.

``GameBundle`` mirrors the reference's (pkg/solvers.py:309-336): both
players' ``DecisionProcess`` objects (same attribute names and values as
pkg/decision_process.py:48-242), the payoff matrix U and its transpose as
``CsrMatrix`` (pkg/kernels.py:33-127).  The arrays come from the native
compiler (csrc/compiler.cpp via ``scfr_compile``), bit-identical to the
reference's; the bundle also keeps the C structs that ``scfr_create``
consumes so a solve does not copy them again.
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import native as N
from .games import FlatGame, Game, validate_game

KIND_DECISION, KIND_OBSERVATION, KIND_END = 0, 1, 2
_KIND_NAMES = {0: "decision", 1: "observation", 2: "end"}


class CsrMatrix:
    """Minimal CSR over float64 (reference pkg/kernels.py:33-127 layout)."""

    __slots__ = ("rows", "cols", "indptr", "indices", "data", "_transpose", "_bundle")

    def __init__(self, rows, cols, indptr, indices, data):
        self.rows, self.cols = int(rows), int(cols)
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(indices, dtype=np.int64)
        self.data = np.ascontiguousarray(data, dtype=np.float64)
        self._transpose = None
        self._bundle = None  # weakref to the GameBundle owning this payoff matrix

    @property
    def nnz(self) -> int:
        return int(self.data.shape[0])

    @property
    def shape(self):
        return (self.rows, self.cols)

    def transposed(self) -> "CsrMatrix":
        return self._transpose

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.rows, self.cols))
        for i in range(self.rows):
            for k in range(self.indptr[i], self.indptr[i + 1]):
                out[i, self.indices[k]] = self.data[k]
        return out

    def nbytes(self) -> int:
        return self.indptr.nbytes + self.indices.nbytes + self.data.nbytes

    def as_c(self) -> N.Csr:
        return N.Csr(self.rows, self.cols, self.nnz, N.ptr(self.indptr, C.c_int64),
                     N.ptr(self.indices, C.c_int64), N.ptr(self.data, C.c_double))

    def __repr__(self) -> str:
        return f"CsrMatrix({self.rows}x{self.cols}, nnz={self.nnz})"


class DecisionProcess:
    """One player's TFSDP with the reference's attributes
    (pkg/decision_process.py:48-65)."""

    _ARRAYS = ("depth", "parent", "node_seq", "seq_node", "dp_node", "dp_first_seq",
               "dp_num_actions", "dp_parent_seq", "level_starts", "game_seq", "dp_infoset",
               "dp_game_node")

    def __init__(self, player: int, view: N.Tfsdp, num_game_nodes: int, flat: FlatGame):
        self.player = player
        self.num_nodes = int(view.num_nodes)
        self.num_decisions = int(view.num_decisions)
        self.num_seqs = int(view.num_seqs)
        self.height = int(view.height)
        self.degree = int(view.degree)
        sizes = {"depth": self.num_nodes, "parent": self.num_nodes, "node_seq": self.num_nodes,
                 "seq_node": self.num_seqs, "dp_node": self.num_decisions,
                 "dp_first_seq": self.num_decisions, "dp_num_actions": self.num_decisions,
                 "dp_parent_seq": self.num_decisions, "level_starts": self.height + 2,
                 "game_seq": num_game_nodes, "dp_infoset": self.num_decisions,
                 "dp_game_node": self.num_decisions}
        for name in self._ARRAYS:
            setattr(self, name, N.view_i64(getattr(view, name), sizes[name]))
        self.kind = N.view_i8(view.kind, self.num_nodes)
        self._flat = flat
        self._labels = None

    # -- derived views (reference pkg/decision_process.py:208-231) ---------
    @property
    def seq_dp(self) -> np.ndarray:
        out = np.full(self.num_seqs, -1, dtype=np.int64)
        out[1:] = np.repeat(np.arange(self.num_decisions), self.dp_num_actions)
        return out

    @property
    def levels(self):
        out = []
        for d in range(1, self.height + 1):
            lo, hi = int(self.level_starts[d]), int(self.level_starts[d + 1])
            parents = self.parent[lo:hi].copy()
            seqs = np.where(self.kind[parents] == KIND_DECISION, self.node_seq[lo:hi] - 1, -1)
            out.append((parents, np.arange(lo, hi, dtype=np.int64), seqs))
        return out

    def _label_tables(self):
        if self._labels is None:
            f = self._flat
            if f.infoset_labels is None:
                dp = [f"I{int(i)}" for i in self.dp_infoset]
                acts = []
                for g in self.dp_game_node:
                    n = int(f.child_ptr[g + 1] - f.child_ptr[g])
                    acts.append(tuple(str(a) for a in range(n)))
            else:
                dp = [f.infoset_labels[int(i)] for i in self.dp_infoset]
                acts = []
                for g in self.dp_game_node:
                    kids = f.child_idx[f.child_ptr[g]:f.child_ptr[g + 1]]
                    acts.append(tuple(f.action_labels[int(c)] for c in kids))
            self._labels = (dp, acts)
        return self._labels

    @property
    def dp_label(self):
        return self._label_tables()[0]

    @property
    def dp_action_labels(self):
        return self._label_tables()[1]

    def seq_label(self, seq: int) -> str:
        if seq == 0:
            return ""
        j = int(np.searchsorted(self.dp_first_seq, seq, side="right") - 1)
        a = seq - int(self.dp_first_seq[j])
        return f"{self.dp_label[j]}/{self.dp_action_labels[j][a]}"

    def uniform_behavior(self) -> np.ndarray:
        return np.repeat(1.0 / self.dp_num_actions, self.dp_num_actions)

    def dump(self) -> str:
        lines = []
        for i in range(self.num_nodes):
            s = int(self.node_seq[i])
            lab = self.seq_label(s) if s > 0 else ("<root>" if s == 0 else "-")
            lines.append(f"{i}\t{_KIND_NAMES[int(self.kind[i])]}\t{int(self.depth[i])}\t"
                         f"{int(self.parent[i])}\t{lab}")
        return "\n".join(lines)

    def as_c(self) -> N.Tfsdp:
        p = lambda a: N.ptr(a, C.c_int64)  # noqa: E731
        return N.Tfsdp(self.num_nodes, self.num_decisions, self.num_seqs, self.height,
                       self.degree, N.ptr(self.kind, C.c_int8), p(self.depth), p(self.parent),
                       p(self.node_seq), p(self.seq_node), p(self.dp_node), p(self.dp_first_seq),
                       p(self.dp_num_actions), p(self.dp_parent_seq), p(self.level_starts),
                       p(self.game_seq), p(self.dp_infoset), p(self.dp_game_node))


def _flat_c(flat: FlatGame) -> N.Game:
    return N.Game(flat.num_nodes, N.ptr(flat.kind, C.c_int8), N.ptr(flat.parent, C.c_int64),
                  N.ptr(flat.child_ptr, C.c_int64), N.ptr(flat.child_idx, C.c_int64),
                  N.ptr(flat.player, C.c_int8), N.ptr(flat.infoset, C.c_int64),
                  N.ptr(flat.prob, C.c_double), N.ptr(flat.payoff, C.c_double))


def compile_flat(flat: FlatGame):
    """Run the native compiler; returns (proc1, proc2, U, UT)."""
    L = N.lib()
    h = C.c_void_p()
    N.check(L.scfr_compile(C.byref(_flat_c(flat)), C.byref(h)))
    try:
        procs = []
        for pl in (1, 2):
            v = N.Tfsdp()
            N.check(L.scfr_compiled_tfsdp(h, pl, C.byref(v)))
            procs.append(DecisionProcess(pl, v, flat.num_nodes, flat))
        mats = []
        for tr in (0, 1):
            m = N.Csr()
            N.check(L.scfr_compiled_payoff(h, tr, C.byref(m)))
            mats.append(CsrMatrix(m.rows, m.cols, N.view_i64(m.indptr, m.rows + 1),
                                  N.view_i64(m.indices, m.nnz), N.view_f64(m.data, m.nnz)))
    finally:
        L.scfr_compiled_free(h)
    mats[0]._transpose, mats[1]._transpose = mats[1], mats[0]
    return procs[0], procs[1], mats[0], mats[1]


def _from_native(gen, param: int, name: str) -> FlatGame:
    L = N.lib()
    out = C.POINTER(N.FlatGameC)()
    N.check(gen(param, C.byref(out)))
    try:
        g = out.contents.game
        n = int(g.num_nodes)
        m = int(np.ctypeslib.as_array(g.child_ptr, shape=(n + 1,))[-1])
        flat = FlatGame(name, N.view_i8(g.kind, n), N.view_i64(g.parent, n),
                        N.view_i64(g.child_ptr, n + 1), N.view_i64(g.child_idx, m),
                        N.view_i8(g.player, n), N.view_i64(g.infoset, n),
                        N.view_f64(g.prob, n), N.view_f64(g.payoff, n))
    finally:
        L.scfr_flat_game_free(out)
    return flat


def flat_liars_dice(faces: int = 6) -> FlatGame:
    """Native generator; same tree as games.liars_dice(faces)."""
    return _from_native(N.lib().scfr_generate_liars_dice, faces, f"liars_dice_1x1x{faces}")


def flat_goofspiel(cards: int = 5) -> FlatGame:
    """Native generator; same tree as games.goofspiel(cards)."""
    return _from_native(N.lib().scfr_generate_goofspiel, cards, f"goofspiel_{cards}")


def load_game_flat(text: str) -> FlatGame:
    """A JSON-lines game file (the reference format, pkg/games.py:554-648)
    read, validated and flattened natively (csrc/jsonl.cpp): the same checks
    and errors as ``games.load_game`` (GameParseError with the line,
    GameValidationError with the node), without building Python node
    objects.  The result feeds ``GameBundle`` directly."""
    from .games import GameParseError, GameValidationError
    raw = text.encode("utf-8")
    out = C.POINTER(N.ParsedGameC)()
    line, node = C.c_int64(-1), C.c_int64(-1)
    L = N.lib()
    status = L.scfr_parse_game_jsonl(raw, len(raw), C.byref(out), C.byref(line), C.byref(node))
    if status == N.EGAME:
        msg = L.scfr_last_error().decode(errors="replace")
        if line.value >= 1:
            raise GameParseError(msg, int(line.value))
        raise GameValidationError(msg, int(node.value) if node.value >= 0 else None)
    N.check(status)
    try:
        pg = out.contents
        g = pg.flat.game
        n = int(g.num_nodes)
        m = int(np.ctypeslib.as_array(g.child_ptr, shape=(n + 1,))[-1])
        flat = FlatGame(pg.name.decode("utf-8"), N.view_i8(g.kind, n), N.view_i64(g.parent, n),
                        N.view_i64(g.child_ptr, n + 1), N.view_i64(g.child_idx, m),
                        N.view_i8(g.player, n), N.view_i64(g.infoset, n),
                        N.view_f64(g.prob, n), N.view_f64(g.payoff, n))
        k = int(pg.flat.num_infosets)

        def strings(base, off, count):
            offs = N.view_i64(off, count + 1)
            blob = C.string_at(base, int(offs[-1])) if count and offs[-1] else b""
            return [blob[offs[i]:offs[i + 1]].decode("utf-8") for i in range(count)]

        flat.infoset_labels = strings(pg.infoset_names, pg.infoset_off, k)
        labels = strings(pg.labels, pg.label_off, n)
        flat.action_labels = [None] + labels[1:]
    finally:
        L.scfr_parsed_game_free(out)
    return flat


class GameBundle:
    """Iteration-invariant structure of one game (pkg/solvers.py:309-336).

    Accepts a ``Game`` (validated with ``validate_game`` unless
    ``validate=False``, like the reference) or a ``FlatGame`` (the native
    generators' output; the compiler itself rejects broken trees and
    perfect-recall violations).
    """

    def __init__(self, game: Game | FlatGame, validate: bool = True):
        if isinstance(game, Game):
            if validate:
                validate_game(game).raise_if_failed()
            self.game = game
            flat = game.flatten()
        elif isinstance(game, FlatGame):
            self.game = None
            flat = game
        else:
            raise TypeError("GameBundle needs a Game or a FlatGame")
        self.flat = flat
        self.name = flat.name
        p1, p2, U, UT = compile_flat(flat)
        self.procs = (p1, p2)
        self.payoff, self.payoff_t = U, UT
        U._bundle = UT._bundle = weakref.ref(self)
        self._c = (p1.as_c(), p2.as_c(), U.as_c(), UT.as_c())
        self._evaluator = None

    @property
    def num_proc_nodes(self) -> int:
        return self.procs[0].num_nodes + self.procs[1].num_nodes

    def reference_nbytes(self) -> int:
        """The reference's GameBundle.nbytes() (pkg/solvers.py:330-332)
        recomputed from the sizes, so ConvergenceRecord.peak_bytes matches."""
        total = 0
        for p in self.procs:
            Nn, Sg, Sp, Jn = p.num_nodes, p.num_seqs, p.num_seqs - 1, p.num_decisions
            ops = (8 * (Nn + 1) + 16 * Sg) + (8 * (Sg + 1) + 16 * Sg)
            ops += (8 * (Nn + 1) + 16 * Sp) + (8 * (Sp + 1) + 16 * Sp)
            ops += (8 * (Jn + 1) + 16 * Sp) + (8 * (Sp + 1) + 16 * Sp) + 8 * Sp
            ls = p.level_starts
            for d in range(1, p.height + 1):
                nd = int(ls[d + 1] - ls[d])
                npar = int(ls[d] - ls[d - 1])
                ops += 56 * nd + 8 * npar + 16
            total += ops
        for m in (self.payoff, self.payoff_t):
            total += 8 * (m.rows + 1) + 16 * m.nnz
        return total

    def reference_state_bytes(self) -> int:
        """Sum of both RegretState.state_bytes() (pkg/solvers.py:136-140)."""
        return sum(8 * (7 * (p.num_seqs - 1) + p.num_seqs + p.num_decisions + 3 * p.num_nodes)
                   for p in self.procs)

    def nbytes(self) -> int:
        return self.reference_nbytes()


def build_bundle(game, validate: bool = True) -> GameBundle:
    return GameBundle(game, validate=validate)


def extract_decision_process(game: Game, player: int) -> DecisionProcess:
    if player not in (1, 2):
        raise ValueError("player must be 1 or 2")
    return GameBundle(game, validate=False).procs[player - 1]
