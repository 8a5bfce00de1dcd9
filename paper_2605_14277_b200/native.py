"""ctypes binding of the in-tree C-ABI library (include/seqcfr_b200.h).

There is no fallback: if ``_lib/libseqcfr_b200.so`` is missing the import of
anything that needs it raises ``NativeLibraryError`` (build it with
``make`` or ``python __graft_entry__.py``).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libseqcfr_b200.so")

OK, EINVAL, EGAME, ENONFINITE, ECUDA, ENOMEM, ENCCL, EOVERFLOW = 0, -1, -2, -3, -4, -5, -6, -7
VARIANT_CODE = {"cfr": 0, "cfr+": 1, "dcfr": 2, "pcfr": 3, "pcfr+": 4}
MODE_CODE = {"sim": 0, "alt": 1}
ENGINE_CODE = {"auto": 0, "levels": 1, "persistent": 2, "persistent_grid": 3, "tiled": 4,
               "persistent_cluster": 5}
ENGINE_NAME = {v: k for k, v in ENGINE_CODE.items()}
DTYPE_CODE = {"f64": 0, "float64": 0, "f32": 1, "float32": 1}
STATE_CODE = {"regrets": 0, "behavior": 1, "accum": 2, "utility": 3}


class NativeLibraryError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


class NcclError(RuntimeError):
    pass


i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
i8p = C.POINTER(C.c_int8)


class Game(C.Structure):
    _fields_ = [("num_nodes", C.c_int64), ("kind", i8p), ("parent", i64p),
                ("child_ptr", i64p), ("child_idx", i64p), ("player", i8p),
                ("infoset", i64p), ("prob", f64p), ("payoff", f64p)]


class Tfsdp(C.Structure):
    _fields_ = [("num_nodes", C.c_int64), ("num_decisions", C.c_int64),
                ("num_seqs", C.c_int64), ("height", C.c_int64), ("degree", C.c_int64),
                ("kind", i8p), ("depth", i64p), ("parent", i64p), ("node_seq", i64p),
                ("seq_node", i64p), ("dp_node", i64p), ("dp_first_seq", i64p),
                ("dp_num_actions", i64p), ("dp_parent_seq", i64p), ("level_starts", i64p),
                ("game_seq", i64p), ("dp_infoset", i64p), ("dp_game_node", i64p)]


class Csr(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("nnz", C.c_int64),
                ("indptr", i64p), ("indices", i64p), ("data", f64p)]


class FlatGameC(C.Structure):
    _fields_ = [("game", Game), ("num_infosets", C.c_int64)]


class ParsedGameC(C.Structure):
    _fields_ = [("flat", FlatGameC), ("name", C.c_char_p), ("labels", C.c_void_p), ("label_off", i64p),
                ("infoset_names", C.c_void_p), ("infoset_off", i64p)]


class KernelStat(C.Structure):
    _fields_ = [("name", C.c_char * 16), ("launches", C.c_int64), ("ms", C.c_double),
                ("bytes", C.c_double)]


class KernelSpan(C.Structure):
    _fields_ = [("name", C.c_char * 16), ("kind", C.c_int32), ("stream", C.c_int32), ("bytes", C.c_double),
                ("start_us", C.c_double), ("end_us", C.c_double)]


class Config(C.Structure):
    _fields_ = [("variant", C.c_int32), ("mode", C.c_int32), ("alpha", C.c_double),
                ("beta", C.c_double), ("gamma", C.c_double), ("batch", C.c_int32),
                ("batch_alpha", f64p), ("batch_beta", f64p), ("batch_gamma", f64p),
                ("engine", C.c_int32), ("dtype", C.c_int32), ("reserved", C.c_int32 * 6)]


_lib = None

_SIGS = {
    "scfr_last_error": ([], C.c_char_p),
    "scfr_abi_version": ([], C.c_int),
    "scfr_compile": ([C.POINTER(Game), C.POINTER(C.c_void_p)], C.c_int),
    "scfr_compiled_tfsdp": ([C.c_void_p, C.c_int, C.POINTER(Tfsdp)], C.c_int),
    "scfr_compiled_payoff": ([C.c_void_p, C.c_int, C.POINTER(Csr)], C.c_int),
    "scfr_compiled_free": ([C.c_void_p], None),
    "scfr_generate_liars_dice": ([C.c_int, C.POINTER(C.POINTER(FlatGameC))], C.c_int),
    "scfr_generate_goofspiel": ([C.c_int, C.POINTER(C.POINTER(FlatGameC))], C.c_int),
    "scfr_flat_game_free": ([C.POINTER(FlatGameC)], None),
    "scfr_parse_game_jsonl": ([C.c_char_p, C.c_int64, C.POINTER(C.POINTER(ParsedGameC)), i64p, i64p], C.c_int),
    "scfr_parsed_game_free": ([C.POINTER(ParsedGameC)], None),
    "scfr_create": ([C.POINTER(Tfsdp), C.POINTER(Tfsdp), C.POINTER(Csr), C.POINTER(Csr),
                     C.POINTER(Config), C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "scfr_nccl_unique_id": ([C.c_char_p], C.c_int),
    "scfr_create_sharded": ([C.POINTER(Tfsdp), C.POINTER(Tfsdp), C.POINTER(Csr), C.POINTER(Csr),
                             C.POINTER(Config), C.c_int, C.c_char_p, C.c_int, C.c_int,
                             C.POINTER(C.c_void_p)], C.c_int),
    "scfr_create_subtree": ([C.POINTER(Tfsdp), C.POINTER(Tfsdp), C.POINTER(Csr), C.POINTER(Csr),
                             C.POINTER(Config), C.c_int, C.c_char_p, C.c_int, C.c_int,
                             C.POINTER(C.c_void_p)], C.c_int),
    "scfr_subtree_plan": ([C.POINTER(Tfsdp), C.POINTER(Tfsdp), C.POINTER(Csr), C.c_int,
                           C.POINTER(C.c_int32), i64p, i64p], C.c_int),
    "scfr_step": ([C.c_void_p, C.c_int64], C.c_int),
    "scfr_set_schedule": ([C.c_void_p, C.c_int, f64p, f64p, f64p, C.c_int64], C.c_int),
    "scfr_engine": ([C.c_void_p, C.POINTER(C.c_int)], C.c_int),
    "scfr_synchronize": ([C.c_void_p], C.c_int),
    "scfr_snapshot": ([C.c_void_p, C.c_int], C.c_int),
    "scfr_iterations": ([C.c_void_p, i64p], C.c_int),
    "scfr_read_average": ([C.c_void_p, C.c_int, C.c_int, f64p], C.c_int),
    "scfr_read_averages": ([C.c_void_p, C.c_int, f64p, f64p], C.c_int),
    "scfr_read_current": ([C.c_void_p, C.c_int, C.c_int, f64p], C.c_int),
    "scfr_read_state": ([C.c_void_p, C.c_int, C.c_int, C.c_int, f64p], C.c_int),
    "scfr_avg_weight": ([C.c_void_p, C.c_int, C.c_int, f64p], C.c_int),
    "scfr_exploitability": ([C.c_void_p, C.c_int, C.c_int, f64p, f64p, f64p], C.c_int),
    "scfr_expected_value": ([C.c_void_p, C.c_int, f64p], C.c_int),
    "scfr_best_response_values": ([C.c_void_p, f64p, f64p, f64p, f64p], C.c_int),
    "scfr_expected_value_of": ([C.c_void_p, f64p, f64p, f64p], C.c_int),
    "scfr_status": ([C.c_void_p, C.POINTER(C.c_int)], C.c_int),
    "scfr_device_bytes": ([C.c_void_p, i64p], C.c_int),
    "scfr_launch_count": ([C.c_void_p, i64p], C.c_int),
    "scfr_last_step_ms": ([C.c_void_p, f64p], C.c_int),
    "scfr_profile_step": ([C.c_void_p, C.c_int64, C.POINTER(KernelStat), C.c_int,
                           C.POINTER(C.c_int)], C.c_int),
    "scfr_timeline": ([C.c_void_p, C.c_int64, C.POINTER(KernelSpan), C.c_int, C.POINTER(C.c_int)],
                      C.c_int),
    "scfr_transfer_bytes": ([i64p, i64p], C.c_int),
    "scfr_destroy": ([C.c_void_p], C.c_int),
}

EXPORTED = tuple(_SIGS)


def lib():
    """Load the native library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"native library not built: {LIB_PATH} is missing (run `make` or "
                f"`python __graft_entry__.py`); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(status: int) -> None:
    if status == OK:
        return
    msg = lib().scfr_last_error().decode(errors="replace")
    if status == EINVAL:
        raise ValueError(msg)
    if status == EGAME:
        from .games import GameValidationError
        raise GameValidationError(msg)
    if status == ENONFINITE:
        raise FloatingPointError(msg)
    if status == ENOMEM:
        raise MemoryError(msg)
    if status == ENCCL:
        raise NcclError(msg)
    if status == EOVERFLOW:
        raise OverflowError(msg)
    raise CudaError(f"[{status}] {msg}")


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def view_i64(p, n: int) -> np.ndarray:
    """Copy n int64 values from a library-owned buffer."""
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    return np.ctypeslib.as_array(p, shape=(n,)).copy()


def view_f64(p, n: int) -> np.ndarray:
    if n == 0:
        return np.zeros(0)
    return np.ctypeslib.as_array(p, shape=(n,)).copy()


def view_i8(p, n: int) -> np.ndarray:
    if n == 0:
        return np.zeros(0, dtype=np.int8)
    return np.ctypeslib.as_array(p, shape=(n,)).copy()


def transfer_bytes() -> tuple[int, int]:
    """Process-wide (h2d, d2h) bytes moved by the library so far."""
    a, b = C.c_int64(), C.c_int64()
    check(lib().scfr_transfer_bytes(C.byref(a), C.byref(b)))
    return int(a.value), int(b.value)
