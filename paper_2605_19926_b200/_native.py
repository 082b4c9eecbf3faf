"""ctypes binding of the CUDA C-ABI library (include/tilecast_b200.h).

This is the only way the host layer reaches the engine: there is no CPU
fallback and no alternative backend. If the library is missing or stale the
import fails loudly with instructions to build it (``python -c "import
__graft_entry__ as g; g.build()"``).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from . import layout as L

LIB_NAME = "libtilecast_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME
ABI_VERSION = 1

_p = C.c_void_p


class TcTables(C.Structure):
    _fields_ = [(n, _p) for n in (
        "kind", "wcol", "didx", "eat", "dcol", "dlock", "ekind", "ecol", "epx",
        "epy", "spx", "spy", "goal_ent", "dirs", "pal", "door_rgb", "key_rgb",
        "goal_rgb", "med_box", "med_cross", "ceil_rgb", "floor_rgb", "coef",
        "fc", "ic", "legal")] + [(n, C.c_int32) for n in (
        "h", "w", "n_doors", "n_entities", "n_spawns", "n_goals", "n_pal",
        "obs_h", "obs_w")]


STATE_FIELDS = ("px", "py", "dx", "dy", "health", "inv", "t", "rkey", "rctr",
                "done", "agoal", "dopen", "ealive")
OUT_FIELDS = ("frames", "zbuf", "rewards", "dones", "truncs", "events",
              "statuses", "rayinfo", "spritevis")


class TcState(C.Structure):
    _fields_ = [(n, _p) for n in STATE_FIELDS]


class TcOut(C.Structure):
    _fields_ = [(n, _p) for n in OUT_FIELDS]


class TcCounters(C.Structure):
    _fields_ = [("violations", C.c_uint64), ("bad_status", C.c_uint32),
                ("next_env", C.c_uint32), ("ctas_done", C.c_uint32), ("pad", C.c_uint32)]


class TcMappedCall(C.Structure):
    """tc_mapped_call: tc_batch_step_mapped's arguments in one struct."""
    _fields_ = [("spec", _p), ("state_in", _p), ("state_out", _p), ("actions_host", _p),
                ("out", _p), ("n", C.c_int64), ("auto_reset", C.c_int32),
                ("validate", C.c_int32), ("counters_dev", _p), ("results_host", _p),
                ("flag_host", _p), ("stream", _p)]


class TcPipeCall(C.Structure):
    """tc_pipe_call: a mapped step plus the successor's output block and gate."""
    _fields_ = [("step", TcMappedCall), ("next_out", _p), ("gate_dev", _p),
                ("speculate", C.c_int32), ("device", C.c_int32)]


class NativeError(RuntimeError):
    """A C-ABI call returned an error status."""


def ptr(a) -> int | None:
    """Raw data pointer of a numpy array or torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if not a.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return a.data_ptr()


def _load() -> C.CDLL:
    path = os.environ.get("TILECAST_B200_LIB", str(LIB_PATH))
    if not Path(path).exists():
        raise ImportError(
            f"CUDA engine library not built: {path} is missing. Build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` from the repo root "
            "(nvcc, sm_100a). There is no CPU fallback.")
    lib = C.CDLL(path)
    P = C.POINTER
    sig = {
        "tc_abi_version": (C.c_int, []),
        "tc_last_error": (C.c_char_p, []),
        "tc_build_info": (C.c_char_p, []),
        "tc_step_kernel": (C.c_char_p, [_p, C.c_int64]),
        "tc_spec_create": (C.c_int, [P(TcTables), P(_p)]),
        "tc_spec_destroy": (C.c_int, [_p]),
        "tc_batch_kernel": (C.c_int, [_p, P(TcState), _p, P(TcOut), C.c_int64, C.c_int32,
                                      C.c_int32, C.c_int32, _p, _p]),
        "tc_batch_step_into": (C.c_int, [_p, P(TcState), P(TcState), _p, P(TcOut), C.c_int64,
                                         C.c_int32, C.c_int32, _p, _p]),
        "tc_batch_steps": (C.c_int, [_p, P(TcState), P(TcState), _p, _p, C.c_int32, C.c_int64,
                                     C.c_int32, C.c_int32, C.c_int32, _p, _p, C.c_uint32, _p]),
        "tc_multi_step": (C.c_int, [_p, P(TcState), P(TcState), _p, P(TcOut), _p, C.c_int32,
                                    C.c_int32, C.c_int32, _p, _p]),
        "tc_batch_step_host": (C.c_int, [_p, P(TcState), P(TcState), _p, _p, P(TcOut), C.c_int64,
                                         C.c_int32, C.c_int32, _p, _p, _p, _p]),
        "tc_batch_step_mapped": (C.c_int, [_p, P(TcState), P(TcState), _p, P(TcOut), C.c_int64,
                                           C.c_int32, C.c_int32, _p, _p, _p, _p]),
        "tc_batch_step_mapped_call": (C.c_int, [_p]),
        "tc_batch_step_pipelined": (C.c_int, [_p]),
        "tc_pipe_cancel": (C.c_int, []),
        "tc_pipe_reset": (C.c_int, []),
        "tc_pipe_stats": (C.c_int, [_p]),
        "tc_debug_mapped_timing": (C.c_int, [_p, C.c_int32]),
        "tc_debug_pipe_trace": (C.c_int, [_p, C.c_int64, _p]),
        "tc_rollout": (C.c_int, [_p, P(TcState), P(TcOut), C.c_int64, C.c_int64, C.c_int64,
                                 C.c_uint64, C.c_int64, C.c_int32, C.c_int32, _p, _p]),
        "tc_seed_streams": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, _p, _p, _p]),
        "tc_policy_actions": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, C.c_int64,
                                        C.c_int64, _p, C.c_int32, _p, _p]),
        "tc_host_cast_ray": (C.c_int, [_p, _p, _p, C.c_int32, C.c_int32, C.c_double,
                                       C.c_double, C.c_double, C.c_double,
                                       P(C.c_int32), P(C.c_int32), P(C.c_int32),
                                       P(C.c_int32), P(C.c_double), P(C.c_double),
                                       P(C.c_int32)]),
        "tc_host_render_into": (C.c_int, [P(TcTables), C.c_double, C.c_double, C.c_double,
                                          C.c_double, _p, _p, C.c_int32, _p, _p,
                                          P(C.c_int32)]),
        "tc_host_batch_kernel": (C.c_int, [P(TcTables), P(TcState), _p, P(TcOut), C.c_int64,
                                           C.c_int32, C.c_int32, C.c_int32, P(C.c_int64)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    if lib.tc_abi_version() != ABI_VERSION:
        raise ImportError(f"{path} has ABI {lib.tc_abi_version()}, expected {ABI_VERSION}; rebuild")
    return lib


_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = _load()
        # a pipelined step still waiting for its actions would hold the GPU
        # until the watchdog's timeout at interpreter exit
        import atexit
        atexit.register(pipe_cancel)
    return _lib


def pipe_cancel() -> None:
    """Cancel a pending pipelined step launch (batch_step_host with
    ``reuse=True``), if any: its kernel exits without effect. Cheap when
    nothing is pending."""
    if _lib is not None:
        _lib.tc_pipe_cancel()


def pipe_reset() -> None:
    """Cancel a pending pipelined launch and clear the watchdog back-off."""
    lib().tc_pipe_reset()


def pipe_stats() -> dict:
    """Pipelined-step counters of this process."""
    out = (C.c_uint64 * 4)()
    lib().tc_pipe_stats(out)
    return {"released": out[0], "cancelled": out[1], "timeouts": out[2], "pending": out[3]}


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().tc_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed ({rc}): {msg}")


def state_struct(arrays: dict) -> TcState:
    s = TcState()
    for n in STATE_FIELDS:
        setattr(s, n, ptr(arrays[n]))
    return s


def out_struct(arrays: dict) -> TcOut:
    o = TcOut()
    for n in OUT_FIELDS:
        setattr(o, n, ptr(arrays.get(n)))
    return o


# The C header mirrors these; a drift is a build bug, caught at import.
assert (L.ST_OK, L.ST_ESCAPED, L.ST_STEP_BUDGET, L.ST_BAD_ACTION) == (0, 1, 2, 3)
assert (L.MODE_RESET, L.MODE_STEP, L.MAX_ENTITIES, L.MAX_DOORS) == (0, 1, 64, 32)
