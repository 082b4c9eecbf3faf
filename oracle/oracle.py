"""Python driver for the oracle port (oracle/tilecast_oracle.c).

TEST INFRASTRUCTURE ONLY -- the checker, never the product. Allowed callers:
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs. It runs the reference's algorithm on the CPU over host numpy
blocks laid out exactly like the reference's StateBlock / OutBlock
(/root/reference/pkg/src/tilecast/tables.py:187-245).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "libtcoracle.so"

_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        from paper_2605_19926_b200._native import TcOut, TcState, TcTables
        L = C.CDLL(str(LIB))
        P, p = C.POINTER, C.c_void_p
        L.orc_batch_kernel.restype = C.c_int64
        L.orc_batch_kernel.argtypes = [P(TcTables), P(TcState), p, P(TcOut), C.c_int64,
                                       C.c_int32, C.c_int32, C.c_int32, C.c_int32]
        L.orc_render_into.restype = C.c_int
        L.orc_render_into.argtypes = [P(TcTables), C.c_double, C.c_double, C.c_double,
                                      C.c_double, p, p, C.c_int32, p, p, p, p]
        L.orc_cast_ray.restype = C.c_int
        L.orc_cast_ray.argtypes = [p, p, p, C.c_int32, C.c_int32, C.c_double, C.c_double,
                                   C.c_double, C.c_double, p, p]
        L.orc_seed_streams.restype = None
        L.orc_seed_streams.argtypes = [C.c_uint64, C.c_int64, C.c_int64, p, p]
        L.orc_policy_actions.restype = None
        L.orc_policy_actions.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64,
                                         C.c_int64, p, C.c_int32, p]
        L.orc_max_threads.restype = C.c_int
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().orc_max_threads())


def alloc_state(n: int, n_doors: int, n_entities: int) -> dict:
    return dict(px=np.zeros(n), py=np.zeros(n), dx=np.zeros(n), dy=np.zeros(n),
                health=np.zeros(n), inv=np.zeros(n, np.uint8), t=np.zeros(n, np.int64),
                rkey=np.zeros(n, np.uint64), rctr=np.zeros(n, np.uint64),
                done=np.zeros(n, np.uint8), agoal=np.zeros(n, np.int32),
                dopen=np.zeros((n, n_doors), np.uint8),
                ealive=np.zeros((n, n_entities), np.uint8))


def alloc_out(n: int, obs_h: int, obs_w: int, debug: bool = False) -> dict:
    o = dict(frames=np.zeros((n, obs_h, obs_w, 3), np.uint8),
             rewards=np.zeros(n), dones=np.zeros(n, np.uint8), truncs=np.zeros(n, np.uint8),
             events=np.zeros(n, np.uint32), statuses=np.zeros(n, np.int32))
    if debug:
        o.update(zbuf=np.zeros((n, obs_w)), rayinfo=np.zeros((n, obs_w, 4), np.int32),
                 spritevis=np.zeros(n, np.uint64))
    return o


def batch_kernel(tables, state: dict, actions, out: dict, mode: int, auto_reset: bool = False,
                 validate: bool = False, n_threads: int | None = None) -> int:
    """The reference's batch_kernel (_pycore.py:346-387) on the CPU."""
    from paper_2605_19926_b200._native import out_struct, ptr, state_struct
    n = state["px"].shape[0]
    nt = n_threads if n_threads is not None else int(os.environ.get("OMP_NUM_THREADS", 0) or
                                                     max_threads())
    acts = None if actions is None else np.ascontiguousarray(actions, dtype=np.int64)
    return int(lib().orc_batch_kernel(
        C.byref(tables.c_struct()), C.byref(state_struct(state)), ptr(acts),
        C.byref(out_struct(out)), n, mode, int(auto_reset), int(validate), nt))


def seed_streams(seed: int, base: int, n: int, state: dict) -> None:
    lib().orc_seed_streams(seed & ((1 << 64) - 1), base, n, state["rkey"].ctypes.data,
                           state["rctr"].ctypes.data)


def policy_actions(policy_key: int, step: int, n_total: int, base: int, n: int,
                   tags: np.ndarray) -> np.ndarray:
    out = np.zeros(n, np.int64)
    tags = np.ascontiguousarray(tags, dtype=np.int64)
    lib().orc_policy_actions(policy_key, step, n_total, base, n, tags.ctypes.data,
                             tags.shape[0], out.ctypes.data)
    return out


def cast_ray(kind, didx, dopen, ox, oy, rx, ry):
    """(status, mapx, mapy, side, perp, wall_u, steps), _pycore.py:38-96."""
    i4 = np.zeros(4, np.int32)
    d2 = np.zeros(2)
    dopen = np.ascontiguousarray(dopen if dopen is not None and len(dopen) else
                                 np.zeros(1, np.uint8), dtype=np.uint8)
    st = lib().orc_cast_ray(kind.ctypes.data, didx.ctypes.data, dopen.ctypes.data,
                            kind.shape[0], kind.shape[1], ox, oy, rx, ry, i4.ctypes.data,
                            d2.ctypes.data)
    return int(st), int(i4[0]), int(i4[1]), int(i4[2]), float(d2[0]), float(d2[1]), int(i4[3])


def render_into(tables, px, py, dx, dy, dopen_row, ealive_row, agoal):
    """(status, frame, zbuf, rayinfo, spritevis), _pycore.py:132-271."""
    frame = np.zeros((tables.obs_height, tables.obs_width, 3), np.uint8)
    zbuf = np.zeros(tables.obs_width)
    ray = np.zeros((tables.obs_width, 4), np.int32)
    vis = np.zeros(1, np.uint64)
    dop = np.ascontiguousarray(dopen_row, dtype=np.uint8)
    eal = np.ascontiguousarray(ealive_row, dtype=np.uint8)
    st = lib().orc_render_into(C.byref(tables.c_struct()), px, py, dx, dy,
                               dop.ctypes.data if dop.size else None,
                               eal.ctypes.data if eal.size else None, agoal,
                               frame.ctypes.data, zbuf.ctypes.data, ray.ctypes.data,
                               vis.ctypes.data)
    return int(st), frame, zbuf, ray, int(vis[0])


class Rollout:
    """batch_reset + batch_step(auto_reset) over host blocks, reference order
    (batch.py:71-138), for tests and the CPU baseline."""

    def __init__(self, spec, n: int, seed: int, base: int = 0, debug: bool = False,
                 n_threads: int | None = None):
        t = spec.tables
        self.tables, self.n, self.n_threads = t, n, n_threads
        self.state = alloc_state(n, t.n_doors, t.n_entities)
        self.out = alloc_out(n, t.obs_height, t.obs_width, debug)
        seed_streams(seed, base, n, self.state)
        batch_kernel(t, self.state, None, self.out, 0, n_threads=n_threads)

    def step(self, actions, validate: bool = False) -> int:
        return batch_kernel(self.tables, self.state, actions, self.out, 1, auto_reset=True,
                            validate=validate, n_threads=self.n_threads)
