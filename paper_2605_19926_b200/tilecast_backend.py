"""Drop-in kernel backend for the reference package, over the C ABI.

The reference selects its kernel module through
``tilecast.backend.set_backend`` (/root/reference/pkg/src/tilecast/backend/__init__.py:28-57);
a backend module exports ``BACKEND_NAME``, ``cast_ray``, ``render_into`` and
``batch_kernel`` with the argument lists of ``_core.pyx:683-763`` (spelled once
in tables.py:257-266). This module implements exactly that interface on top
of ``libtilecast_b200.so``: numpy buffers in, the same buffers mutated / filled
out, with host<->device copies around one launch of the CUDA step kernel.

Installing it as ``tilecast.backend._core`` (see INTEGRATION.md and
tests/ref_shim.py) makes the reference's own API -- and its own test suite --
run on the B200 kernel unmodified.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import torch

from . import _native as N
from . import layout as L

BACKEND_NAME = "compiled"  # the name the reference's tests require (test_backends.py:35)

_TABLE_ORDER = ("kind", "wcol", "didx", "eat", "dcol", "dlock", "ekind", "ecol", "epx",
                "epy", "spx", "spy", "goal_ent", "dirs", "pal", "door_rgb", "key_rgb",
                "goal_rgb", "med_box", "med_cross", "ceil_rgb", "floor_rgb", "coef", "fc",
                "ic")
_STATE_ORDER = ("px", "py", "dx", "dy", "health", "inv", "t", "rkey", "rctr", "done",
                "agoal", "dopen", "ealive")

_lock = threading.Lock()
_specs: dict = {}
_ALL_LEGAL = np.ones(L.A_COUNT, dtype=np.uint8)


def _c(a: np.ndarray, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


class _Tables:
    """Adapter giving a reference table tuple the c_struct() of our Tables."""

    def __init__(self, arrays: dict, obs_h: int, obs_w: int):
        self.a = arrays
        self.obs_h, self.obs_w = obs_h, obs_w

    def c_struct(self) -> N.TcTables:
        s = N.TcTables()
        for k, v in self.a.items():
            setattr(s, k, N.ptr(v) if v.size else None)
        s.legal = N.ptr(_ALL_LEGAL)
        a = self.a
        s.h, s.w = a["kind"].shape
        s.n_doors, s.n_entities = a["dcol"].shape[0], a["ekind"].shape[0]
        s.n_spawns, s.n_goals = a["spx"].shape[0], a["goal_ent"].shape[0]
        s.n_pal = a["pal"].shape[0]
        s.obs_h, s.obs_w = self.obs_h, self.obs_w
        return s


def _tables(arrays: tuple, obs_h: int, obs_w: int) -> _Tables:
    dt = (np.uint8, np.uint8, np.int16, np.int16, np.uint8, np.uint8, np.uint8, np.uint8,
          np.float64, np.float64, np.float64, np.float64, np.int32, np.float64, np.uint8,
          np.uint8, np.uint8, np.uint8, np.uint8, np.uint8, np.uint8, np.uint8, np.float64,
          np.float64, np.int64)
    return _Tables({k: _c(a, t) for k, a, t in zip(_TABLE_ORDER, arrays, dt)}, obs_h, obs_w)


def _device_spec(arrays: tuple, obs_h: int, obs_w: int):
    """tc_spec* cached per table set (the reference's tables are immutable,
    tables.py:179-182, and live as long as their EnvSpec)."""
    from .engine import resolve_device
    key = (tuple((a.__array_interface__["data"][0], a.shape) for a in arrays), obs_h, obs_w)
    with _lock:
        hit = _specs.get(key)
        if hit is not None:
            return hit
        dev = resolve_device()
        tb = _tables(arrays, obs_h, obs_w)
        handle = C.c_void_p()
        with torch.cuda.device(dev):
            N.check(N.lib().tc_spec_create(C.byref(tb.c_struct()), C.byref(handle)),
                    "tc_spec_create")
        hit = (handle, dev, tb, arrays)  # keep the arrays alive with the key
        _specs[key] = hit
        return hit


def cast_ray(kind, didx, dopen, ox, oy, rx, ry):
    """(status, mapx, mapy, side, perp, wall_u, steps) -- _core.pyx:683-691."""
    kind, didx = _c(kind, np.uint8), _c(didx, np.int16)
    dopen = _c(dopen, np.uint8)
    st, mx, my, sd, steps = (C.c_int32() for _ in range(5))
    perp, wu = C.c_double(), C.c_double()
    N.check(N.lib().tc_host_cast_ray(
        N.ptr(kind), N.ptr(didx), N.ptr(dopen) if dopen.size else None, kind.shape[0],
        kind.shape[1], float(ox), float(oy), float(rx), float(ry), C.byref(st), C.byref(mx),
        C.byref(my), C.byref(sd), C.byref(perp), C.byref(wu), C.byref(steps)),
        "tc_host_cast_ray")
    return st.value, mx.value, my.value, sd.value, perp.value, wu.value, steps.value


def render_into(kind, wcol, didx, dcol, ekind, ecol, epx, epy, pal, door_rgb, key_rgb,
                goal_rgb, med_box, med_cross, ceil_rgb, floor_rgb, coef, fc,
                px, py, dx, dy, dopen_row, ealive_row, agoal, frame, zbuf):
    """Render one frame into `frame` / `zbuf`; returns the status -- _core.pyx:694-712."""
    n_doors = np.asarray(dcol).shape[0]
    # tables the render path does not read get neutral placeholders
    arrays = (kind, wcol, didx, np.full(np.asarray(kind).shape, -1, np.int16), dcol,
              np.zeros(n_doors, np.uint8), ekind, ecol, epx, epy, np.array([0.5]),
              np.array([0.5]), np.zeros(0, np.int32), np.zeros((4, 2)), pal, door_rgb,
              key_rgb, goal_rgb, med_box, med_cross, ceil_rgb, floor_rgb, coef, fc,
              np.array([1, 0, 0], np.int64))
    tb = _tables(arrays, frame.shape[0], frame.shape[1])
    out_frame = np.zeros(frame.shape, np.uint8)
    out_z = np.zeros(frame.shape[1])
    st = C.c_int32()
    dop = _c(dopen_row, np.uint8)
    eal = _c(ealive_row, np.uint8)
    N.check(N.lib().tc_host_render_into(
        C.byref(tb.c_struct()), float(px), float(py), float(dx), float(dy),
        N.ptr(dop) if dop.size else None, N.ptr(eal) if eal.size else None, int(agoal),
        N.ptr(out_frame), N.ptr(out_z), C.byref(st)), "tc_host_render_into")
    frame[...] = out_frame
    zbuf[...] = out_z
    return st.value


def batch_kernel(*args):
    """Reset (mode 0) or step (mode 1) envs 0..n-1 in place; returns the
    collision-invariant violation count -- _core.pyx:715-763 / _pycore.py:346-387.
    n_threads is accepted and ignored (results never depend on it)."""
    tables = args[:25]
    state = dict(zip(_STATE_ORDER, args[25:38]))
    actions, frames, zbuf, rewards, dones, truncs, events, statuses = args[38:46]
    mode, auto_reset, validate, _n_threads = args[46:50]
    n = state["px"].shape[0]
    handle, dev, _tb, _keep = _device_spec(tables, frames.shape[1], frames.shape[2])
    with torch.cuda.device(dev):
        ts = {}
        for k, a in state.items():
            h = np.ascontiguousarray(a)
            if h.dtype == np.uint64:
                h = h.view(np.int64)
            ts[k] = torch.from_numpy(h).to(dev)
        outs = {
            "frames": torch.empty(frames.shape, dtype=torch.uint8, device=dev),
            "zbuf": torch.empty(zbuf.shape, dtype=torch.float64, device=dev),
            "rewards": torch.zeros(n, dtype=torch.float64, device=dev),
            "dones": torch.zeros(n, dtype=torch.uint8, device=dev),
            "truncs": torch.zeros(n, dtype=torch.uint8, device=dev),
            "events": torch.zeros(n, dtype=torch.int32, device=dev),
            "statuses": torch.zeros(n, dtype=torch.int32, device=dev),
        }
        acts = None
        if mode == L.MODE_STEP:
            acts = torch.from_numpy(np.ascontiguousarray(actions, dtype=np.int64)).to(dev)
        counters = torch.zeros(3, dtype=torch.int64, device=dev)
        N.check(N.lib().tc_batch_kernel(
            handle, C.byref(N.state_struct(ts)), N.ptr(acts), C.byref(N.out_struct(outs)), n,
            int(mode), int(auto_reset), int(validate), N.ptr(counters),
            torch.cuda.current_stream(dev).cuda_stream), "tc_batch_kernel")
        for k, a in state.items():
            h = ts[k].cpu().numpy()
            a[...] = h.view(a.dtype) if a.dtype == np.uint64 else h
        frames[...] = outs["frames"].cpu().numpy()
        zbuf[...] = outs["zbuf"].cpu().numpy()
        statuses[...] = outs["statuses"].cpu().numpy()
        if mode == L.MODE_STEP:
            rewards[...] = outs["rewards"].cpu().numpy()
            dones[...] = outs["dones"].cpu().numpy()
            truncs[...] = outs["truncs"].cpu().numpy()
            events[...] = outs["events"].cpu().numpy().view(np.uint32)
        return int(counters[0].item())
