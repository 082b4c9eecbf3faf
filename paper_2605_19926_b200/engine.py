"""Device-resident engine plumbing: per-spec handles, SoA state/output blocks.

The reference keeps state in a host ``StateBlock`` and outputs in an
``OutBlock`` (/root/reference/pkg/src/tilecast/tables.py:187-245). Here the
same arrays, same dtypes and same [env, ...] layout live in HBM as torch
tensors (torch is only the allocator / stream provider), and every call goes
through the C ABI in ``_native``. u64 / u32 fields are held in int64 / int32
storage and reinterpreted bit-for-bit on the host.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, fields

import numpy as np
import torch

from . import _native as N
from .tables import Tables

_spec_lock = threading.Lock()
_spec_cache: dict = {}


def resolve_device(device=None) -> torch.device:
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("tilecast_b200 needs a CUDA device (B200, sm_100a); "
                               "there is no CPU fallback")
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise RuntimeError(f"tilecast_b200 runs on CUDA devices only, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class DeviceSpec:
    """Packed, device-resident tables of one spec on one GPU (tc_spec*)."""

    def __init__(self, tables: Tables, device: torch.device):
        self.tables = tables
        self.device = device
        handle = N.C.c_void_p()
        with torch.cuda.device(device):
            N.check(N.lib().tc_spec_create(N.C.byref(tables.c_struct()), N.C.byref(handle)),
                    "tc_spec_create")
        self.handle = handle

    def __del__(self):  # pragma: no cover - interpreter teardown order varies
        h = getattr(self, "handle", None)
        if h is not None and h.value and N._lib is not None:
            try:
                with torch.cuda.device(self.device):
                    N._lib.tc_spec_destroy(h)
            except Exception:
                pass


def device_spec(spec, device: torch.device) -> DeviceSpec:
    key = (spec, device.index)
    with _spec_lock:
        ds = _spec_cache.get(key)
        if ds is None:
            ds = DeviceSpec(spec.tables, device)
            _spec_cache[key] = ds
        return ds


@dataclass
class DeviceState:
    """StateBlock in HBM (tables.py:187-215)."""

    px: torch.Tensor
    py: torch.Tensor
    dx: torch.Tensor
    dy: torch.Tensor
    health: torch.Tensor
    inv: torch.Tensor
    t: torch.Tensor
    rkey: torch.Tensor   # u64 bits in int64 storage
    rctr: torch.Tensor   # u64 bits in int64 storage
    done: torch.Tensor
    agoal: torch.Tensor
    dopen: torch.Tensor
    ealive: torch.Tensor

    @staticmethod
    def alloc(n: int, n_doors: int, n_entities: int, device) -> DeviceState:
        f64 = dict(dtype=torch.float64, device=device)
        return DeviceState(
            px=torch.zeros(n, **f64), py=torch.zeros(n, **f64), dx=torch.zeros(n, **f64),
            dy=torch.zeros(n, **f64), health=torch.zeros(n, **f64),
            inv=torch.zeros(n, dtype=torch.uint8, device=device),
            t=torch.zeros(n, dtype=torch.int64, device=device),
            rkey=torch.zeros(n, dtype=torch.int64, device=device),
            rctr=torch.zeros(n, dtype=torch.int64, device=device),
            done=torch.zeros(n, dtype=torch.uint8, device=device),
            agoal=torch.zeros(n, dtype=torch.int32, device=device),
            dopen=torch.zeros((n, n_doors), dtype=torch.uint8, device=device),
            ealive=torch.zeros((n, n_entities), dtype=torch.uint8, device=device))

    def tensors(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}

    def copy_from(self, other: DeviceState) -> None:
        for f in fields(self):
            getattr(self, f.name).copy_(getattr(other, f.name), non_blocking=True)

    def to_host(self) -> dict:
        """numpy copies with the reference's dtypes (u64 / u32 reinterpreted)."""
        out = {f.name: getattr(self, f.name).cpu().numpy() for f in fields(self)}
        out["rkey"] = out["rkey"].view(np.uint64)
        out["rctr"] = out["rctr"].view(np.uint64)
        return out

    def c_struct(self) -> N.TcState:
        # the tensors of a block never change identity: build the struct once
        c = self.__dict__.get("_c")
        if c is None:
            c = N.state_struct(self.tensors())
            self.__dict__["_c"] = c
        return c


@dataclass
class DeviceOut:
    """OutBlock in HBM (tables.py:223-245) plus optional debug taps."""

    frames: torch.Tensor
    rewards: torch.Tensor
    dones: torch.Tensor
    truncs: torch.Tensor
    events: torch.Tensor     # u32 bits in int32 storage
    statuses: torch.Tensor
    zbuf: torch.Tensor | None = None
    rayinfo: torch.Tensor | None = None
    spritevis: torch.Tensor | None = None

    @staticmethod
    def alloc(n: int, obs_h: int, obs_w: int, device, debug: bool = False) -> DeviceOut:
        # rewards (f64) and dones (u8) share one allocation so a host read of
        # a step's results is a single D2H copy
        res = torch.zeros(n * 9, dtype=torch.uint8, device=device)
        o = DeviceOut(
            frames=torch.empty((n, obs_h, obs_w, 3), dtype=torch.uint8, device=device),
            rewards=res[:8 * n].view(torch.float64),
            dones=res[8 * n:],
            truncs=torch.zeros(n, dtype=torch.uint8, device=device),
            events=torch.zeros(n, dtype=torch.int32, device=device),
            statuses=torch.zeros(n, dtype=torch.int32, device=device))
        if debug:
            o.zbuf = torch.zeros((n, obs_w), dtype=torch.float64, device=device)
            o.rayinfo = torch.zeros((n, obs_w, 4), dtype=torch.int32, device=device)
            o.spritevis = torch.zeros(n, dtype=torch.int64, device=device)
        return o

    def tensors(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}

    def c_struct(self) -> N.TcOut:
        c = self.__dict__.get("_c")
        if c is None:
            c = N.out_struct(self.tensors())
            self.__dict__["_c"] = c
        return c


def new_counters(device) -> torch.Tensor:
    """tc_counters (24 bytes, zeroed) accumulated on device, read lazily."""
    return torch.zeros(3, dtype=torch.int64, device=device)


def read_counters(c: torch.Tensor) -> tuple[int, int]:
    v = c.cpu().numpy()
    return int(v[0]), int(v[1]) & 0xFFFFFFFF


def launch_step_into(ds: DeviceSpec, st_in: DeviceState, st_out: DeviceState,
                     actions: torch.Tensor, out: DeviceOut, n: int, auto_reset: bool,
                     validate: bool, counters: torch.Tensor | None) -> None:
    """One fused step reading st_in and writing st_out (tc_batch_step_into)."""
    with torch.cuda.device(ds.device):
        N.check(N.lib().tc_batch_step_into(
            ds.handle, N.C.byref(st_in.c_struct()), N.C.byref(st_out.c_struct()),
            N.ptr(actions), N.C.byref(out.c_struct()), n, 1 if auto_reset else 0,
            1 if validate else 0, N.ptr(counters), stream_ptr(ds.device)), "tc_batch_step_into")


def launch_batch(ds: DeviceSpec, st: DeviceState, actions: torch.Tensor | None,
                 out: DeviceOut, n: int, mode: int, auto_reset: bool, validate: bool,
                 counters: torch.Tensor | None) -> None:
    with torch.cuda.device(ds.device):
        N.check(N.lib().tc_batch_kernel(
            ds.handle, N.C.byref(st.c_struct()), N.ptr(actions), N.C.byref(out.c_struct()),
            n, mode, 1 if auto_reset else 0, 1 if validate else 0, N.ptr(counters),
            stream_ptr(ds.device)), "tc_batch_kernel")
