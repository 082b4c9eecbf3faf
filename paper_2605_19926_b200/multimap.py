"""Heterogeneous-map batches.

The reference steps a homogeneous batch: every env of one ``batch_kernel``
call shares one spec's tables (``tables.py:251-273``; the limit is stated in
``SPEC.md:408``). A ``MultiMapBatch`` lifts that at the host layer: N envs
split into contiguous groups, group g running spec g. Each group is one
homogeneous sub-batch: one step launch per group per step, issued by ONE
native call (tc_multi_step) onto side streams forked from and joined back
into the caller's stream, so the groups run concurrently and fill each
other's tails. Every group writes into views of ONE set of batch-wide
tensors: frames (N, H, W, 3), rewards, dones, truncs, events. A consumer
sees one (N, ...) observation tensor with no gather copy.

Env i (global index) draws from ``split(from_seed(seed), i)``
(``batch.py:81-85``) whatever its group, so group g's trajectory equals a
homogeneous ``batch_reset(spec_g, n_g, seed, base=offset_g)`` run.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import ctypes as C

import numpy as np
import torch

from . import _native as N
from . import layout as L
from .batch import BatchState, ContractError, _check_host_actions
from .engine import (DeviceOut, DeviceState, device_spec, launch_batch, new_counters,
                     resolve_device, stream_ptr)


def _alloc_outs(n: int, h: int, w: int, device) -> DeviceOut:
    return DeviceOut.alloc(n, h, w, device)


def _view(o: DeviceOut, a: int, b: int) -> DeviceOut:
    return DeviceOut(frames=o.frames[a:b], rewards=o.rewards[a:b], dones=o.dones[a:b],
                     truncs=o.truncs[a:b], events=o.events[a:b], statuses=o.statuses[a:b])


@dataclass
class MultiMapBatch:
    """N envs over several specs (contiguous groups), one output block."""

    groups: tuple[BatchState, ...]
    offsets: tuple[int, ...]
    n: int
    _ob: DeviceOut
    _spare: DeviceOut | None = field(default=None, repr=False)
    _ccache: dict = field(default_factory=dict, repr=False)
    _views: dict = field(default_factory=dict, repr=False)

    @property
    def frames(self) -> torch.Tensor:
        """(N, obs_height, obs_width, 3) uint8 observations of every group."""
        return self._ob.frames

    @property
    def specs(self) -> tuple:
        return tuple(g.spec for g in self.groups)

    def group_of(self, i: int) -> int:
        if not (0 <= i < self.n):
            raise ContractError(f"environment index {i} out of range [0, {self.n})")
        return int(np.searchsorted(np.asarray(self.offsets), i, side="right")) - 1

    def check(self) -> None:
        for g in self.groups:
            g.check()

    def host_states(self) -> list[dict]:
        return [g.host_state() for g in self.groups]


def multi_reset(specs: Sequence, counts: Sequence[int], seed: int, *,
                device=None) -> MultiMapBatch:
    """Reset sum(counts) envs; group g (spec g) holds envs
    [offset_g, offset_g + counts[g])."""
    specs, counts = list(specs), [int(c) for c in counts]
    if not specs or len(specs) != len(counts):
        raise ContractError("specs and counts must be non-empty and of equal length")
    if any(c < 1 for c in counts):
        raise ContractError(f"every group needs >= 1 env, got {counts}")
    shapes = {(s.tables.obs_height, s.tables.obs_width) for s in specs}
    if len(shapes) != 1:
        raise ContractError(f"all specs must share one observation shape, got {sorted(shapes)}")
    (h, w), = shapes
    dev = resolve_device(device)
    n = sum(counts)
    offsets = tuple(int(x) for x in np.concatenate([[0], np.cumsum(counts)[:-1]]))
    ob = _alloc_outs(n, h, w, dev)
    groups = []
    for spec, c, off in zip(specs, counts, offsets):
        ds = device_spec(spec, dev)
        t = spec.tables
        sb = DeviceState.alloc(c, t.n_doors, t.n_entities, dev)
        gob = _view(ob, off, off + c)
        counters = new_counters(dev)
        with torch.cuda.device(dev):
            N.check(N.lib().tc_seed_streams(seed & 0xFFFFFFFFFFFFFFFF, off, c, N.ptr(sb.rkey),
                                            N.ptr(sb.rctr), stream_ptr(dev)), "tc_seed_streams")
        launch_batch(ds, sb, None, gob, c, L.MODE_RESET, False, False, counters)
        groups.append(BatchState(spec=spec, n=c, _ds=ds, _sb=sb, _ob=gob, _counters=counters,
                                 base=off, n_total=n))
    return MultiMapBatch(groups=tuple(groups), offsets=offsets, n=n, _ob=ob)


def _group_arrays(mb: MultiMapBatch, sbs_in, sbs_out, outs):
    """ctypes argument arrays for tc_multi_step, cached per buffer set (a
    reuse=True loop alternates between two)."""
    key = (tuple(id(x) for x in sbs_in), tuple(id(x) for x in sbs_out),
           tuple(id(x) for x in outs))
    hit = mb._ccache.get(key)
    if hit is None:
        g = len(mb.groups)
        hit = (
            (C.c_void_p * g)(*[grp._ds.handle.value for grp in mb.groups]),
            (N.TcState * g)(*[x.c_struct() for x in sbs_in]),
            (N.TcState * g)(*[x.c_struct() for x in sbs_out]),
            (N.TcOut * g)(*[x.c_struct() for x in outs]),
            (C.c_int64 * g)(*[grp.n for grp in mb.groups]),
            (C.c_void_p * g)(*[N.ptr(grp._counters) for grp in mb.groups]),
            (sbs_in, sbs_out, outs),  # keep the keyed objects alive
        )
        if len(mb._ccache) > 8:
            mb._ccache.clear()
        mb._ccache[key] = hit
    return hit


def multi_step(mb: MultiMapBatch, actions, *, validate: bool = False,
               reuse: bool = False) -> tuple[MultiMapBatch, torch.Tensor, torch.Tensor]:
    """Step every env once (auto-reset on); ``actions`` is (N,) with group g's
    actions at [offset_g, offset_g + n_g), each checked against its group's
    action set (host arrays on the host; device tensors in the kernel, raised
    by ``check()``). One native call (tc_multi_step): the groups' step
    launches run concurrently. Returns (next batch, rewards f64[N], dones
    bool[N]) as views of the successor's output block (valid until it is
    recycled by a later ``reuse=True`` step)."""
    dev = mb._ob.frames.device
    if isinstance(actions, torch.Tensor) and actions.is_cuda:
        if actions.shape != (mb.n,):
            raise ContractError(f"actions must have shape ({mb.n},), got {tuple(actions.shape)}")
        acts = actions.to(torch.int64).contiguous()
    else:
        host = actions.cpu().numpy() if isinstance(actions, torch.Tensor) else np.asarray(actions)
        if host.shape != (mb.n,):
            raise ContractError(f"actions must have shape ({mb.n},), got {host.shape}")
        host = np.ascontiguousarray(host, dtype=np.int64)
        for g, off in zip(mb.groups, mb.offsets):
            _check_host_actions(g, host[off:off + g.n])
        acts = torch.from_numpy(host).to(dev)
    h, w = mb._ob.frames.shape[1:3]
    ob = mb._spare if (reuse and mb._spare is not None) else _alloc_outs(mb.n, h, w, dev)
    # per-group views of the output block, made once per block (the cache
    # holds the block itself, so its id cannot be reused while cached)
    cached = mb._views.get(id(ob)) if reuse else None
    outs = cached[1] if cached is not None else [_view(ob, off, off + g.n)
                                                 for g, off in zip(mb.groups, mb.offsets)]
    if reuse:
        mb._views[id(ob)] = (ob, outs)
    sbs_in, sbs_out = [], []
    for g in mb.groups:
        t = g.spec.tables
        sbs_in.append(g._sb)
        sbs_out.append(g._retired[0] if reuse and g._retired
                       else DeviceState.alloc(g.n, t.n_doors, t.n_entities, dev))
    arrs = _group_arrays(mb, sbs_in, sbs_out, outs)
    with torch.cuda.device(dev):
        N.check(N.lib().tc_multi_step(arrs[0], arrs[1], arrs[2], N.ptr(acts), arrs[3], arrs[4],
                                      len(mb.groups), 1, 1 if validate else 0, arrs[5],
                                      stream_ptr(dev)), "tc_multi_step")
    new_groups = tuple(
        BatchState(spec=g.spec, n=g.n, _ds=g._ds, _sb=so, _ob=go, _counters=g._counters,
                   base=g.base, n_total=g.n_total, _retired=(g._sb, g._ob) if reuse else ())
        for g, so, go in zip(mb.groups, sbs_out, outs))
    new = MultiMapBatch(groups=new_groups, offsets=mb.offsets, n=mb.n, _ob=ob,
                        _spare=mb._ob if reuse else None, _ccache=mb._ccache,
                        _views=mb._views if reuse else {})
    if validate:
        new.check()
    return new, ob.rewards, ob.dones.view(torch.bool)
