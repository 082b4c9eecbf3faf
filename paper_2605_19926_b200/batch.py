"""Batched reset/step over N same-spec environments, device resident.

API of the reference's ``tilecast.batch`` (/root/reference/pkg/src/tilecast/batch.py:27-179):
``batch_reset``, ``batch_step`` (auto-reset, ``reuse`` double-buffering,
``validate``), ``policy_actions``, ``throughput_probe``. Differences, all
consequences of keeping the step on the GPU with no host round trip:

* observations, state and per-step outputs are torch CUDA tensors
  (``BatchState.frames`` is ``uint8[N, H, W, 3]`` in HBM);
* ``batch_step`` returns device tensors ``(rewards f64[N], dones bool[N])``;
* per-env engine faults (unsealed maps, illegal actions passed as a device
  tensor) are accumulated in device counters and raised by
  ``BatchState.check()`` -- called by ``state()``/``states`` and, with
  ``validate=True`` or ``sync_checks=True``, by ``batch_step`` itself (the
  reference raises inside every call, tables.py:267-272, batch.py:133-135);
* the per-env RNG split (a host loop in the reference, batch.py:81-85) and
  the policy draw run on the device; they are bit-identical.

Envs can be a shard of a larger batch: ``base`` / ``n_total`` make env i use
the global index ``base + i`` for its reset stream and policy counters, so a
trajectory does not depend on how many GPUs the batch is split over.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from . import _native as N
from . import layout as L
from . import rng
from .dynamics import ACTION_NAMES, Action, EnvState, state_from_arrays
from .engine import (DeviceOut, DeviceSpec, DeviceState, device_spec, launch_batch,
                     launch_step_into, new_counters, read_counters, resolve_device,
                     stream_ptr)
from .geometry import ContractError
from .suite import EnvSpec


@dataclass
class BatchState:
    """N environments' device state plus their observation block.

    With ``reuse=True`` stepping recycles the predecessor's buffers: a state
    is then valid only until its successor is stepped (batch.py:31-34).
    """

    spec: EnvSpec
    n: int
    _ds: DeviceSpec
    _sb: DeviceState
    _ob: DeviceOut
    _counters: torch.Tensor
    base: int = 0
    n_total: int = 0
    _retired: tuple = field(default=(), repr=False)
    _stage: "_ActionStage | None" = field(default=None, repr=False)
    # chained multi-step launches (batch_steps): per-env / per-CTA epoch
    # flags in device memory and the batch's next epoch (one list shared by
    # the whole lineage of states)
    _chain: list = field(default_factory=list, repr=False)

    @property
    def device(self) -> torch.device:
        return self._ds.device

    @property
    def frames(self) -> torch.Tensor:
        """(n, obs_height, obs_width, 3) uint8 observations in HBM."""
        N.pipe_cancel()  # work on these tensors must not queue behind a gated launch
        return self._ob.frames

    def check(self) -> None:
        """Raise for faults accumulated on the device since the batch began."""
        N.pipe_cancel()
        viol, bad = read_counters(self._counters)
        if bad & (1 << L.ST_BAD_ACTION):
            raise ContractError(
                f"an action outside {self.spec.id!r}'s action set reached the device")
        if bad & ((1 << L.ST_ESCAPED) | (1 << L.ST_STEP_BUDGET)):
            raise RuntimeError("render invariant violated: " + (
                "ray escaped the map (unsealed?)" if bad & (1 << L.ST_ESCAPED)
                else "ray exceeded its boundary-step budget"))
        if viol:
            raise RuntimeError(f"collision invariant violated in {viol} environment step(s)")

    def host_state(self) -> dict:
        N.pipe_cancel()
        return self._sb.to_host()

    def state(self, i: int) -> EnvState:
        if not (0 <= i < self.n):
            raise ContractError(f"environment index {i} out of range [0, {self.n})")
        self.check()
        return state_from_arrays(self._sb.to_host(), i)

    @property
    def states(self) -> tuple[EnvState, ...]:
        self.check()
        a = self._sb.to_host()
        return tuple(state_from_arrays(a, i) for i in range(self.n))

    @property
    def last_terminated(self) -> torch.Tensor:
        return (self._ob.dones != 0) & (self._ob.truncs == 0)

    @property
    def last_truncated(self) -> torch.Tensor:
        return self._ob.truncs != 0

    @property
    def last_events(self) -> np.ndarray:
        N.pipe_cancel()
        return self._ob.events.cpu().numpy().view(np.uint32)


class _ActionStage:
    """Two pinned host buffers + device buffers for async action upload.

    A buffer is rewritten only after the event recorded behind its previous
    H2D copy has fired, so no copy ever reads a half-written buffer."""

    def __init__(self, n: int, device: torch.device):
        self.pinned = [torch.empty(n, dtype=torch.int64, pin_memory=True) for _ in range(2)]
        self.dev = [torch.empty(n, dtype=torch.int64, device=device) for _ in range(2)]
        self.events = [torch.cuda.Event() for _ in range(2)]
        self.k = 0
        self.np = [p.numpy() for p in self.pinned]
        # batch_step_host's synchronous staging (actions in, rewards / dones out)
        # results land as [rewards f64[n] | dones u8[n]], one D2H copy
        self._h_act = torch.empty(n, dtype=torch.int64, pin_memory=True)
        self._h_res = torch.empty(9 * n, dtype=torch.uint8, pin_memory=True)
        self.h_act = self._h_act.numpy()
        res = self._h_res.numpy()
        self.h_rew = res[:8 * n].view(np.float64)
        self.h_done = res[8 * n:].view(np.bool_)
        # [0] bad action, [1] results ready, [4] / [5] pipelined gate go /
        # cancel, [6] expired (tc_batch_step_pipelined)
        self._h_flag = torch.zeros(8, dtype=torch.int32, pin_memory=True)
        # the pipelined step's gate lines and result hand-off counters
        self.gate_dev = torch.zeros(4096, dtype=torch.int32, device=device)
        self.h_flag = self._h_flag.numpy()
        self.h_flag_ptr = self._h_flag.data_ptr()
        self.h_act_ptr = self._h_act.data_ptr()
        self.h_rew_ptr = self._h_res.data_ptr()
        self.h_done_ptr = self.h_rew_ptr + 8 * n
        self.dev_ptr = self.dev[0].data_ptr()
        self.calls: dict = {}
        self.fn = None  # cached ctypes entry point of batch_step_host
        self.dev_index = torch.device(device).index

    def __del__(self):
        # a pipelined step launched by this stage may still be waiting at its
        # gate in this stage's pinned words: cancel it and let it exit before
        # the pinned / device buffers go back to torch's allocators
        try:
            if N.pipe_stats()["pending"]:
                N.pipe_cancel()
                torch.cuda.synchronize(self.dev_index)
        except Exception:
            pass

    def next_buffer(self) -> np.ndarray:
        """The next pinned buffer, once the H2D copy that last read it is done."""
        self.k ^= 1
        self.events[self.k].synchronize()
        return self.np[self.k]

    def upload(self) -> torch.Tensor:
        k = self.k
        self.dev[k].copy_(self.pinned[k], non_blocking=True)
        self.events[k].record(torch.cuda.current_stream(self.dev[k].device))
        return self.dev[k]


def batch_reset(spec: EnvSpec, n: int, seed: int, *, device=None, base: int = 0,
                n_total: int | None = None, debug: bool = False) -> BatchState:
    """Reset n envs; env i draws from stream split(from_seed(seed), base + i)."""
    if n < 1:
        raise ContractError(f"batch size must be >= 1, got {n}")
    dev = resolve_device(device)
    ds = device_spec(spec, dev)
    t = spec.tables
    sb = DeviceState.alloc(n, t.n_doors, t.n_entities, dev)
    ob = DeviceOut.alloc(n, t.obs_height, t.obs_width, dev, debug=debug)
    counters = new_counters(dev)
    with torch.cuda.device(dev):
        N.check(N.lib().tc_seed_streams(seed & rng.M64, base, n, N.ptr(sb.rkey),
                                        N.ptr(sb.rctr), stream_ptr(dev)), "tc_seed_streams")
    launch_batch(ds, sb, None, ob, n, L.MODE_RESET, False, False, counters)
    return BatchState(spec=spec, n=n, _ds=ds, _sb=sb, _ob=ob, _counters=counters,
                      base=base, n_total=n_total if n_total is not None else base + n)


def batch_steps(bs: BatchState, actions: torch.Tensor, *, outs: Sequence[DeviceOut] | None = None,
                validate: bool = False) -> BatchState:
    """K consecutive batch_steps (auto-reset) in one native call:
    ``actions`` is a (K, n) int64 CUDA tensor, row k = step k's actions.
    K launches of the step kernel chained at CTA granularity
    (tc_batch_steps: a step's CTAs start as the previous step's CTAs free
    their slots, each env waiting only for its own state), equal to K
    ``batch_step`` calls with ``reuse=True``. ``outs`` is a ring of output
    blocks (step k writes ``outs[k % len(outs)]``; default: a second block,
    then this batch's own block, as ``reuse=True`` recycles it).
    Returns the state after the last step, whose ``frames`` / ``_ob`` are
    that step's output block. The states between are not returned (the two
    state blocks ping-pong)."""
    t = bs.spec.tables
    if not (isinstance(actions, torch.Tensor) and actions.is_cuda and actions.dim() == 2
            and actions.shape[1] == bs.n):
        raise ContractError(f"actions must be a (K, {bs.n}) CUDA tensor")
    acts = actions.to(torch.int64).contiguous()
    k = acts.shape[0]
    if k == 0:
        return bs
    if outs is None:
        other = bs._retired[1] if bs._retired else DeviceOut.alloc(
            bs.n, t.obs_height, t.obs_width, bs.device)
        outs = [other, bs._ob] if k > 1 else [other]  # bs's own block is recycled from step 1
    outs = list(outs)
    sb = bs._retired[0] if bs._retired else DeviceState.alloc(bs.n, t.n_doors, t.n_entities,
                                                               bs.device)
    if not bs._chain:
        # [ready epochs u32[n] | one-wave done epochs, a row of 2048 per ring
        # slot (<= 64) -- or the multi-wave ticket counters u32[n]]
        bs._chain.extend([torch.zeros(bs.n + max(bs.n, 64 * 2048), dtype=torch.int32,
                                      device=bs.device), 1])
    flags, epoch = bs._chain
    ring = (N.TcOut * len(outs))(*[o.c_struct() for o in outs])
    with torch.cuda.device(bs.device):
        N.check(N.lib().tc_batch_steps(
            bs._ds.handle, N.C.byref(bs._sb.c_struct()), N.C.byref(sb.c_struct()), N.ptr(acts),
            ring, len(outs), bs.n, k, 1, 1 if validate else 0, N.ptr(bs._counters),
            N.ptr(flags), epoch & 0xFFFFFFFF, stream_ptr(bs.device)), "tc_batch_steps")
    bs._chain[1] = epoch + k
    final_sb, spare_sb = (sb, bs._sb) if k % 2 == 1 else (bs._sb, sb)
    final_ob = outs[(k - 1) % len(outs)]
    spare_ob = outs[(k - 2) % len(outs)] if len(outs) > 1 else bs._ob
    new = BatchState(spec=bs.spec, n=bs.n, _ds=bs._ds, _sb=final_sb, _ob=final_ob,
                     _counters=bs._counters, base=bs.base, n_total=bs.n_total,
                     _retired=(spare_sb, spare_ob), _stage=bs._stage, _chain=bs._chain)
    if validate:
        new.check()
    return new


def _coerce_actions(bs: BatchState, actions) -> torch.Tensor:
    """Host-side contract checks (batch.py:92-106), then an async H2D copy
    through a pinned staging buffer. CUDA tensors are checked on the device."""
    if isinstance(actions, torch.Tensor) and actions.is_cuda:
        if actions.shape != (bs.n,):
            raise ContractError(f"actions must have shape ({bs.n},), got {tuple(actions.shape)}")
        return actions.to(torch.int64).contiguous()
    if bs._stage is None:
        bs._stage = _ActionStage(bs.n, bs.device)
    host = actions.cpu().numpy() if isinstance(actions, torch.Tensor) else actions
    if not isinstance(host, np.ndarray):
        host = np.asarray(host, dtype=np.int64)
    if host.shape != (bs.n,):
        raise ContractError(f"actions must have shape ({bs.n},), got {host.shape}")
    buf = bs._stage.next_buffer()            # pinned int64[n]; one conversion pass
    np.copyto(buf, host, casting="unsafe")
    if (buf.view(np.uint64) >= L.A_COUNT).any():  # negatives wrap to huge
        raise ContractError(f"action tags must be in [0, {L.A_COUNT})")
    legal = bs.spec.tables.legal
    if not legal.all():
        ok = np.take(legal, buf) != 0
        if not ok.all():
            bad = int(buf[~ok][0])
            names = ", ".join(ACTION_NAMES[a] for a in bs.spec.action_set)
            raise ContractError(f"action {ACTION_NAMES[Action(bad)]!r} is not in "
                                f"{bs.spec.id!r}'s action set ({names})")
    return bs._stage.upload()


def _check_host_actions(bs: BatchState, actions) -> np.ndarray:
    """The reference's host-side action contract (batch.py:92-106), in one
    counting pass over the actions."""
    acts = np.ascontiguousarray(actions, dtype=np.int64)
    if acts.shape != (bs.n,):
        raise ContractError(f"actions must have shape ({bs.n},), got {acts.shape}")
    try:
        counts = np.bincount(acts, minlength=L.A_COUNT)
    except ValueError:  # a negative tag
        raise ContractError(f"action tags must be in [0, {L.A_COUNT})") from None
    if counts.shape[0] > L.A_COUNT:
        raise ContractError(f"action tags must be in [0, {L.A_COUNT})")
    legal = bs.spec.tables.legal
    if (counts[legal == 0] != 0).any():
        ok = np.take(legal, acts) != 0
        bad = int(acts[~ok][0])
        names = ", ".join(ACTION_NAMES[a] for a in bs.spec.action_set)
        raise ContractError(f"action {ACTION_NAMES[Action(bad)]!r} is not in "
                            f"{bs.spec.id!r}'s action set ({names})")
    return acts


PIPELINE_MAX_ENVS = 1 << 16  # batch_step_host pipelines batches up to this size


def batch_step_host(bs: BatchState, actions, *, validate: bool = False,
                    reuse: bool = False, pipeline: bool = True
                    ) -> tuple[BatchState, np.ndarray, np.ndarray]:
    """batch_step with the reference's return types: host actions in, numpy
    ``(rewards f64[N], dones bool[N])`` out (batch.py:136-138), the state and
    frames staying on the GPU. One native call (tc_batch_step_mapped): the
    step kernel reads the actions straight from pinned host memory and its
    last CTA writes rewards / dones back to pinned host memory; no copy-engine
    transfers, one launch, one synchronisation. The reference's action
    contract (batch.py:92-106) is checked by the kernel: a violation leaves
    ``bs`` untouched and raises the reference's ContractError.

    With ``reuse=True`` (and ``pipeline``) the call also launches the next
    step of the ping-pong before waiting for this one's results
    (tc_batch_step_pipelined): the next ``batch_step_host(new, ...,
    reuse=True)`` only writes its actions and opens that launch's gate. Any
    other use of the batch or the library cancels the waiting launch (see
    ``pipeline_drain``); it never changes results."""
    spec, t = bs.spec, bs.spec.tables
    acts = actions if (type(actions) is np.ndarray and actions.dtype == np.int64
                       and actions.flags.c_contiguous) else \
        np.ascontiguousarray(actions, dtype=np.int64)
    if acts.shape != (bs.n,):
        raise ContractError(f"actions must have shape ({bs.n},), got {acts.shape}")
    if reuse and bs._retired:
        sb, ob = bs._retired
    else:
        sb = DeviceState.alloc(bs.n, t.n_doors, t.n_entities, bs.device)
        ob = DeviceOut.alloc(bs.n, t.obs_height, t.obs_width, bs.device,
                             debug=bs._ob.zbuf is not None)
    stg = bs._stage
    if stg is None:
        stg = bs._stage = _ActionStage(bs.n, bs.device)
    stg.h_act[:] = acts  # pinned, read by the kernel over the bus
    stg.h_flag[0] = 0
    # the call struct of a (state in, state out) pair is built once; a step
    # passes one pointer (tc_batch_step_mapped_call)
    # the successor of a reuse=True step writes this step's input state and
    # bs's output block: the pipelined call launches it ahead of its actions
    # (not for batches of many waves: a step of milliseconds gains nothing
    # from a launch made early, and its host-side copies outlast the watchdog)
    spec_next = bool(reuse and pipeline and bs.n <= PIPELINE_MAX_ENVS)
    key = (id(bs._sb), id(sb), id(ob), validate, id(bs._ob), spec_next)
    call = stg.calls.get(key)
    if call is None:
        si, so, oc, nc = bs._sb.c_struct(), sb.c_struct(), ob.c_struct(), bs._ob.c_struct()
        cs = N.TcPipeCall(N.TcMappedCall(bs._ds.handle.value, N.C.addressof(si),
                                         N.C.addressof(so), stg.h_act_ptr, N.C.addressof(oc),
                                         bs.n, 1, 1 if validate else 0, N.ptr(bs._counters),
                                         stg.h_rew_ptr, stg.h_flag_ptr, stream_ptr(bs.device)),
                          N.C.addressof(nc), stg.gate_dev.data_ptr(), 1 if spec_next else 0,
                          stg.dev_index)
        if len(stg.calls) > 8:
            stg.calls.clear()
        # keep the structs and blocks alive with the key
        stg.calls[key] = call = (N.C.addressof(cs), cs, si, so, oc, nc, bs._sb, sb, ob, bs._ob)
    if stg.fn is None:
        stg.fn = N.lib().tc_batch_step_pipelined
    rc = stg.fn(call[0])  # (the call makes the batch's device current itself)
    if rc:
        N.check(rc, "tc_batch_step_mapped")
    if stg.h_flag[0]:
        # the kernel saw an action outside the contract: the step is void
        # (bs is still valid; on this path the kernel reports bad actions
        # through the flag only, so the sticky fault counters are untouched)
        # -- raise the reference's error for the first offending action
        _check_host_actions(bs, acts)
        raise ContractError("action outside the spec's action set")
    rewards = stg.h_rew.copy()
    dones = stg.h_done.copy()
    # the successor: bs's fields with the new blocks (a __dict__ copy: this
    # call is on the host's per-step critical path)
    new = object.__new__(BatchState)
    d = new.__dict__
    d.update(bs.__dict__)
    d["_sb"], d["_ob"] = sb, ob
    d["_retired"] = (bs._sb, bs._ob) if reuse else ()
    if validate:
        new.check()
    return new, rewards, dones


def pipeline_drain() -> None:
    """End a ``batch_step_host(..., reuse=True)`` loop: cancel the step
    launched ahead of its actions (it exits without effect), so work queued
    on the stream after it runs at once instead of after the watchdog's
    timeout. Accessing a batch's frames / state does this implicitly."""
    N.pipe_cancel()


def batch_step(bs: BatchState, actions: Sequence[Action | int] | np.ndarray | torch.Tensor, *,
               validate: bool = False, reuse: bool = False, sync_checks: bool = False,
               copy_outputs: bool = True) -> tuple[BatchState, torch.Tensor, torch.Tensor]:
    """Step every env once; finished episodes auto-reset in the same launch
    (their frame shows the new episode; the terminal reward / done flag are
    still reported). Returns (next_state, rewards, dones) as device tensors.

    The step is out-of-place (the old BatchState stays valid, batch.py:31-34)
    but needs no state copy: the kernel reads the old blocks and writes the
    new ones. With ``copy_outputs=False`` rewards / dones are views of the
    successor's output block (valid until that block is recycled by a later
    ``reuse=True`` step) -- one launch per step, nothing else."""
    spec, t = bs.spec, bs.spec.tables
    acts = _coerce_actions(bs, actions)
    if reuse and bs._retired:
        sb, ob = bs._retired
    else:
        sb = DeviceState.alloc(bs.n, t.n_doors, t.n_entities, bs.device)
        ob = DeviceOut.alloc(bs.n, t.obs_height, t.obs_width, bs.device,
                             debug=bs._ob.zbuf is not None)
    launch_step_into(bs._ds, bs._sb, sb, acts, ob, bs.n, True, validate, bs._counters)
    new = BatchState(spec=spec, n=bs.n, _ds=bs._ds, _sb=sb, _ob=ob, _counters=bs._counters,
                     base=bs.base, n_total=bs.n_total,
                     _retired=(bs._sb, bs._ob) if reuse else (),
                     _stage=bs._stage, _chain=bs._chain)
    if validate or sync_checks:
        new.check()
    rewards, dones = ob.rewards, ob.dones.view(torch.bool)
    if copy_outputs:
        rewards, dones = rewards.clone(), dones.clone()
    return new, rewards, dones


_pinned_cache: dict = {}


def to_host(*tensors: torch.Tensor) -> tuple[np.ndarray, ...]:
    """Copy device tensors to host numpy arrays with async copies into pinned
    buffers and ONE stream synchronisation (instead of one sync per .cpu())."""
    outs = []
    dev = tensors[0].device
    for k, x in enumerate(tensors):
        key = (k, x.dtype, tuple(x.shape))
        buf = _pinned_cache.get(key)
        if buf is None:
            buf = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
            _pinned_cache[key] = buf
        buf.copy_(x, non_blocking=True)
        outs.append(buf)
    torch.cuda.current_stream(dev).synchronize()
    return tuple(b.numpy().copy() for b in outs)


def batch_step_inplace(bs: BatchState, actions: torch.Tensor) -> BatchState:
    """Throughput form of batch_step: mutate bs's state in place (no state
    copy), one kernel launch, no host work beyond the launch."""
    launch_batch(bs._ds, bs._sb, actions, bs._ob, bs.n, L.MODE_STEP, True, False,
                 bs._counters)
    return bs


def policy_actions(spec: EnvSpec, n: int, steps: int, seed: int = 0) -> np.ndarray:
    """The (steps, n) uniform-random action table of a seeded rollout
    (batch.py:141-153), computed on the host like the reference."""
    tags = np.array([int(a) for a in spec.action_set], dtype=np.int64)
    counters = np.arange(steps * n, dtype=np.uint64).reshape(steps, n)
    return tags[rng.policy_uniform(rng.policy_key(seed), counters, tags.shape[0])]


def policy_actions_device(spec: EnvSpec, step: int, n: int, seed: int, *, base: int = 0,
                          n_total: int | None = None, out: torch.Tensor | None = None,
                          device=None) -> torch.Tensor:
    """Row ``step`` of policy_actions(spec, n_total, ..., seed) for envs
    [base, base+n), drawn on the device."""
    dev = resolve_device(device if out is None else out.device)
    if out is None:
        out = torch.empty(n, dtype=torch.int64, device=dev)
    tags = np.array([int(a) for a in spec.action_set], dtype=np.int64)
    with torch.cuda.device(dev):
        N.check(N.lib().tc_policy_actions(
            rng.policy_key(seed), step, n_total if n_total is not None else base + n, base, n,
            tags.ctypes.data, tags.shape[0], N.ptr(out), stream_ptr(dev)), "tc_policy_actions")
    return out


def rollout(bs: BatchState, k_steps: int, seed: int, *, step0: int = 0,
            frames: torch.Tensor | None = None, record: bool = False) -> dict:
    """K fused steps in ONE launch with the seeded uniform policy drawn on the
    device (== batch_step with policy_actions(spec, n_total, ..., seed)
    rows step0..step0+K-1). ``frames`` is a [R, N, H, W, 3] ring (R >= 1;
    default: the batch's own frame block, R = 1); with ``record`` the
    per-step rewards/dones/truncs/events come back as [K, N] tensors."""
    t = bs.spec.tables
    dev = bs.device
    ring = bs._ob.frames.unsqueeze(0) if frames is None else frames
    if ring.dim() != 5 or tuple(ring.shape[1:]) != (bs.n, t.obs_height, t.obs_width, 3):
        raise ContractError("frames must be [R, N, H, W, 3] uint8")
    res = {}
    if record:
        res = dict(
            rewards=torch.zeros((k_steps, bs.n), dtype=torch.float64, device=dev),
            dones=torch.zeros((k_steps, bs.n), dtype=torch.uint8, device=dev),
            truncs=torch.zeros((k_steps, bs.n), dtype=torch.uint8, device=dev),
            events=torch.zeros((k_steps, bs.n), dtype=torch.int32, device=dev))
    o = N.TcOut()
    o.frames = N.ptr(ring)
    o.statuses = N.ptr(bs._ob.statuses)
    for k, v in res.items():
        setattr(o, k, N.ptr(v))
    with torch.cuda.device(dev):
        N.check(N.lib().tc_rollout(
            bs._ds.handle, N.C.byref(bs._sb.c_struct()), N.C.byref(o), bs.n, bs.base,
            bs.n_total, rng.policy_key(seed), step0, k_steps, ring.shape[0],
            N.ptr(bs._counters), stream_ptr(dev)), "tc_rollout")
    res["frames"] = ring
    return res


def throughput_probe(spec: EnvSpec, n: int, steps: int, seed: int = 0, *,
                     device=None) -> float:
    """Aggregate env-steps/s under the seeded uniform policy, wall-clock,
    through batch_step with host actions (batch.py:156-179 semantics)."""
    if n < 1 or steps < 1:
        raise ContractError("n and steps must both be >= 1")
    bs = batch_reset(spec, n, seed, device=device)
    all_actions = policy_actions(spec, n, steps, seed)
    for s in range(min(3, steps)):
        bs, _, _ = batch_step(bs, all_actions[s], reuse=True)
    torch.cuda.synchronize(bs.device)
    start = time.perf_counter()
    for s in range(steps):
        bs, _, _ = batch_step(bs, all_actions[s], reuse=True)
    torch.cuda.synchronize(bs.device)
    elapsed = time.perf_counter() - start
    bs.check()
    return (n * steps) / elapsed
