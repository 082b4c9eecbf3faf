"""The pipelined host step (tc_batch_step_pipelined via batch_step_host with
reuse=True): each call launches the next step ahead of its actions behind a
gate; the next call only writes its actions and opens the gate. Results
must be those of the ordinary step sequence -- checked against the oracle
(the reference's batch_step semantics, batch.py:109-138) -- whether the
waiting launch is released, cancelled by another call or access, or timed
out by the watchdog."""

from __future__ import annotations

import time

import numpy as np
import pytest
import torch

import paper_2605_19926_b200 as tc
from paper_2605_19926_b200 import _native as N
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _check_final(bs, r):
    tc.pipeline_drain()
    assert np.array_equal(bs.frames.cpu().numpy(), r.out["frames"])
    host = bs.host_state()
    for k, v in r.state.items():
        assert np.array_equal(host[k], v), k
    bs.check()


@pytest.mark.parametrize("env,n,steps", [
    ("my-way-home", 4096, 40),      # one wave (lean_kernel one env per warp), the e2e config
    ("key-door", 16384, 12),        # multi-wave (env tickets, next action prefetched)
    ("dmlab-random-goal-01", 37, 60),  # fewer envs than CTAs, frequent resets
    ("my-way-home-short", 1024, 240),  # a long resident loop through many auto-resets
])
def test_pipelined_host_loop_vs_oracle(env, n, steps):
    if env == "my-way-home-short":
        spec = tc.make_env("my-way-home", max_steps=30)
    else:
        spec = tc.make_env(env, max_steps=25) if n < 100 else tc.make_env(env)
    seed = 11
    acts = tc.policy_actions(spec, n, steps, seed)
    bs = tc.batch_reset(spec, n, seed, device=DEV)
    N.pipe_reset()
    s0 = N.pipe_stats()
    got = []
    # the GPU loop first (the oracle between calls would outlast the
    # watchdog's timeout), then the oracle over the same actions
    for s in range(steps):
        bs, rew, done = tc.batch_step_host(bs, acts[s], reuse=True)
        got.append((rew, done))
    s1 = N.pipe_stats()
    # every step after the first ran as a released pipelined launch (one
    # watchdog timeout tolerated: a host hiccup > 1 ms, then 8 steps of back-off)
    assert s1["released"] - s0["released"] >= steps - 1 - 9 * (s1["timeouts"] - s0["timeouts"])
    assert s1["timeouts"] - s0["timeouts"] <= 1, (s0, s1)
    assert s1["pending"] == 1 or s1["timeouts"] > s0["timeouts"]
    r = orc.Rollout(spec, n, seed)
    for s in range(steps):
        r.step(acts[s])
        assert np.array_equal(got[s][0], r.out["rewards"]), s
        assert np.array_equal(got[s][1], r.out["dones"] != 0), s
    _check_final(bs, r)
    assert N.pipe_stats()["pending"] == 0


def test_pipeline_cancel_paths_vs_oracle():
    """Every way a waiting launch is dropped: frames access, another batch's
    step, a device-path step, a rejected action, a non-reuse call -- the
    trajectory stays the oracle's."""
    spec = tc.make_env("key-door", max_steps=30)
    n, steps, seed = 2048, 48, 5
    acts = tc.policy_actions(spec, n, steps, seed)
    bs = tc.batch_reset(spec, n, seed, device=DEV)
    other_spec = tc.make_env("my-way-home")
    ob = tc.batch_reset(other_spec, 512, 3, device=DEV)
    oacts = tc.policy_actions(other_spec, 512, steps, 3)
    N.pipe_reset()
    t0 = N.pipe_stats()
    log = []  # (step, rewards, dones or None, other batch's rewards or None)
    for s in range(steps):
        k = s % 8
        orw = None
        if k == 1:
            _ = bs.frames  # access cancels the waiting launch
        elif k == 2:
            # another batch steps on the same stream: mismatch -> cancel
            ob, orw, _ = tc.batch_step_host(ob, oacts[s], reuse=True)
        elif k == 4:
            bad = acts[s].copy()
            bad[n // 3] = 99
            with pytest.raises(tc.ContractError):
                tc.batch_step_host(bs, bad, reuse=True)
        if k == 5:
            # an ordinary device-path step of the same batch
            bs, rd, dd = tc.batch_step(bs, acts[s], reuse=True)
            rew, done = rd.cpu().numpy(), dd.cpu().numpy()
        elif k == 6:
            bs, rew, done = tc.batch_step_host(bs, acts[s], reuse=False)
        else:
            bs, rew, done = tc.batch_step_host(bs, acts[s], reuse=True)
        log.append((s, rew, done, orw))
    t1 = N.pipe_stats()
    assert t1["released"] - t0["released"] >= steps // 8 * 2
    assert t1["cancelled"] - t0["cancelled"] >= steps // 8 * 4
    assert t1["timeouts"] == t0["timeouts"]
    r = orc.Rollout(spec, n, seed)
    orr = orc.Rollout(other_spec, 512, 3)
    for s, rew, done, orw in log:
        r.step(acts[s])
        assert np.array_equal(rew, r.out["rewards"]), s
        assert np.array_equal(done, r.out["dones"] != 0), s
        if orw is not None:
            orr.step(oacts[s])
            assert np.array_equal(orw, orr.out["rewards"]), s
    _check_final(bs, r)
    tc.pipeline_drain()
    assert np.array_equal(ob.frames.cpu().numpy(), orr.out["frames"])


def test_pipeline_off_and_sync_without_drain():
    spec = tc.make_env("my-way-home")
    n, seed = 1024, 2
    acts = tc.policy_actions(spec, n, 10, seed)
    bs = tc.batch_reset(spec, n, seed, device=DEV)
    N.pipe_reset()
    to0 = N.pipe_stats()["timeouts"]
    got = []
    for s in range(4):
        bs, rew, _ = tc.batch_step_host(bs, acts[s], reuse=True, pipeline=False)
        got.append(rew)
        assert N.pipe_stats()["pending"] == 0
    for s in range(4, 8):
        if s == 6:
            time.sleep(0.02)  # the watchdog cancels the waiting launch
        bs, rew, _ = tc.batch_step_host(bs, acts[s], reuse=True)
        got.append(rew)
    assert N.pipe_stats()["timeouts"] == to0 + 1
    bs, rew, _ = tc.batch_step_host(bs, acts[8], reuse=True)  # backing off: no launch ahead
    got.append(rew)
    assert N.pipe_stats()["pending"] == 0
    N.pipe_reset()
    bs, rew, _ = tc.batch_step_host(bs, acts[9], reuse=True)
    got.append(rew)
    # a plain device synchronize with a launch still waiting: the watchdog
    # cancels it within its timeout (no hang)
    assert N.pipe_stats()["pending"] == 1
    t = time.perf_counter()
    torch.cuda.synchronize()
    assert time.perf_counter() - t < 1.0
    assert N.pipe_stats()["pending"] == 0 and N.pipe_stats()["timeouts"] == to0 + 2
    r = orc.Rollout(spec, n, seed)
    for s in range(10):
        r.step(acts[s])
        assert np.array_equal(got[s], r.out["rewards"]), s
    _check_final(bs, r)
    N.pipe_reset()
