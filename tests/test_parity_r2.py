"""Round-2 parity cases: the configurations and callers round 1 left unpinned.

All through the product's C ABI; the checkers are the reference's own
digests (tests/golden/digests_r2.json, made by make_golden_r2.py from the
reference's compiled backend) and the oracle port. Mirrors the reference's
cross-backend tests (pkg/tests/test_backends.py:40-120, test_batch.py:26-120),
its acceptance digest (test_acceptance.py:243-277) and its binding
equivalence tests (pkg/bindings/tests/test_equivalence.py:26-89).
"""

from __future__ import annotations

import ctypes as C
import hashlib
import json
import random

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from _digest import Digest

import paper_2605_19926_b200 as tc
from paper_2605_19926_b200 import _native as N
from paper_2605_19926_b200 import layout as L
from paper_2605_19926_b200.engine import DeviceOut, launch_batch
from paper_2605_19926_b200.synthetic import large_tilemap
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

DEV = "cuda:0"
GOLD = json.loads((GOLDEN / "digests_r2.json").read_text())

# must match tests/golden/make_golden_r2.py LARGE_MAPS
LARGE_MAPS = {
    "large-64x64": (64, 64, 2, 6, 8, 11, False),
    "large-96x80": (96, 80, 6, 12, 8, 12, True),
    "large-160x128": (160, 128, 4, 16, 16, 13, True),
    "doors32-20x20": (20, 20, 32, 6, 8, 21, True),
    "doors32-90x72": (90, 72, 32, 10, 8, 22, True),
}


def large_spec(name, max_steps=40, **kw):
    w, h, nd, ne, ns, seed, das = LARGE_MAPS[name]
    m = large_tilemap(random.Random(seed), w, h, n_doors=nd, n_entities=ne, n_spawns=ns,
                      doors_at_spawns=das)
    return tc.EnvSpec(id=name, map=m, action_set=tc.suite.STRAFE_ACTIONS,
                      goal_mode=tc.GoalMode.RANDOM_PER_EPISODE, max_steps=max_steps,
                      living_reward=0.01, health_decay=0.5, health_restore=10.0, **kw)


def run_digest(spec, n, steps, seed):
    acts = tc.policy_actions(spec, n, steps, seed)
    bs = tc.batch_reset(spec, n, seed, device=DEV)
    d = Digest()
    d.frames(bs.frames.cpu().numpy())
    for s in range(steps):
        bs, rew, done = tc.batch_step(bs, acts[s], reuse=True)
        d.step(bs.host_state(), rew.cpu().numpy(), done.cpu().numpy(),
               bs._ob.truncs.cpu().numpy(), bs.last_events, bs.frames.cpu().numpy())
    bs.check()
    return d, bs


def assert_digest(d, case):
    assert d.hexdigest() == case["digest"], case
    assert d.reward_sum == case["reward_sum"] and d.dones == case["dones"], case
    assert d.events_or == case["events_or"], case


def compare_with_oracle(spec, n, steps, seed, check_steps, debug=True):
    acts = tc.policy_actions(spec, n, steps, seed)
    bs = tc.batch_reset(spec, n, seed, device=DEV, debug=debug)
    r = orc.Rollout(spec, n, seed, debug=debug)
    assert np.array_equal(bs.frames.cpu().numpy(), r.out["frames"]), "reset frames"
    for s in range(steps):
        bs, rew, done = tc.batch_step(bs, acts[s], reuse=True)
        r.step(acts[s])
        if s in check_steps:
            assert np.array_equal(rew.cpu().numpy(), r.out["rewards"]), s
            assert np.array_equal(done.cpu().numpy(), r.out["dones"] != 0), s
            assert np.array_equal(bs.last_events, r.out["events"]), s
            assert np.array_equal(bs.frames.cpu().numpy(), r.out["frames"]), s
            host = bs.host_state()
            for k, v in r.state.items():
                assert np.array_equal(host[k], v), (s, k)
            if debug:
                assert np.array_equal(bs._ob.zbuf.cpu().numpy(), r.out["zbuf"]), s
                assert np.array_equal(bs._ob.rayinfo.cpu().numpy(), r.out["rayinfo"]), s
                assert np.array_equal(bs._ob.spritevis.cpu().numpy().view(np.uint64),
                                      r.out["spritevis"]), s
    bs.check()
    return bs, r


# ---------------------------------------------------------------- C1
def test_c1_one_env_1000_steps_reference_digest():
    """BASELINE configs[0]: my-way-home, 1 env, 1000 steps; digest and final
    state equal the reference's."""
    case = GOLD["c1"]
    d, bs = run_digest(tc.make_env("my-way-home"), 1, case["steps"], case["seed"])
    assert_digest(d, case)
    host = bs.host_state()
    fin = case["final"]
    for k in ("px", "py", "dx", "dy", "health"):
        assert [float.hex(float(v)) for v in host[k]] == fin[k], k
    for k in ("inv", "t", "rkey", "rctr", "done", "agoal"):
        assert [int(v) for v in host[k]] == fin[k], k
    assert hashlib.sha256(bs.frames.cpu().numpy().tobytes()).hexdigest() == fin["frame_sha"]


# ---------------------------------------------------- large maps / doors
@pytest.mark.parametrize("name", sorted(LARGE_MAPS))
def test_large_and_32_door_maps_reference_digest(name):
    """Maps beyond 4096 cells (SURVEY §8(d) large-map variant) and 32-door
    maps (the reference's limit): digests equal the reference's."""
    case = GOLD[name]
    d, _ = run_digest(large_spec(name), case["n"], case["steps"], case["seed"])
    assert_digest(d, case)


def test_large_map_wide_obs_reference_digest():
    case = GOLD["large-96x80-128x96"]
    spec = large_spec("large-96x80", obs_width=128, obs_height=96)
    d, _ = run_digest(spec, case["n"], case["steps"], case["seed"])
    assert_digest(d, case)


@pytest.mark.parametrize("name", ["large-160x128", "doors32-90x72", "doors32-20x20"])
def test_large_maps_debug_taps_vs_oracle(name):
    """Per-ray hit cell / side / steps, z-buffer and sprite visibility,
    bit-exact against the oracle on the large and 32-door maps."""
    compare_with_oracle(large_spec(name, max_steps=30), 64, 40, 5, check_steps={0, 7, 19, 39})


# ----------------------------------------------------------------- C5
def test_c5_bench_map_reference_digest():
    import bench
    case = GOLD["c5-map"]
    d, _ = run_digest(bench.synthetic_spec(), case["n"], case["steps"], case["seed"])
    assert_digest(d, case)


def test_c5_bench_map_131072_envs_vs_oracle():
    """The C5 bench map (random.Random(20260518)) at the bench's 131072 envs
    per GPU (multi-wave, dynamic env tickets): every 10th step bit-exact."""
    import bench
    spec = bench.synthetic_spec()
    compare_with_oracle(spec, 131072, 20, 0, check_steps={0, 9, 19}, debug=False)


# ------------------------------------------------- callers
def _indices_for(spec, tags):
    lut = {int(a): i for i, a in enumerate(spec.action_set)}
    return np.vectorize(lut.__getitem__)(tags)


def test_gym_vecenv_1000_steps_reference_digest():
    """test_equivalence.py:26-43: VecEnv key-door 8 envs x 1000 steps, seed
    42, action indices from policy_actions -- digest equals the reference
    core rollout's."""
    from paper_2605_19926_b200 import gym
    case = GOLD["vec-key-door"]
    spec = tc.make_env("key-door")
    n, steps, seed = case["n"], case["steps"], case["seed"]
    idx = _indices_for(spec, tc.policy_actions(spec, n, steps, seed))
    v = gym.make_vec("key-door", n, seed=seed)
    d = Digest()
    d.frames(v.observations.cpu().numpy())
    for s in range(steps):
        obs, r, dn, info = v.step(idx[s])
        d.step(v._bs.host_state(), r.cpu().numpy(), dn.cpu().numpy(),
               info["truncated"].cpu().numpy(), v._bs.last_events, obs.cpu().numpy())
    v.check()
    assert_digest(d, case)


def test_gym_scalar_env_1000_steps_reference_digest():
    """test_equivalence.py:46-70: the scalar Env (simple, seed 7), reset with
    seed + s whenever the episode is done -- digest of (obs, reward,
    terminated, truncated) equals the reference scalar core's."""
    from paper_2605_19926_b200 import gym
    case = GOLD["scalar-simple"]
    spec = tc.make_env("simple")
    steps, seed = case["steps"], case["seed"]
    idx = _indices_for(spec, tc.policy_actions(spec, 1, steps, seed)[:, 0])
    env = gym.make("simple")
    obs, _ = env.reset(seed=seed)
    h = hashlib.blake2b(digest_size=16)
    h.update(obs.tobytes())
    done, rsum, resets = False, 0.0, 0
    for s in range(steps):
        if done:
            obs, _ = env.reset(seed=seed + s)
            h.update(obs.tobytes())
            resets += 1
        o, r, term, trunc, _ = env.step(int(idx[s]))
        done = term or trunc
        h.update(np.float64(r).tobytes())
        h.update(bytes([term, trunc]))
        h.update(o.tobytes())
        rsum += r
    assert (h.hexdigest(), rsum, resets) == (case["digest"], case["reward_sum"], case["resets"])


def test_scalar_api_matches_oracle():
    """tc.reset / tc.step (dynamics.py, one env, no auto-reset) against the
    oracle's batch kernel on one env with auto_reset off (the reference's
    scalar step is exactly that, dynamics.py:140)."""
    spec = tc.make_env("key-door", max_steps=60)
    t = spec.tables
    rnd = random.Random(b"scalar-vs-oracle")
    for seed in range(4):
        state, obs = tc.reset(spec, tc.split(tc.from_seed(seed), 0))
        st = orc.alloc_state(1, t.n_doors, t.n_entities)
        out = orc.alloc_out(1, t.obs_height, t.obs_width)
        orc.seed_streams(seed, 0, 1, st)
        orc.batch_kernel(t, st, None, out, 0, n_threads=1)
        assert np.array_equal(obs, out["frames"][0])
        while not state.done:
            a = int(rnd.choice(spec.action_set))
            res = tc.step(spec, state, a)
            orc.batch_kernel(t, st, np.array([a]), out, 1, auto_reset=False, n_threads=1)
            assert res.reward == out["rewards"][0] and res.done == bool(out["dones"][0])
            assert res.info["truncated"] == bool(out["truncs"][0])
            assert np.array_equal(res.observation, out["frames"][0])
            state = res.state
            assert state.pose.position.x == st["px"][0] and state.t == st["t"][0]
            assert state.health == st["health"][0]


def test_cli_bench_reward_sum_reference():
    """test_equivalence.py:73-89: the CLI bench report's reward_sum."""
    from paper_2605_19926_b200 import cli
    case = GOLD["cli-key-door"]
    rep = cli.bench(case["env"], case["n"], case["steps"], case["seed"], 64, 64)
    assert rep["results"]["reward_sum"] == case["reward_sum"]


# ------------------------------------------------------------ C ABI
def test_host_batch_kernel_abi_vs_oracle():
    """tc_host_batch_kernel (host blocks in/out, the reference's batch_kernel
    signature over the C ABI): reset + 25 steps with validation, every
    output and state array equal to the oracle's."""
    spec = tc.make_env("key-door", max_steps=9)
    t = spec.tables
    n = 50
    ours = orc.alloc_state(n, t.n_doors, t.n_entities)
    ref = orc.alloc_state(n, t.n_doors, t.n_entities)
    oo = orc.alloc_out(n, t.obs_height, t.obs_width, debug=True)
    ro = orc.alloc_out(n, t.obs_height, t.obs_width, debug=True)
    for st in (ours, ref):
        orc.seed_streams(11, 0, n, st)
    viol = C.c_int64(-1)
    lib = N.lib()
    N.check(lib.tc_host_batch_kernel(C.byref(t.c_struct()), C.byref(N.state_struct(ours)),
                                     None, C.byref(N.out_struct(oo)), n, 0, 0, 0,
                                     C.byref(viol)), "tc_host_batch_kernel")
    orc.batch_kernel(t, ref, None, ro, 0, n_threads=1)
    assert np.array_equal(oo["frames"], ro["frames"])
    acts = tc.policy_actions(spec, n, 25, 11)
    for s in range(25):
        N.check(lib.tc_host_batch_kernel(C.byref(t.c_struct()), C.byref(N.state_struct(ours)),
                                         acts[s].ctypes.data, C.byref(N.out_struct(oo)), n, 1,
                                         1, 1, C.byref(viol)), "tc_host_batch_kernel")
        rv = orc.batch_kernel(t, ref, acts[s], ro, 1, auto_reset=True, validate=True,
                              n_threads=1)
        assert viol.value == rv == 0
        for k in ("frames", "rewards", "dones", "truncs", "events", "statuses", "zbuf",
                  "rayinfo", "spritevis"):
            assert np.array_equal(oo[k], ro[k]), (s, k)
        for k in ref:
            assert np.array_equal(ours[k], ref[k]), (s, k)


def test_batch_step_host_abi_vs_oracle():
    """tc_batch_step_host (copy-engine H2D actions, D2H rewards / dones, one
    stream sync) against the oracle, device state carried between calls."""
    spec = tc.make_env("dmlab-random-goal-01", max_steps=15)
    n, steps, seed = 700, 30, 6
    bs = tc.batch_reset(spec, n, seed, device=DEV)
    t = spec.tables
    from paper_2605_19926_b200.engine import DeviceState
    other = DeviceState.alloc(n, t.n_doors, t.n_entities, bs.device)
    out = DeviceOut.alloc(n, t.obs_height, t.obs_width, bs.device)
    acts_dev = torch.empty(n, dtype=torch.int64, device=DEV)
    rew = np.zeros(n)
    done = np.zeros(n, np.uint8)
    r = orc.Rollout(spec, n, seed)
    acts = tc.policy_actions(spec, n, steps, seed)
    cur, nxt = bs._sb, other
    for s in range(steps):
        a = np.ascontiguousarray(acts[s])
        N.check(N.lib().tc_batch_step_host(
            bs._ds.handle, C.byref(cur.c_struct()), C.byref(nxt.c_struct()), a.ctypes.data,
            N.ptr(acts_dev), C.byref(out.c_struct()), n, 1, 0, N.ptr(bs._counters),
            rew.ctypes.data, done.ctypes.data, torch.cuda.current_stream().cuda_stream),
            "tc_batch_step_host")
        r.step(acts[s])
        assert np.array_equal(rew, r.out["rewards"]) and np.array_equal(done, r.out["dones"]), s
        cur, nxt = nxt, cur
    assert np.array_equal(out.frames.cpu().numpy(), r.out["frames"])
    host = cur.to_host()
    for k, v in r.state.items():
        assert np.array_equal(host[k], v), k


# ------------------------------------------- round-1 advisor findings
def test_device_policy_feeds_step_back_to_back():
    """A policy kernel writes the actions and the step kernel that reads them
    follows immediately on the stream (programmatic dependent launch on the
    step): the step must see the policy kernel's writes. One action buffer
    rewritten every step, no host sync in between; compared with the oracle
    at the end."""
    spec = tc.make_env("my-way-home", max_steps=17)
    n, k, seed = 4096, 30, 12
    bs = tc.batch_reset(spec, n, seed, device=DEV)
    acts_dev = torch.empty(n, dtype=torch.int64, device=DEV)
    rews = []
    for s in range(k):
        tc.policy_actions_device(spec, s, n, seed, out=acts_dev)
        bs, rew, done = tc.batch_step(bs, acts_dev, reuse=True, copy_outputs=False)
        rews.append(rew.clone())
    torch.cuda.synchronize()
    r = orc.Rollout(spec, n, seed)
    acts = tc.policy_actions(spec, n, k, seed)
    for s in range(k):
        r.step(acts[s])
        assert np.array_equal(rews[s].cpu().numpy(), r.out["rewards"]), s
    assert np.array_equal(bs.frames.cpu().numpy(), r.out["frames"])
    host = bs.host_state()
    for key, v in r.state.items():
        assert np.array_equal(host[key], v), key
    bs.check()


def test_multi_wave_without_counters():
    """tc_batch_kernel with counters = NULL on a batch larger than one wave:
    the static interleaved schedule steps every env exactly once."""
    spec = tc.make_env("my-way-home", max_steps=11)
    n, steps, seed = 20000, 6, 3
    bs = tc.batch_reset(spec, n, seed, device=DEV)
    out = DeviceOut.alloc(n, 64, 64, bs.device)
    r = orc.Rollout(spec, n, seed)
    acts = tc.policy_actions(spec, n, steps, seed)
    for s in range(steps):
        a = torch.from_numpy(acts[s]).to(DEV)
        launch_batch(bs._ds, bs._sb, a, out, n, L.MODE_STEP, True, False, None)
        r.step(acts[s])
    assert np.array_equal(out.rewards.cpu().numpy(), r.out["rewards"])
    assert np.array_equal(out.frames.cpu().numpy(), r.out["frames"])
    host = bs.host_state()
    for key, v in r.state.items():
        assert np.array_equal(host[key], v), key


def test_zero_direction_reports_step_budget():
    """A zero view direction (restored state / render_into) makes every ray
    (0, 0): the reference's cast_ray runs out its step budget
    (_pycore.py:60-90) and so must the kernel -- no spin."""
    spec = tc.make_env("simple")
    t = spec.tables
    frame = np.zeros((t.obs_height, t.obs_width, 3), np.uint8)
    zbuf = np.zeros(t.obs_width)
    st = C.c_int32(-1)
    N.check(N.lib().tc_host_render_into(C.byref(t.c_struct()), 1.5, 1.5, 0.0, 0.0, None, None,
                                        -1, frame.ctypes.data, zbuf.ctypes.data,
                                        C.byref(st)), "tc_host_render_into")
    ost, *_ = orc.render_into(t, 1.5, 1.5, 0.0, 0.0, np.zeros(0, np.uint8),
                              np.zeros(0, np.uint8), -1)
    assert st.value == ost == L.ST_STEP_BUDGET


# ------------------------------------------------ chained multi-step launches
@pytest.mark.parametrize("env,n,k,ring,taps", [
    ("my-way-home", 4096, 30, 3, False), ("key-door", 600, 25, 2, False),
    ("health-gathering", 1000, 20, 4, False), ("my-way-home", 20000, 6, 2, False),
    ("key-door", 16384, 12, 2, False), ("key-door", 9000, 10, 1, False),
    ("dmlab-static-03@128", 8192, 6, 2, False), ("my-way-home", 4096, 6, 2, True),
    # far fewer CTAs than slots: many launches resident at once, finishing
    # out of order (the per-slot done rows)
    ("health-gathering", 256, 40, 3, False), ("key-door", 128, 40, 2, False)])
def test_batch_steps_chained_equal_oracle(env, n, k, ring, taps):
    """tc.batch_steps: K step launches chained per env / CTA (no grid-wide
    wait between them) == K reference steps: the final state, the last
    `ring` steps' frames / rewards / dones from the output ring, bit-exact.
    One-wave batches chain per CTA; multi-wave ones (20000, 16384, 9000 envs
    at 64x64, 8192 at 128x128) per env with per-launch ticket counters, ring
    1 included (every step rewrites the same block); a ring with a debug-tap
    block runs K ordinary launches (the tapped kernel does not chain)."""
    from paper_2605_19926_b200.engine import DeviceOut
    env, _, obs = env.partition("@")
    size = {"obs_width": int(obs), "obs_height": int(obs)} if obs else {}
    spec = tc.make_env(env, max_steps=13, **size)
    seed = 21
    bs = tc.batch_reset(spec, n, seed, device=DEV)
    acts = tc.policy_actions(spec, n, 2 * k, seed)
    oh, ow = spec.tables.obs_height, spec.tables.obs_width
    outs = [DeviceOut.alloc(n, oh, ow, bs.device, debug=taps and r == 0) for r in range(ring)]
    r = orc.Rollout(spec, n, seed)
    # two calls back to back: epochs continue, the second call's first
    # launch waits for the first call's last one
    for part in range(2):
        rows = torch.from_numpy(acts[part * k:(part + 1) * k]).to(DEV)
        bs = tc.batch_steps(bs, rows, outs=outs)
        snaps = {}
        for s in range(k):
            r.step(acts[part * k + s])
            if s >= k - ring:
                snaps[s] = (r.out["frames"].copy(), r.out["rewards"].copy(),
                            r.out["dones"].copy())
        torch.cuda.synchronize()
        for s, (fr, rw, dn) in snaps.items():
            o = outs[s % ring]
            assert np.array_equal(o.frames.cpu().numpy(), fr), (part, s)
            assert np.array_equal(o.rewards.cpu().numpy(), rw), (part, s)
            assert np.array_equal(o.dones.cpu().numpy(), dn), (part, s)
        host = bs.host_state()
        for key, v in r.state.items():
            assert np.array_equal(host[key], v), (part, key)
        assert torch.equal(bs.frames, outs[(k - 1) % ring].frames)
    bs.check()
    # an ordinary step after a chain continues from the chained state
    bs, rew, done = tc.batch_step(bs, acts[0], reuse=True)
    r.step(acts[0])
    assert np.array_equal(bs.frames.cpu().numpy(), r.out["frames"])
