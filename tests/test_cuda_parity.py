"""CUDA path vs the oracle (and the reference's golden fixtures), bit-exact.

Every test calls the product through its C ABI (via the host layer); the
oracle port is only the checker. Mirrors the reference's cross-backend
parity suite (pkg/tests/test_backends.py:40-120, test_batch.py:26-120).
"""

from __future__ import annotations

import math
import random

import numpy as np
import pytest
import torch

from conftest import GOLDEN, unpack_map
from _digest import Digest

import paper_2605_19926_b200 as tc
from paper_2605_19926_b200 import layout as L
from paper_2605_19926_b200.tables import build_tables
from paper_2605_19926_b200.synthetic import random_tilemap
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _assert_state(bs, ref_state, where=""):
    host = bs.host_state()
    for k, v in ref_state.items():
        assert np.array_equal(host[k], v), f"{where}: state {k} differs"


def _compare_rollout(spec, n, steps, seed, check_every=1, debug=False):
    acts = tc.policy_actions(spec, n, steps, seed)
    bs = tc.batch_reset(spec, n, seed, device=DEV, debug=debug)
    r = orc.Rollout(spec, n, seed, debug=debug)
    assert np.array_equal(bs.frames.cpu().numpy(), r.out["frames"]), "reset frames"
    _assert_state(bs, r.state, "reset")
    for s in range(steps):
        bs, rew, done = tc.batch_step(bs, acts[s], reuse=True)
        r.step(acts[s])
        if s % check_every == 0 or s == steps - 1:
            assert np.array_equal(rew.cpu().numpy(), r.out["rewards"]), s
            assert np.array_equal(done.cpu().numpy(), r.out["dones"] != 0), s
            assert np.array_equal(bs._ob.truncs.cpu().numpy(), r.out["truncs"]), s
            assert np.array_equal(bs.last_events, r.out["events"]), s
            fr = bs.frames.cpu().numpy()
            if not np.array_equal(fr, r.out["frames"]):
                bad = np.argwhere((fr != r.out["frames"]).any(axis=-1))
                raise AssertionError(f"step {s}: {len(bad)} pixels differ, first {bad[:5]}")
            _assert_state(bs, r.state, f"step {s}")
            if debug:
                assert np.array_equal(bs._ob.zbuf.cpu().numpy(), r.out["zbuf"]), s
                assert np.array_equal(bs._ob.rayinfo.cpu().numpy(), r.out["rayinfo"]), s
                assert np.array_equal(bs._ob.spritevis.cpu().numpy().view(np.uint64),
                                      r.out["spritevis"]), s
    bs.check()
    return bs


@pytest.mark.parametrize("env", ["simple", "key-door", "key-corridor", "health-gathering",
                                 "my-way-home", "dmlab-static-01", "dmlab-random-goal-02",
                                 "dmlab-static-03"])
def test_shipped_env_rollouts_bitexact(env):
    spec = tc.make_env(env, max_steps=45)
    _compare_rollout(spec, 96, 120, seed=1, debug=True)


@pytest.mark.parametrize("wh", [(64, 64), (128, 128), (8, 8), (40, 24), (37, 29), (96, 33),
                                (256, 160)])
def test_observation_sizes_bitexact(wh):
    w, h = wh
    spec = tc.make_env("health-gathering", obs_width=w, obs_height=h, max_steps=30)
    _compare_rollout(spec, 40, 50, seed=4, debug=True)


def test_synthetic_maps_bitexact():
    for s in range(12):
        tmap = random_tilemap(random.Random(1000 + s))
        spec = tc.EnvSpec(id=f"syn{s}", map=tmap, action_set=tc.suite.STRAFE_ACTIONS,
                          goal_mode=tc.GoalMode.RANDOM_PER_EPISODE, max_steps=25,
                          living_reward=0.01, health_decay=1.0, health_restore=10.0)
        _compare_rollout(spec, 64, 60, seed=s, debug=True)


def test_golden_digests(golden_digests):
    for case in golden_digests:
        spec = tc.make_env(case["env"], **case["overrides"])
        n, steps, seed = case["n"], case["steps"], case["seed"]
        acts = tc.policy_actions(spec, n, steps, seed)
        bs = tc.batch_reset(spec, n, seed, device=DEV)
        d = Digest()
        d.frames(bs.frames.cpu().numpy())
        for s in range(steps):
            bs, rew, done = tc.batch_step(bs, acts[s], reuse=True)
            d.step(bs.host_state(), rew.cpu().numpy(), done.cpu().numpy(),
                   bs._ob.truncs.cpu().numpy(), bs.last_events, bs.frames.cpu().numpy())
        assert d.hexdigest() == case["digest"], case
        assert d.reward_sum == case["reward_sum"] and d.dones == case["dones"]


def test_golden_frames_render_frame():
    g = np.load(GOLDEN / "golden_frames.npz")
    from paper_2605_19926_b200.maps import SHIPPED_MAPS
    for key in g.files:
        env, sx, sy, dx, dy = key.split("|")
        tmap = tc.parse_map(SHIPPED_MAPS[env])
        pose = tc.Pose.looking(tc.Vec2(float(sx), float(sy)), tc.Vec2(float(dx), float(dy)))
        assert np.array_equal(tc.render_frame(tmap, pose), g[key]), key


def test_random_frames_render_frame():
    g = np.load(GOLDEN / "frames_random.npz")
    m = 0
    while f"f{m}_frame" in g.files:
        tmap = unpack_map(g[f"f{m}_map"])
        exp = g[f"f{m}_frame"]
        px, py, dx, dy = g[f"f{m}_pose"]
        pose = tc.Pose.looking(tc.Vec2(px, py), tc.Vec2(dx, dy))
        got = tc.render_frame(tmap, pose, exp.shape[1], exp.shape[0],
                              door_open=[bool(v) for v in g[f"f{m}_dopen"]])
        assert np.array_equal(got, exp), m
        m += 1


def test_cast_ray_dda_matches_reference_rays():
    g = np.load(GOLDEN / "rays.npz")
    m = 0
    while f"m{m}_kind" in g.files:
        kind, didx, dopen = g[f"m{m}_kind"], g[f"m{m}_didx"], g[f"m{m}_dopen"]
        ndoor = int(didx.max()) + 1 if didx.max() >= 0 else 0
        tmap = _map_from_arrays(kind, didx, ndoor)
        for q, iexp, fexp in zip(g[f"m{m}_q"], g[f"m{m}_i"], g[f"m{m}_f"]):
            hit = tc.cast_ray_dda(tmap, tc.Vec2(q[0], q[1]), tc.Vec2(q[2], q[3]),
                                  door_open=[bool(v) for v in dopen])
            assert (hit.cell[0], hit.cell[1], int(hit.side), hit.steps) == \
                (int(iexp[1]), int(iexp[2]), int(iexp[3]), int(iexp[4]))
            assert hit.perp_distance == fexp[0] and hit.wall_u == fexp[1]
        m += 1


def _map_from_arrays(kind, didx, ndoor):
    doors = [None] * ndoor
    for y, x in zip(*np.nonzero(didx >= 0)):
        doors[int(didx[y, x])] = tc.Door((int(x), int(y)), tc.KeyColor.RED, False)
    floor = np.argwhere(kind == 0)
    spawn = (int(floor[0][1]), int(floor[0][0]))
    return tc.TileMap(kind, np.zeros_like(kind), doors, [], [spawn])


def test_scalar_api_matches_batch():
    spec = tc.make_env("key-door")
    n = 4
    bs = tc.batch_reset(spec, n, seed=7, device=DEV)
    root = tc.from_seed(7)
    states = []
    for i in range(n):
        st, obs = tc.reset(spec, tc.split(root, i))
        assert bs.state(i) == st
        assert np.array_equal(bs.frames[i].cpu().numpy(), obs)
        states.append(st)
    rnd = random.Random(b"batch-vs-scalar")
    for _ in range(40):
        acts = [rnd.choice(spec.action_set) for _ in range(n)]
        bs, rewards, dones = tc.batch_step(bs, [int(a) for a in acts])
        rewards, dones = rewards.cpu().numpy(), dones.cpu().numpy()
        for i in range(n):
            r = tc.step(spec, states[i], acts[i])
            assert rewards[i] == r.reward and dones[i] == r.done
            if r.done:
                states[i], obs = tc.reset(spec, r.state.rng)
                assert np.array_equal(bs.frames[i].cpu().numpy(), obs)
            else:
                states[i] = r.state
                assert np.array_equal(bs.frames[i].cpu().numpy(), r.observation)
            assert bs.state(i) == states[i]


def test_rollout_kernel_equals_batch_steps():
    spec = tc.make_env("dmlab-random-goal-01", max_steps=20)
    n, k, seed = 200, 37, 5
    a = tc.batch_reset(spec, n, seed, device=DEV)
    b = tc.batch_reset(spec, n, seed, device=DEV)
    ring = torch.empty((k, n, 64, 64, 3), dtype=torch.uint8, device=DEV)
    res = tc.rollout(a, k, seed, frames=ring, record=True)
    acts = tc.policy_actions(spec, n, k, seed)
    for s in range(k):
        b, rew, done = tc.batch_step(b, acts[s], reuse=True)
        assert torch.equal(res["frames"][s], b.frames), s
        assert torch.equal(res["rewards"][s], rew), s
        assert torch.equal(res["dones"][s] != 0, done), s
    ha, hb = a.host_state(), b.host_state()
    for key in ha:
        assert np.array_equal(ha[key], hb[key]), key


def test_rollout_continuation_and_sharding():
    """Global env indices: two half-shards stepped separately == one batch."""
    spec = tc.make_env("key-door", max_steps=30)
    n, k, seed = 256, 40, 9
    full = tc.batch_reset(spec, n, seed, device=DEV)
    tc.rollout(full, k // 2, seed)
    tc.rollout(full, k - k // 2, seed, step0=k // 2)
    halves = [tc.batch_reset(spec, n // 2, seed, device=DEV, base=b, n_total=n)
              for b in (0, n // 2)]
    for h in halves:
        tc.rollout(h, k, seed)
    hf = full.host_state()
    for j, h in enumerate(halves):
        hh = h.host_state()
        sl = slice(j * n // 2, (j + 1) * n // 2)
        for key in hf:
            assert np.array_equal(hf[key][sl], hh[key]), key
        assert torch.equal(full.frames[sl], h.frames)


def test_device_policy_actions_match_host_table():
    spec = tc.make_env("health-gathering")
    table = tc.policy_actions(spec, 1000, 4, seed=3)
    for s in range(4):
        row = tc.policy_actions_device(spec, s, 1000, 3, device=DEV)
        assert np.array_equal(row.cpu().numpy(), table[s])
        part = tc.policy_actions_device(spec, s, 300, 3, base=500, n_total=1000, device=DEV)
        assert np.array_equal(part.cpu().numpy(), table[s, 500:800])


def test_validate_and_contract_errors():
    spec = tc.make_env("simple")
    bs = tc.batch_reset(spec, 8, 0, device=DEV)
    with pytest.raises(tc.ContractError):
        tc.batch_step(bs, [int(tc.Action.STRAFE_LEFT)] * 8)
    with pytest.raises(tc.ContractError):
        tc.batch_step(bs, [0] * 7)
    with pytest.raises(tc.ContractError):
        tc.batch_step(bs, [9] * 8)
    bs, _, _ = tc.batch_step(bs, [0] * 8, validate=True)
    bad = torch.full((8,), int(tc.Action.STRAFE_LEFT), dtype=torch.int64, device=DEV)
    bs, _, _ = tc.batch_step(bs, bad)
    with pytest.raises(tc.ContractError):
        bs.check()


def test_auto_reset_reports_final_step():
    spec = tc.make_env("simple", max_steps=2)
    bs = tc.batch_reset(spec, 3, seed=1, device=DEV)
    noop = [int(tc.Action.NOOP)] * 3
    bs, _, dones = tc.batch_step(bs, noop)
    assert not dones.any()
    bs, _, dones = tc.batch_step(bs, noop)
    assert dones.all() and bs.last_truncated.all() and not bs.last_terminated.any()
    for i in range(3):
        assert bs.state(i).t == 0 and not bs.state(i).done


def test_large_batch_matches_oracle_sample():
    """BASELINE C2 size (4096 envs): full bit-exact compare on every 10th step."""
    spec = tc.make_env("my-way-home")
    _compare_rollout(spec, 4096, 30, seed=0, check_every=10)


def test_batch_step_host_matches_device_path():
    spec = tc.make_env("key-door", max_steps=25)
    n, steps = 300, 40
    acts = tc.policy_actions(spec, n, steps, 2)
    a = tc.batch_reset(spec, n, 2, device=DEV)
    b = tc.batch_reset(spec, n, 2, device=DEV)
    for s in range(steps):
        a, ra, da = tc.batch_step(a, acts[s], reuse=True)
        b, rb, db = tc.batch_step_host(b, acts[s], reuse=True)
        assert isinstance(rb, np.ndarray) and rb.dtype == np.float64 and db.dtype == np.bool_
        assert np.array_equal(ra.cpu().numpy(), rb) and np.array_equal(da.cpu().numpy(), db)
        assert torch.equal(a.frames, b.frames)
    ha, hb = a.host_state(), b.host_state()
    for k in ha:
        assert np.array_equal(ha[k], hb[k]), k
    with pytest.raises(tc.ContractError):
        tc.batch_step_host(b, [int(tc.Action.STRAFE_LEFT)] * n)
    bad = acts[0].copy()
    bad[n // 2] = 99
    with pytest.raises(tc.ContractError):
        tc.batch_step_host(b, bad)
    bad[n // 2] = -1
    with pytest.raises(tc.ContractError):
        tc.batch_step_host(b, bad)
    # a rejected step leaves the state usable and unchanged
    a, ra, da = tc.batch_step(a, acts[1], reuse=True)
    b, rb, db = tc.batch_step_host(b, acts[1], reuse=True)
    assert np.array_equal(ra.cpu().numpy(), rb) and torch.equal(a.frames, b.frames)
    b.check()


@pytest.mark.parametrize("n", [1, 5, 37])
def test_batch_step_host_small_batches(n):
    # fewer envs than CTAs: idle CTAs still take part in the result hand-off
    spec = tc.make_env("dmlab-random-goal-01", max_steps=12)
    acts = tc.policy_actions(spec, n, 30, 4)
    a = tc.batch_reset(spec, n, 4, device=DEV)
    b = tc.batch_reset(spec, n, 4, device=DEV)
    for s in range(30):
        a, ra, da = tc.batch_step(a, acts[s], reuse=True)
        b, rb, db = tc.batch_step_host(b, acts[s], reuse=True)
        assert np.array_equal(ra.cpu().numpy(), rb) and np.array_equal(da.cpu().numpy(), db)
    assert torch.equal(a.frames, b.frames)


def test_gym_vecenv_and_env_match_core():
    from paper_2605_19926_b200 import gym
    spec = tc.make_env("simple", max_steps=30)
    n, steps = 8, 50
    tags = np.array([int(a) for a in spec.action_set])
    rnd = np.random.default_rng(0)
    idx = rnd.integers(0, len(tags), size=(steps, n))
    v = gym.make_vec("simple", n, seed=3, max_steps=30)
    vd = gym.make_vec("simple", n, seed=3, max_steps=30)
    bs = tc.batch_reset(spec, n, 3, device=DEV)
    for s in range(steps):
        obs, r, d, info = v.step(idx[s])
        obs2, r2, d2, _ = vd.step(torch.as_tensor(idx[s], device=DEV))
        bs, rr, dd = tc.batch_step(bs, tags[idx[s]])
        assert torch.equal(obs, bs.frames) and torch.equal(obs2, bs.frames)
        assert torch.equal(r, rr) and torch.equal(d, dd) and torch.equal(r2, rr)
    v.check()
    vd.check()
    e = gym.make("simple", max_steps=30)
    obs, _ = e.reset(seed=3)
    assert np.array_equal(obs, tc.batch_reset(spec, 1, 3, device=DEV).frames[0].cpu().numpy())
    o, rwd, term, trunc, info = e.step(0)
    assert o.shape == (64, 64, 3) and isinstance(rwd, float)


def test_cli_bench_report_schema():
    from paper_2605_19926_b200 import cli
    rep = cli.bench("key-door", 64, 20, 0, 64, 64)
    assert rep["schema_version"] == 1 and rep["kind"] == "bench"
    assert set(rep["config"]) >= {"env", "n", "steps", "seed", "width", "height", "threads"}
    assert set(rep["results"]) >= {"steps_per_second", "frames_per_second", "us_per_frame",
                                   "reward_sum"}
    assert rep["results"]["steps_per_second"] > 0


@pytest.mark.parametrize("env,n,m", [("my-way-home", 4096, 300), ("key-door", 2048, 1)])
def test_back_to_back_steps_without_sync(env, n, m):
    """Consecutive one-wave step launches overlap (per-CTA launch chain,
    csrc batch_kernel): K steps of two batches on the same spec and stream,
    actions pre-staged on the device, no host read in between -- the final
    state, frames and last outputs equal the oracle's."""
    spec = tc.make_env(env, max_steps=23)
    k = 40
    runs = []
    for nn, seed in ((n, 3), (m, 4)):
        acts = tc.policy_actions(spec, nn, k, seed)
        runs.append((tc.batch_reset(spec, nn, seed, device=DEV),
                     torch.from_numpy(acts).to(DEV), orc.Rollout(spec, nn, seed), acts))
    torch.cuda.synchronize()
    states = [r[0] for r in runs]
    outs = [None, None]
    for s in range(k):
        for j, (_, acts_dev, _, _) in enumerate(runs):
            states[j], rew, done = tc.batch_step(states[j], acts_dev[s], reuse=True,
                                                 copy_outputs=False)
            outs[j] = (rew, done)
    torch.cuda.synchronize()
    for j, (_, _, r, acts) in enumerate(runs):
        for s in range(k):
            r.step(acts[s])
        bs = states[j]
        assert np.array_equal(outs[j][0].cpu().numpy(), r.out["rewards"]), j
        assert np.array_equal(outs[j][1].cpu().numpy(), r.out["dones"] != 0), j
        assert np.array_equal(bs.frames.cpu().numpy(), r.out["frames"]), j
        _assert_state(bs, r.state, f"batch {j}")
        bs.check()


def test_multimap_batch_matches_per_group_oracle():
    """Heterogeneous maps (multimap.py): groups over different specs (a
    synthetic map, key-door with doors / sprites, my-way-home) share one
    output block; group g equals the oracle's homogeneous run with base =
    its offset, whether stepped with numpy or device actions."""
    syn = tc.EnvSpec(id="syn-mm", map=random_tilemap(random.Random(77)),
                     action_set=tc.suite.STRAFE_ACTIONS,
                     goal_mode=tc.GoalMode.RANDOM_PER_EPISODE, max_steps=19,
                     living_reward=0.01, health_decay=1.0, health_restore=10.0)
    specs = [syn, tc.make_env("key-door", max_steps=31), tc.make_env("my-way-home", max_steps=27)]
    counts = [700, 129, 1500]
    seed, k = 9, 45
    mb = tc.multi_reset(specs, counts, seed, device=DEV)
    n = sum(counts)
    assert mb.frames.shape == (n, 64, 64, 3)
    refs, acts = [], []
    for spec, c, off in zip(specs, counts, mb.offsets):
        refs.append(orc.Rollout(spec, c, seed, base=off))
        acts.append(tc.policy_actions(spec, c, k, seed + off))
    assert np.array_equal(mb.frames.cpu().numpy(),
                          np.concatenate([r.out["frames"] for r in refs])), "reset frames"
    full = np.concatenate(acts, axis=1)
    full_dev = torch.from_numpy(full).to(DEV)
    for s in range(k):
        a = full[s] if s % 2 == 0 else full_dev[s]
        mb, rew, done = tc.multi_step(mb, a, reuse=True)
        for r, ac in zip(refs, acts):
            r.step(ac[s])
        if s % 7 == 0 or s == k - 1:
            assert np.array_equal(rew.cpu().numpy(),
                                  np.concatenate([r.out["rewards"] for r in refs])), s
            assert np.array_equal(done.cpu().numpy(),
                                  np.concatenate([r.out["dones"] != 0 for r in refs])), s
            assert np.array_equal(mb.frames.cpu().numpy(),
                                  np.concatenate([r.out["frames"] for r in refs])), s
            for g, r in zip(mb.groups, refs):
                _assert_state(g, r.state, f"step {s} group {g.spec.id}")
    mb.check()
    assert mb.group_of(0) == 0 and mb.group_of(700) == 1 and mb.group_of(n - 1) == 2
