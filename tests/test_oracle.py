"""The oracle port (oracle/tilecast_oracle.c) pinned against the reference:
golden fixtures generated FROM the reference (tests/golden/make_golden.py),
the reference's own known-answer tests, and -- when oracle/_ref is built --
the reference's compiled kernel run side by side."""

from __future__ import annotations

import math
import random
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, unpack_map
from _digest import Digest

import paper_2605_19926_b200 as tc
from paper_2605_19926_b200 import rng
from paper_2605_19926_b200.tables import build_tables
from oracle import oracle as orc


def oracle_digest(env, overrides, n, steps, seed, n_threads=None):
    spec = tc.make_env(env, **overrides)
    acts = tc.policy_actions(spec, n, steps, seed)
    r = orc.Rollout(spec, n, seed, n_threads=n_threads)
    d = Digest()
    d.frames(r.out["frames"])
    for s in range(steps):
        r.step(acts[s])
        d.step(r.state, r.out["rewards"], r.out["dones"], r.out["truncs"], r.out["events"],
               r.out["frames"])
    return d


SMALL = lambda cases: [c for c in cases if c["n"] * c["steps"] <= 20000]  # noqa: E731


def test_oracle_matches_reference_digests(golden_digests):
    for case in SMALL(golden_digests):
        d = oracle_digest(case["env"], case["overrides"], case["n"], case["steps"], case["seed"])
        assert d.hexdigest() == case["digest"], case
        assert d.reward_sum == case["reward_sum"]
        assert d.dones == case["dones"]
        assert d.events_or == case["events_or"]


@pytest.mark.slow
def test_oracle_matches_reference_digests_large(golden_digests):
    for case in golden_digests:
        if case in SMALL(golden_digests):
            continue
        d = oracle_digest(case["env"], case["overrides"], case["n"], case["steps"], case["seed"])
        assert d.hexdigest() == case["digest"], case


def test_oracle_thread_count_invariance():
    a = oracle_digest("health-gathering", {}, 64, 40, 9, n_threads=1).hexdigest()
    b = oracle_digest("health-gathering", {}, 64, 40, 9, n_threads=4).hexdigest()
    assert a == b


def test_oracle_golden_frames():
    g = np.load(GOLDEN / "golden_frames.npz")
    from paper_2605_19926_b200.maps import SHIPPED_MAPS
    for key in g.files:
        env, sx, sy, dx, dy = key.split("|")
        tmap = tc.parse_map(SHIPPED_MAPS[env])
        t = build_tables(tmap)
        goal = int(t.goal_ent[0]) if t.goal_ent.size else -1
        st, frame, *_ = orc.render_into(t, float(sx), float(sy), float(dx), float(dy),
                                        np.zeros(t.n_doors, np.uint8),
                                        np.ones(t.n_entities, np.uint8), goal)
        assert st == 0
        assert np.array_equal(frame, g[key]), key


def test_oracle_rays_match_reference():
    g = np.load(GOLDEN / "rays.npz")
    m = 0
    while f"m{m}_kind" in g.files:
        kind, didx, dopen = g[f"m{m}_kind"], g[f"m{m}_didx"], g[f"m{m}_dopen"]
        for q, iexp, fexp in zip(g[f"m{m}_q"], g[f"m{m}_i"], g[f"m{m}_f"]):
            st, mx, my, side, perp, wu, steps = orc.cast_ray(kind, didx, dopen, *q)
            assert (st, mx, my, side, steps) == tuple(int(v) for v in iexp)
            assert perp == fexp[0] and wu == fexp[1]
        m += 1
    assert m >= 10


def test_oracle_random_frames_match_reference():
    g = np.load(GOLDEN / "frames_random.npz")
    m = 0
    while f"f{m}_frame" in g.files:
        tmap = unpack_map(g[f"f{m}_map"])
        frame_exp = g[f"f{m}_frame"]
        t = build_tables(tmap, obs_width=frame_exp.shape[1], obs_height=frame_exp.shape[0])
        px, py, dx, dy = g[f"f{m}_pose"]
        goal = int(t.goal_ent[0]) if t.goal_ent.size else -1
        st, frame, *_ = orc.render_into(t, px, py, dx, dy, g[f"f{m}_dopen"],
                                        np.ones(t.n_entities, np.uint8), goal)
        assert st == 0 and np.array_equal(frame, frame_exp), m
        m += 1


def test_splitmix_kat():
    # pkg/tests/test_rng.py:38-47 known-answer values
    s = rng.RngState(0, 0)
    vals = []
    for _ in range(3):
        v, s = rng.next_u64(rng.RngState(s.key, s.counter))
        vals.append(v)
    ref = rng.mix(0), rng.mix(rng.GOLDEN), rng.mix(2 * rng.GOLDEN & rng.M64)
    assert tuple(vals) == ref
    assert rng.mix(0x9E3779B97F4A7C15) == 0xE220A8397B1DCDAF
    assert rng.mix(0x9E3779B97F4A7C15 * 2 & rng.M64) == 0x6E789E6AA1B965F4
    assert rng.mix(0x9E3779B97F4A7C15 * 3 & rng.M64) == 0x06C45D188009454F


def test_seed_streams_and_policy_match_host():
    keys, ctrs = rng.seed_streams(7, 3, 50)
    st = orc.alloc_state(50, 0, 0)
    orc.seed_streams(7, 3, 50, st)
    root = rng.from_seed(7)
    for i in range(50):
        assert int(keys[i]) == rng.split(root, 3 + i).key == int(st["rkey"][i])
    spec = tc.make_env("health-gathering")
    table = tc.policy_actions(spec, 40, 5, seed=11)
    tags = np.array([int(a) for a in spec.action_set], np.int64)
    for s in range(5):
        row = orc.policy_actions(rng.policy_key(11), s, 40, 10, 20, tags)
        assert np.array_equal(row, table[s, 10:30])


def test_oracle_vs_reference_compiled_side_by_side():
    """Step-by-step comparison with the reference's own compiled kernel."""
    ref_dir = ROOT / "oracle" / "_ref"
    if not (ref_dir / "tilecast").exists():
        pytest.skip("oracle/_ref not built")
    sys.path.insert(0, str(ref_dir))
    try:
        import tilecast as ref
        from tilecast.batch import batch_reset, batch_step
    finally:
        sys.path.remove(str(ref_dir))
    for env, ov in (("key-door", {"max_steps": 30}), ("health-gathering", {}),
                    ("dmlab-random-goal-02", {"max_steps": 40, "obs_width": 48,
                                              "obs_height": 32})):
        spec_r, spec_m = ref.make_env(env, **ov), tc.make_env(env, **ov)
        n, steps = 24, 50
        acts = tc.policy_actions(spec_m, n, steps, 3)
        bs = batch_reset(spec_r, n, 3)
        r = orc.Rollout(spec_m, n, 3)
        assert np.array_equal(bs.frames, r.out["frames"])
        for s in range(steps):
            bs, rew, done = batch_step(bs, acts[s], reuse=True)
            r.step(acts[s])
            assert np.array_equal(bs.frames, r.out["frames"])
            assert np.array_equal(rew, r.out["rewards"])
            for k in r.state:
                assert np.array_equal(getattr(bs._sb, k), r.state[k]), (env, s, k)
