"""Host-side layer (CPU only): registry, map parsing, tables, RNG, sharding
-- all pinned against fixtures generated from the reference."""

from __future__ import annotations

import random

import numpy as np
import pytest

from conftest import GOLDEN, unpack_map

import paper_2605_19926_b200 as tc
from paper_2605_19926_b200 import rng
from paper_2605_19926_b200.shard import shard_range
from paper_2605_19926_b200.synthetic import random_tilemap
from paper_2605_19926_b200.tables import Tables

REF_IDS = ("dmlab-random-goal-01", "dmlab-random-goal-02", "dmlab-random-goal-03",
           "dmlab-static-01", "dmlab-static-02", "dmlab-static-03", "health-gathering",
           "key-corridor", "key-door", "my-way-home", "simple")


def test_registry_ids_match_reference():
    assert tc.registered_ids() == REF_IDS


def test_tables_match_reference_fixture():
    g = np.load(GOLDEN / "tables.npz")
    for env in REF_IDS:
        t = tc.make_env(env).tables
        for f in Tables.ARRAY_FIELDS:
            ref = g[f"{env}|{f}"]
            got = getattr(t, f)
            assert got.dtype == ref.dtype and got.shape == ref.shape, (env, f)
            assert np.array_equal(got, ref), (env, f)


def test_synthetic_maps_match_reference_generator():
    g = np.load(GOLDEN / "synthetic_maps.npz")
    for s in range(20):
        assert random_tilemap(random.Random(s)) == unpack_map(g[f"s{s}"]), s


def test_make_env_overrides_and_contracts():
    s = tc.make_env("key-door", obs_width=96, obs_height=48, max_steps=7)
    assert (s.obs_width, s.obs_height, s.max_steps) == (96, 48, 7)
    assert s.tables.coef.shape == (96,)
    with pytest.raises(tc.ContractError):
        tc.make_env("nope")
    with pytest.raises(tc.ContractError):
        tc.make_env("key-door", action_set=())
    with pytest.raises(tc.ContractError):
        tc.make_env("key-door", obs_width=4)


def test_register_env_and_parse_errors():
    spec = tc.register_env("unit-test-room", "#####\n#S.G#\n#####\n", max_steps=9)
    assert spec.tables.goal_ent.tolist() == [0]
    with pytest.raises(tc.ContractError):
        tc.register_env("unit-test-room", "#####\n#S.G#\n#####\n")
    with pytest.raises(tc.MapParseError):
        tc.parse_map("#####\n#S.G.\n#####\n")   # unsealed
    with pytest.raises(tc.MapParseError):
        tc.parse_map("#####\n#..G#\n#####\n")   # no spawn
    with pytest.raises(tc.MapParseError):
        tc.parse_map("#####\n#S?G#\n#####\n")   # unknown symbol


def test_rng_streams():
    assert rng.mix(0x9E3779B97F4A7C15) == 0xE220A8397B1DCDAF
    root = rng.from_seed(3)
    keys, ctrs = rng.seed_streams(3, 100, 8)
    assert [int(k) for k in keys] == [rng.split(root, 100 + i).key for i in range(8)]
    assert not ctrs.any()
    s = rng.RngState(12345, 7)
    v, s2 = rng.next_below(s, 10)
    assert 0 <= v < 10 and s2.counter == 8
    big = rng.policy_uniform(rng.policy_key(0), np.arange(1000, dtype=np.uint64), 5)
    assert big.min() >= 0 and big.max() < 5


@pytest.mark.parametrize("n,world", [(4096, 1), (4096, 8), (1 << 20, 8), (10, 3), (7, 7)])
def test_shard_range_partitions(n, world):
    shards = [shard_range(n, world, r) for r in range(world)]
    assert sum(s.n for s in shards) == n
    assert shards[0].base == 0
    for a, b in zip(shards, shards[1:]):
        assert a.base + a.n == b.base
    assert max(s.n for s in shards) - min(s.n for s in shards) <= 1


def test_event_tags_and_actions():
    assert tc.event_tags((1 << 0) | (1 << 9)) == ("picked_key_red", "truncated")
    assert tc.ACTIONS_BY_NAME["noop"] == tc.Action.NOOP
    assert len(tc.suite.NAV_ACTIONS) == 5 and len(tc.suite.STRAFE_ACTIONS) == 7


def test_multimap_contracts():
    """Heterogeneous-map batches check their groups on the host before any
    device work (multimap.py)."""
    a = tc.make_env("my-way-home")
    b = tc.make_env("key-door", obs_width=32, obs_height=32)
    with pytest.raises(tc.ContractError, match="observation shape"):
        tc.multi_reset([a, b], [4, 4], seed=0)
    with pytest.raises(tc.ContractError, match=">= 1 env"):
        tc.multi_reset([a, a], [4, 0], seed=0)
    with pytest.raises(tc.ContractError, match="equal length"):
        tc.multi_reset([a], [4, 4], seed=0)


def test_multimap_group_index():
    from paper_2605_19926_b200.multimap import MultiMapBatch
    mb = MultiMapBatch(groups=(), offsets=(0, 700, 829), n=2329, _ob=None)
    assert [mb.group_of(i) for i in (0, 699, 700, 828, 829, 2328)] == [0, 0, 1, 1, 2, 2]
    with pytest.raises(tc.ContractError):
        mb.group_of(2329)
