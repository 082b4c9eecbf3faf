"""Round-2 golden fixtures, generated FROM THE REFERENCE (run here, in the
container that has /root/reference; never on the GPU box):

    python tests/golden/make_golden_r2.py

Writes tests/golden/digests_r2.json: rollout digests (SURVEY.md §8(c) recipe,
tests/_digest.py order) computed by the reference's compiled backend
(oracle/_ref) for the cases round 1 left unpinned (VERDICT r01 "next" 1):

* C1 -- my-way-home, 1 env, 1000 steps (BASELINE.json configs[0]) with the
  final state;
* maps larger than 4096 cells (64x64 tiles and beyond) at the C5 density;
* 32-door maps (the reference's limit, pkg/src/tilecast/tables.py:110-113);
* the C5 bench map (bench.synthetic_spec, random.Random(20260518));
* the binding equivalence cases of pkg/bindings/tests/test_equivalence.py:26-89
  (VecEnv key-door 8 x 1000 seed 42; scalar simple 1000 steps seed 7 with
  the test's reset-on-done rule; CLI bench key-door 4 x 200 seed 9 reward sum).

The maps come from paper_2605_19926_b200.synthetic.large_tilemap (seeded
random.Random); the map arrays go to the reference as its own TileMap.
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))

import tilecast as ref  # noqa: E402
from tilecast import backend as ref_backend  # noqa: E402
from tilecast.batch import batch_reset, batch_step, policy_actions  # noqa: E402
from tilecast import geometry as rg  # noqa: E402
from tilecast import suite as rs  # noqa: E402

import bench  # noqa: E402  (the C5 spec definition)
from paper_2605_19926_b200.synthetic import large_tilemap  # noqa: E402

STATE_ORDER = ("px", "py", "dx", "dy", "health", "inv", "t", "rctr", "done", "agoal",
               "dopen", "ealive")

# (name, width, height, n_doors, n_entities, n_spawns, map seed, doors_at_spawns)
LARGE_MAPS = [
    ("large-64x64", 64, 64, 2, 6, 8, 11, False),
    ("large-96x80", 96, 80, 6, 12, 8, 12, True),
    ("large-160x128", 160, 128, 4, 16, 16, 13, True),
    ("doors32-20x20", 20, 20, 32, 6, 8, 21, True),
    ("doors32-90x72", 90, 72, 32, 10, 8, 22, True),
]


def ref_tilemap(m):
    doors = tuple(rg.Door(tuple(d.tile), rg.KeyColor(int(d.color)), bool(d.locked))
                  for d in m.doors)
    ents = tuple(rg.EntityInit(rg.EntityKind(int(e.kind)), tuple(e.tile),
                               None if e.color is None else rg.KeyColor(int(e.color)))
                 for e in m.entities)
    return rg.TileMap(np.array(m.kind), np.array(m.wall_color), doors, ents,
                      tuple(tuple(s) for s in m.spawn_candidates))


def large_spec_kwargs(name):
    for nm, w, h, nd, ne, ns, seed, das in LARGE_MAPS:
        if nm == name:
            return dict(width=w, height=h, n_doors=nd, n_entities=ne, n_spawns=ns,
                        seed=seed, doors_at_spawns=das)
    raise KeyError(name)


def ref_large_spec(name, max_steps=40, **kw):
    a = large_spec_kwargs(name)
    m = large_tilemap(random.Random(a["seed"]), a["width"], a["height"], n_doors=a["n_doors"],
                      n_entities=a["n_entities"], n_spawns=a["n_spawns"],
                      doors_at_spawns=a["doors_at_spawns"])
    return rs.EnvSpec(id=name, map=ref_tilemap(m), action_set=rs.STRAFE_ACTIONS,
                      goal_mode=rs.GoalMode.RANDOM_PER_EPISODE, max_steps=max_steps,
                      living_reward=0.01, health_decay=0.5, health_restore=10.0, **kw)


def ref_c5_spec():
    import paper_2605_19926_b200 as tc
    ours = bench.synthetic_spec()
    return rs.EnvSpec(id=ours.id, map=ref_tilemap(ours.map), action_set=rs.STRAFE_ACTIONS,
                      goal_mode=rs.GoalMode.RANDOM_PER_EPISODE, max_steps=ours.max_steps,
                      obs_width=ours.obs_width, obs_height=ours.obs_height,
                      living_reward=ours.living_reward, health_decay=ours.health_decay,
                      health_restore=ours.health_restore), tc


def digest_spec(spec, n, steps, seed, keep_final=False):
    acts = policy_actions(spec, n, steps, seed)
    bs = batch_reset(spec, n, seed)
    h = hashlib.blake2b(digest_size=16)
    h.update(bs.frames.tobytes())
    rsum, dones, evor = 0.0, 0, 0
    for s in range(steps):
        bs, r, d = batch_step(bs, acts[s], reuse=True)
        for k in STATE_ORDER:
            h.update(np.ascontiguousarray(getattr(bs._sb, k)).tobytes())
        h.update(r.tobytes())
        h.update(d.tobytes())
        h.update(bs._ob.truncs.tobytes())
        h.update(bs._ob.events.tobytes())
        h.update(bs.frames.tobytes())
        rsum += float(r.sum())
        dones += int(d.sum())
        evor |= int(np.bitwise_or.reduce(bs._ob.events))
    out = dict(n=n, steps=steps, seed=seed, digest=h.hexdigest(), reward_sum=rsum,
               dones=dones, events_or=evor)
    if keep_final:
        fin = {}
        for k in ("px", "py", "dx", "dy", "health"):
            fin[k] = [float.hex(float(v)) for v in getattr(bs._sb, k)]
        for k in ("inv", "t", "rkey", "rctr", "done", "agoal"):
            fin[k] = [int(v) for v in getattr(bs._sb, k)]
        fin["frame_sha"] = hashlib.sha256(bs.frames.tobytes()).hexdigest()
        out["final"] = fin
    return out


def scalar_case(steps=1000, seed=7):
    """pkg/bindings/tests/test_equivalence.py:46-70 on the core scalar API:
    reset(split(from_seed(seed + s), 0)) whenever the episode is done."""
    spec = ref.make_env("simple")
    tags = policy_actions(spec, 1, steps, seed)[:, 0]
    state, obs = ref.reset(spec, ref.split(ref.from_seed(seed), 0))
    h = hashlib.blake2b(digest_size=16)
    h.update(obs.tobytes())
    rsum, resets = 0.0, 0
    for s in range(steps):
        if state.done:
            state, obs = ref.reset(spec, ref.split(ref.from_seed(seed + s), 0))
            h.update(obs.tobytes())
            resets += 1
        res = ref.step(spec, state, int(tags[s]))
        state = res.state
        h.update(np.float64(res.reward).tobytes())
        h.update(bytes([res.info["terminated"], res.info["truncated"]]))
        h.update(res.observation.tobytes())
        rsum += res.reward
    return dict(env="simple", steps=steps, seed=seed, digest=h.hexdigest(),
                reward_sum=rsum, resets=resets)


def main() -> None:
    print("reference backend:", ref_backend.backend_name())
    out = {}
    spec = ref.make_env("my-way-home")
    out["c1"] = dict(env="my-way-home", **digest_spec(spec, 1, 1000, 0, keep_final=True))
    print("c1", out["c1"]["digest"])
    for nm, *_ in LARGE_MAPS:
        spec = ref_large_spec(nm)
        n, steps = (96, 60) if "doors32" not in nm else (128, 80)
        out[nm] = dict(map=nm, **digest_spec(spec, n, steps, 3))
        print(nm, out[nm])
    spec = ref_large_spec("large-96x80", obs_width=128, obs_height=96)
    out["large-96x80-128x96"] = dict(map="large-96x80", obs=[128, 96],
                                     **digest_spec(spec, 48, 40, 4))
    print(out["large-96x80-128x96"])
    c5, _ = ref_c5_spec()
    out["c5-map"] = dict(**digest_spec(c5, 4096, 30, 0))
    print("c5", out["c5-map"])
    out["vec-key-door"] = dict(env="key-door", **digest_spec(ref.make_env("key-door"), 8, 1000,
                                                            42))
    print("vec", out["vec-key-door"])
    out["scalar-simple"] = scalar_case()
    print("scalar", out["scalar-simple"])
    cli = digest_spec(ref.make_env("key-door"), 4, 200, 9)
    out["cli-key-door"] = dict(env="key-door", n=4, steps=200, seed=9,
                               reward_sum=cli["reward_sum"])
    (HERE / "digests_r2.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
