"""Regenerate the golden fixtures in tests/golden/ FROM THE REFERENCE.

Run here (the container that has /root/reference), never on the GPU box:

    python tests/golden/make_golden.py

It imports the reference package (compiled backend from oracle/_ref, built by
oracle/build_ref.sh, else /root/reference/pkg/src with the pure-Python
backend) and records:

* golden_frames.npz  -- the 8 pinned poses of pkg/tools/gen_goldens.py:19-28
                        (the reference's own golden npz is absent from the
                        snapshot);
* digests.json       -- rollout digests (SURVEY.md §8(c) recipe) for the
                        shipped envs, with reward sums / done counts;
* rays.npz           -- random sealed maps (pkg/tests/conftest.py:40-92) with
                        50 rays each and the reference cast_ray results;
* frames_random.npz  -- render_frame on random maps/poses with doors and
                        entities, plus zbuf;
* synthetic_maps.npz -- conftest.random_tilemap(random.Random(s)) arrays for
                        s in 0..19, pinning our synthetic-map generator;
* tables.npz         -- build_tables output (tables.py:92-184) of every
                        registered env, pinning our registry + map parser.

``python tests/golden/make_golden.py tables`` regenerates only tables.npz.
"""

from __future__ import annotations

import hashlib
import importlib.util
import json
import math
import random
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF_BUILT = ROOT / "oracle" / "_ref"
REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")

sys.path.insert(0, str(REF_BUILT if REF_BUILT.exists() else REF_SRC))
import tilecast as ref  # noqa: E402
from tilecast import backend as ref_backend  # noqa: E402
from tilecast.batch import batch_reset, batch_step, policy_actions  # noqa: E402
from tilecast.geometry import CellTag, Pose, Vec2  # noqa: E402
from tilecast.mapdsl import load_map_file, parse_map  # noqa: E402
from tilecast.render import render_frame  # noqa: E402

_spec = importlib.util.spec_from_file_location("ref_conftest", REF_TESTS / "conftest.py")
ref_conftest = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(ref_conftest)

D = 0.7071067811865476
POSES = [  # pkg/tools/gen_goldens.py:19-28
    ("simple", 1.5, 1.5, 1.0, 0.0), ("simple", 1.5, 1.5, 0.0, 1.0),
    ("key-door", 1.5, 1.5, D, D), ("key-corridor", 1.5, 3.5, 1.0, 0.0),
    ("my-way-home", 4.5, 2.5, 0.0, 1.0), ("my-way-home", 20.5, 12.5, -D, D),
    ("health-gathering", 7.5, 8.5, -1.0, 0.0), ("dmlab-02", 1.5, 1.5, 0.0, 1.0),
]

# (env, overrides, n, steps, seed); the SURVEY.md §8(c) list plus small cases
DIGEST_CASES = [
    ("my-way-home", {}, 16, 50, 0),
    ("key-door", {}, 16, 50, 0),
    ("my-way-home", {}, 4096, 100, 0),
    ("key-door", {}, 16384, 20, 0),
    ("dmlab-static-03", {"obs_width": 128, "obs_height": 128}, 8192, 20, 0),
    ("health-gathering", {}, 1024, 300, 0),
    ("my-way-home", {"max_steps": 37}, 4096, 100, 0),
    ("key-door", {"max_steps": 150}, 4096, 200, 1),
    ("dmlab-random-goal-01", {"max_steps": 60}, 4096, 200, 2),
    ("simple", {"max_steps": 120}, 4096, 300, 3),
    ("dmlab-random-goal-01", {"max_steps": 30}, 32, 80, 2),
    ("key-corridor", {"max_steps": 25}, 64, 60, 4),
    ("dmlab-static-02", {"obs_width": 40, "obs_height": 24}, 64, 40, 5),
    ("dmlab-random-goal-03", {"obs_width": 37, "obs_height": 29}, 48, 40, 6),
]

STATE_ORDER = ("px", "py", "dx", "dy", "health", "inv", "t", "rctr", "done", "agoal",
               "dopen", "ealive")


def digest_case(env, overrides, n, steps, seed):
    spec = ref.make_env(env, **overrides)
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
    return dict(env=env, overrides=overrides, n=n, steps=steps, seed=seed,
                digest=h.hexdigest(), reward_sum=rsum, dones=dones, events_or=evor)


def main() -> None:
    print("reference backend:", ref_backend.backend_name())
    maps_dir = REF_SRC / "tilecast" / "maps"
    frames = {}
    for env, sx, sy, dx, dy in POSES:
        tmap = parse_map(load_map_file(maps_dir / f"{env}.map")).unwrap()
        frames[f"{env}|{sx}|{sy}|{dx}|{dy}"] = render_frame(tmap, Pose.looking(Vec2(sx, sy),
                                                                                Vec2(dx, dy)))
    np.savez_compressed(HERE / "golden_frames.npz", **frames)

    # random maps + rays (test_backends.py:40-54 style)
    rng = random.Random(b"graft-rays")
    rays = {}
    for m in range(12):
        t = ref_conftest.random_tilemap(rng)
        floor = [(x, y) for y in range(t.height) for x in range(t.width)
                 if t.kind[y, x] == CellTag.FLOOR]
        flags = np.array([rng.random() < 0.5 for _ in t.doors], dtype=np.uint8)
        q, res = [], []
        for _ in range(50):
            fx, fy = rng.choice(floor)
            ox, oy = fx + rng.uniform(0.1, 0.9), fy + rng.uniform(0.1, 0.9)
            a = rng.uniform(0.0, 2.0 * math.pi)
            rx, ry = math.cos(a), math.sin(a)
            if m == 0 and len(q) < 8:  # axis-aligned and diagonal cases
                rx, ry = [(1.0, 0.0), (0.0, 1.0), (-1.0, 0.0), (0.0, -1.0),
                          (D, D), (-D, D), (D, -D), (-D, -D)][len(q)]
            st = ref_backend.active().cast_ray(t.kind, t.door_index, flags, ox, oy, rx, ry)
            q.append((ox, oy, rx, ry))
            res.append(st)
        rays[f"m{m}_kind"] = t.kind
        rays[f"m{m}_didx"] = t.door_index
        rays[f"m{m}_dopen"] = flags
        rays[f"m{m}_q"] = np.array(q)
        rays[f"m{m}_i"] = np.array([[r[0], r[1], r[2], r[3], r[6]] for r in res], np.int32)
        rays[f"m{m}_f"] = np.array([[r[4], r[5]] for r in res])
    np.savez_compressed(HERE / "rays.npz", **rays)

    # random maps + frames with doors / sprites (test_backends.py:57-69 style)
    rng = random.Random(b"graft-frames")
    fr = {}
    for m in range(16):
        t = ref_conftest.random_tilemap(rng)
        floor = [(x, y) for y in range(t.height) for x in range(t.width)
                 if t.kind[y, x] == CellTag.FLOOR]
        fx, fy = rng.choice(floor)
        a = rng.uniform(0.0, 2.0 * math.pi)
        pose = Pose.looking(Vec2(fx + 0.37, fy + 0.61), Vec2(math.cos(a), math.sin(a)))
        flags = [rng.random() < 0.5 for _ in t.doors]
        w, h = [(64, 64), (128, 128), (40, 24), (37, 29)][m % 4]
        frame = render_frame(t, pose, w, h, door_open=flags)
        fr[f"f{m}_frame"] = frame
        fr[f"f{m}_pose"] = np.array([pose.position.x, pose.position.y,
                                     pose.direction.x, pose.direction.y])
        fr[f"f{m}_dopen"] = np.array(flags, dtype=np.uint8)
        fr[f"f{m}_map"] = _pack_map(t)
    np.savez_compressed(HERE / "frames_random.npz", **fr)

    syn = {}
    for s in range(20):
        t = ref_conftest.random_tilemap(random.Random(s))
        syn[f"s{s}"] = _pack_map(t)
    np.savez_compressed(HERE / "synthetic_maps.npz", **syn)

    digests = []
    for case in DIGEST_CASES:
        d = digest_case(*case)
        print(d)
        digests.append(d)
    (HERE / "digests.json").write_text(json.dumps(digests, indent=1) + "\n")


def _pack_map(t) -> np.ndarray:
    """kind, wall_color, then door / entity / spawn records, as one int64 blob:
    [h, w, kind..., wcol..., nd, (x, y, color, locked)*, ne, (kind, x, y, color)*,
     ns, (x, y)*]"""
    out = [t.height, t.width, *t.kind.ravel().tolist(), *t.wall_color.ravel().tolist()]
    out.append(len(t.doors))
    for d in t.doors:
        out += [d.tile[0], d.tile[1], int(d.color), int(d.locked)]
    out.append(len(t.entities))
    for e in t.entities:
        out += [int(e.kind), e.tile[0], e.tile[1], -1 if e.color is None else int(e.color)]
    out.append(len(t.spawn_candidates))
    for s in t.spawn_candidates:
        out += [s[0], s[1]]
    return np.array(out, dtype=np.int64)


def export_tables() -> None:
    from tilecast.suite import make_env, registered_ids
    out = {}
    fields = ("kind", "wcol", "didx", "eat", "dcol", "dlock", "ekind", "ecol", "epx", "epy",
              "spx", "spy", "goal_ent", "dirs", "pal", "door_rgb", "key_rgb", "goal_rgb",
              "med_box", "med_cross", "ceil_rgb", "floor_rgb", "coef", "fc", "ic", "legal")
    for env in registered_ids():
        t = make_env(env).tables
        for f in fields:
            out[f"{env}|{f}"] = getattr(t, f)
    np.savez_compressed(HERE / "tables.npz", **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["tables"]:
        export_tables()
    else:
        main()
        export_tables()
