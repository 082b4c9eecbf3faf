"""Small workload exercising every kernel path, for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run):

    compute-sanitizer --tool memcheck python tools/sanitize_case.py

Paths: batch_kernel with debug taps (G=16 / G=32, staged-band and direct
compose, sprites, doors, odd frame shapes), the lean kernel one wave (one
env per warp) and multi-wave (two envs per warp, env tickets), the u8
large-map march, the mapped host step, the fused rollout, the one-launch
heterogeneous step, reset / scalar paths."""
import random
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2605_19926_b200 as tc  # noqa: E402
from paper_2605_19926_b200.synthetic import large_tilemap, random_tilemap  # noqa: E402

cases = [tc.make_env("key-door", max_steps=20), tc.make_env("health-gathering", max_steps=20),
         tc.make_env("dmlab-random-goal-03", obs_width=128, obs_height=128, max_steps=15),
         tc.make_env("key-corridor", obs_width=37, obs_height=29, max_steps=15)]
tmap = random_tilemap(random.Random(7))
cases.append(tc.EnvSpec(id="syn", map=tmap, action_set=tc.suite.STRAFE_ACTIONS,
                        goal_mode=tc.GoalMode.RANDOM_PER_EPISODE, max_steps=12,
                        health_decay=1.0, health_restore=5.0))
big = large_tilemap(random.Random(13), 160, 128, n_doors=4, n_entities=16, n_spawns=16,
                    doors_at_spawns=True)
cases.append(tc.EnvSpec(id="big", map=big, action_set=tc.suite.STRAFE_ACTIONS,
                        goal_mode=tc.GoalMode.RANDOM_PER_EPISODE, max_steps=12,
                        health_decay=1.0, health_restore=5.0))
for spec in cases:
    for debug in (True, False):
        n = 96
        acts = tc.policy_actions(spec, n, 12, 1)
        bs = tc.batch_reset(spec, n, 1, debug=debug)
        for s in range(12):
            bs, r, d = tc.batch_step(bs, acts[s], reuse=True)
        bs, r, d = tc.batch_step_host(bs, acts[0], reuse=True)
        tc.rollout(bs, 4, 1)
        bs.check()
# multi-wave lean kernel (two envs per warp, tickets) and its mapped host path
spec = tc.make_env("my-way-home", max_steps=9)
n = 6000
acts = tc.policy_actions(spec, n, 3, 2)
bs = tc.batch_reset(spec, n, 2)
for s in range(3):
    bs, r, d = tc.batch_step(bs, acts[s], reuse=True)
bs, r, d = tc.batch_step_host(bs, acts[0], reuse=True)
bs.check()
# one-launch heterogeneous step
specs = [cases[0], cases[4], tc.make_env("my-way-home", max_steps=11)]
mb = tc.multi_reset(specs, [70, 50, 90], 3)
import numpy as np  # noqa: E402
for s in range(4):
    mb, r, d = tc.multi_step(mb, np.concatenate([tc.policy_actions(sp, c, 1, s)[0] for sp, c in
                                                 zip(specs, [70, 50, 90])]), reuse=True)
mb.check()
torch.cuda.synchronize()
print("sanitize case ok")
