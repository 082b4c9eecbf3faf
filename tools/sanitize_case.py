"""Small workload exercising every kernel path, for compute-sanitizer."""
import random
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2605_19926_b200 as tc  # noqa: E402
from paper_2605_19926_b200.synthetic import random_tilemap  # noqa: E402

cases = [tc.make_env("key-door", max_steps=20), tc.make_env("health-gathering", max_steps=20),
         tc.make_env("dmlab-random-goal-03", obs_width=128, obs_height=128, max_steps=15),
         tc.make_env("key-corridor", obs_width=37, obs_height=29, max_steps=15)]
tmap = random_tilemap(random.Random(7))
cases.append(tc.EnvSpec(id="syn", map=tmap, action_set=tc.suite.STRAFE_ACTIONS,
                        goal_mode=tc.GoalMode.RANDOM_PER_EPISODE, max_steps=12,
                        health_decay=1.0, health_restore=5.0))
for spec in cases:
    n = 96
    acts = tc.policy_actions(spec, n, 30, 1)
    bs = tc.batch_reset(spec, n, 1, debug=True)
    for s in range(30):
        bs, r, d = tc.batch_step(bs, acts[s], reuse=True)
    bs, r, d = tc.batch_step_host(bs, acts[0], reuse=True)
    tc.rollout(bs, 10, 1)
    bs.check()
torch.cuda.synchronize()
print("sanitize case ok")
