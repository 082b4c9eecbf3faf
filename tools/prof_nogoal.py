"""my-way-home with the goal removed, saturation rollout, for ncu comparison."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2605_19926_b200 as tc  # noqa: E402
from paper_2605_19926_b200.maps import SHIPPED_MAPS  # noqa: E402

goal = len(sys.argv) > 1 and sys.argv[1] == "goal"
base = tc.make_env("my-way-home")
spec = base if goal else tc.EnvSpec(
    id="mwh-nogoal", map=tc.parse_map(SHIPPED_MAPS["my-way-home"].replace("G", ".")),
    action_set=base.action_set, goal_mode=base.goal_mode, max_steps=base.max_steps)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
bs = tc.batch_reset(spec, n, 0, device="cuda:0")
tc.rollout(bs, 2, 0)
tc.rollout(bs, 4, 0, step0=2)
torch.cuda.synchronize()
print("ok", spec.id, n)
