"""Does the sprite code's footprint matter? my-way-home with / without its goal."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2605_19926_b200 as tc  # noqa: E402
from paper_2605_19926_b200.maps import SHIPPED_MAPS  # noqa: E402

base = tc.make_env("my-way-home")
nog = tc.EnvSpec(id="mwh-nogoal", map=tc.parse_map(SHIPPED_MAPS["my-way-home"].replace("G", ".")),
                 action_set=base.action_set, goal_mode=base.goal_mode, max_steps=base.max_steps)
for spec in (base, nog, base, nog):
    for n in (4096, 65536):
        bs = tc.batch_reset(spec, n, 0, device="cuda:0")
        tc.rollout(bs, 2, 0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tc.rollout(bs, 10, 0, step0=2)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 10
        print(f"{spec.id:12s} n={n:6d} rollout {us:8.1f} us/step {n/us:7.1f} M/s", flush=True)
