"""Short fixed workload for ncu: reset + a few fused steps of a bench config,
rotating over a ring of output blocks larger than L2 (like bench.py) so the
profiled launch's frame writes reach DRAM.

    python tools/prof_step.py [c2|c3|c4|c5] [steps]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_19926_b200 as tc  # noqa: E402
from paper_2605_19926_b200 import layout as L  # noqa: E402
from paper_2605_19926_b200.engine import DeviceOut, launch_batch  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
spec = bench.make_spec(cfg)
n = bench.CONFIGS[cfg][2]
dev = torch.device("cuda", 0)
bs = tc.batch_reset(spec, n, 0, device=dev)
fb = n * spec.obs_height * spec.obs_width * 3
ring = max(2, -(-2 * bench.L2_BYTES // fb))
outs = [DeviceOut.alloc(n, spec.obs_height, spec.obs_width, dev) for _ in range(ring)]
for s in range(steps):
    a = tc.policy_actions_device(spec, s, n, 0, device=dev)
    launch_batch(bs._ds, bs._sb, a, outs[s % ring], n, L.MODE_STEP, True, False, bs._counters)
torch.cuda.synchronize()
bs.check()
print("ok", cfg, n, steps, "ring", ring)
