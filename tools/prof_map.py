"""Short fixed workload for ncu on one synthetic map of bench_multimap.py:
reset + a few fused steps over a ring of output blocks larger than L2.

    python tools/prof_map.py MAP_INDEX [envs] [steps]

(used to compare sprite-heavy and sprite-free random maps)
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_19926_b200 as tc  # noqa: E402
from bench_multimap import spec_for  # noqa: E402
from paper_2605_19926_b200 import layout as L  # noqa: E402
from paper_2605_19926_b200.engine import DeviceOut, launch_batch  # noqa: E402

k = int(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
spec = spec_for(k)
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
print("ok map", k, n, steps, "ring", ring)
