"""One env per SM (latency view) for ncu: rollout of K steps, n envs."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_19926_b200 as tc  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 148
k = int(sys.argv[3]) if len(sys.argv) > 3 else 50
spec = bench.make_spec(cfg)
bs = tc.batch_reset(spec, n, 0, device="cuda:0")
tc.rollout(bs, 2, 0)
tc.rollout(bs, k, 0, step0=2)
torch.cuda.synchronize()
bs.check()
print("ok", cfg, n, k)
