"""Throughput vs batch size for the per-step kernel and the fused rollout."""
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
ns = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [148, 592, 1184, 2368, 4096, 8192, 16384, 65536]
spec = bench.make_spec(cfg)
dev = torch.device("cuda", 0)
for n in ns:
    bs = tc.batch_reset(spec, n, 0, device=dev)
    K = 20
    acts = torch.stack([tc.policy_actions_device(spec, s, n, 0, device=dev) for s in range(K + 3)])
    out = DeviceOut.alloc(n, spec.obs_height, spec.obs_width, dev)
    for s in range(3):
        launch_batch(bs._ds, bs._sb, acts[s], out, n, L.MODE_STEP, True, False, bs._counters)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(K):
        launch_batch(bs._ds, bs._sb, acts[3 + s], out, n, L.MODE_STEP, True, False, bs._counters)
    e1.record()
    torch.cuda.synchronize()
    step_us = e0.elapsed_time(e1) * 1e3 / K
    rb = tc.batch_reset(spec, n, 0, device=dev)
    tc.rollout(rb, 2, 0)
    torch.cuda.synchronize()
    e0.record()
    tc.rollout(rb, K, 0, step0=2)
    e1.record()
    torch.cuda.synchronize()
    roll_us = e0.elapsed_time(e1) * 1e3 / K
    print(f"{cfg} n={n:6d} step {step_us:8.1f} us ({n/step_us:7.1f} M/s)   rollout {roll_us:8.1f} us/step ({n/roll_us:7.1f} M/s)", flush=True)
    del bs, rb, out
