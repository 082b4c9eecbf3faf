"""Timed-region cost vs K (steps per region) for the chained step graph, as
bench.py times it: t(K) = K * per_step + fixed. Separates the fixed cost of a
region (graph start, first unchained launch, last launch's tail) from the
steady-state step period.

    python tools/sweep_k.py [c2] [1,2,5,10,20,50,200]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_19926_b200 as tc  # noqa: E402
from paper_2605_19926_b200.engine import DeviceOut  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
ks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 5, 10, 20, 50, 200]
spec = bench.make_spec(cfg)
dev = torch.device("cuda", 0)
n = bench.CONFIGS[cfg][2] if bench.CONFIGS[cfg][0] != "synthetic" else 1 << 20
H, W = spec.obs_height, spec.obs_width
ring = max(2, -(-2 * bench.L2_BYTES // (n * H * W * 3)))
outs = [DeviceOut.alloc(n, H, W, dev) for _ in range(ring)]
W0 = 5
kmax = max(ks)
acts = torch.empty((W0 + kmax, n), dtype=torch.int64, device=dev)
for s in range(W0 + kmax):
    tc.policy_actions_device(spec, s, n, 0, out=acts[s])
stream = torch.cuda.current_stream(dev)
mode = sys.argv[3] if len(sys.argv) > 3 else "graph"
res = []
for K in ks:
    row = []
    for rep in range(3):
        bs = [tc.batch_reset(spec, n, 0, device=dev)]
        bs[0] = tc.batch_steps(bs[0], acts[:W0], outs=outs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if mode == "graph":
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(dev)
            cap.wait_stream(stream)
            with torch.cuda.stream(cap):
                with torch.cuda.graph(g, stream=cap):
                    bs[0] = tc.batch_steps(bs[0], acts[W0:W0 + K], outs=outs)
            torch.cuda.synchronize()
            bench.clock_warm(stream)
            e0.record(stream)
            g.replay()
            e1.record(stream)
            del g
        else:
            # the K chained launches enqueued directly on the stream while the
            # device spin runs (their host launch cost is hidden behind it)
            bench.clock_warm(stream, ms=4.0)
            e0.record(stream)
            bs[0] = tc.batch_steps(bs[0], acts[W0:W0 + K], outs=outs)
            e1.record(stream)
        torch.cuda.synchronize()
        row.append(e0.elapsed_time(e1) * 1e3)
    t = float(np.median(row))
    res.append((K, t))
    print(f"{cfg} {mode} K={K:4d} region {t:9.1f} us  {t / K:7.2f} us/step  {n * K / t:7.1f} M/s",
          flush=True)
k_arr = np.array([r[0] for r in res], float)
t_arr = np.array([r[1] for r in res], float)
slope, icpt = np.polyfit(k_arr, t_arr, 1)
print(f"{cfg} fit: per_step {slope:.2f} us, fixed {icpt:.1f} us per region")
