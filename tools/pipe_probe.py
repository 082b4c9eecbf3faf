"""Per-call host time of the pipelined host step (batch_step_host, reuse=True)
and the pipeline counters: python tools/pipe_probe.py [env] [n] [steps]."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_19926_b200 as tc  # noqa: E402
from paper_2605_19926_b200 import _native as N  # noqa: E402

env = sys.argv[1] if len(sys.argv) > 1 else "my-way-home"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
K = int(sys.argv[3]) if len(sys.argv) > 3 else 300
spec = tc.make_env(env)
acts = tc.policy_actions(spec, n, K + 5, 1)
for pipeline in (False, True):
    bs = tc.batch_reset(spec, n, 1)
    for s in range(5):
        bs, r, d = tc.batch_step_host(bs, acts[s], reuse=True, pipeline=pipeline)
    tc.pipeline_drain()
    torch.cuda.synchronize()
    N.pipe_reset()
    s0 = N.pipe_stats()
    ts = np.zeros(K)
    t00 = time.perf_counter()
    for s in range(K):
        t0 = time.perf_counter()
        bs, r, d = tc.batch_step_host(bs, acts[5 + s], reuse=True, pipeline=pipeline)
        ts[s] = time.perf_counter() - t0
    el = time.perf_counter() - t00
    tc.pipeline_drain()
    torch.cuda.synchronize()
    s1 = N.pipe_stats()
    us = ts * 1e6
    print(f"{env} n={n} pipeline={pipeline}: {1e6 * el / K:.1f} us/step "
          f"({n * K / el / 1e6:.1f} M env-steps/s); call p10/p50/p90/max "
          f"{np.percentile(us, 10):.1f}/{np.median(us):.1f}/{np.percentile(us, 90):.1f}/{us.max():.1f} us; "
          f"released {s1['released'] - s0['released']} cancelled {s1['cancelled'] - s0['cancelled']} "
          f"timeouts {s1['timeouts'] - s0['timeouts']}", flush=True)
    print("  first 12 calls (us):", np.round(us[:12], 1).tolist(), flush=True)
