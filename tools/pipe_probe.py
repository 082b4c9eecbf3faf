"""Per-call host time of the pipelined host step (batch_step_host, reuse=True)
and the pipeline counters: python tools/pipe_probe.py [env] [n] [steps]."""
import ctypes as C
import os
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
if env in ("c2", "c3", "c4", "c5", "large"):  # a bench config's spec
    import bench
    spec = bench.make_spec(env)
else:
    spec = tc.make_env(env)
acts = tc.policy_actions(spec, n, K + 5, 1)
for pipeline in (False, True):
    bs = tc.batch_reset(spec, n, 1)
    for s in range(5):
        bs, r, d = tc.batch_step_host(bs, acts[s], reuse=True, pipeline=pipeline)
    tc.pipeline_drain()
    torch.cuda.synchronize()
    N.pipe_reset()
    N.lib().tc_debug_mapped_timing(None, 1)
    s0 = N.pipe_stats()
    ts = np.zeros(K)
    t00 = time.perf_counter()
    for s in range(K):
        t0 = time.perf_counter()
        bs, r, d = tc.batch_step_host(bs, acts[5 + s], reuse=True, pipeline=pipeline)
        ts[s] = time.perf_counter() - t0
    el = time.perf_counter() - t00
    split = np.zeros(3)
    N.lib().tc_debug_mapped_timing(split.ctypes.data, 2)
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
    if pipeline and os.environ.get("TILECAST_PIPE_TRACE") == "1":
        g = C.c_int32()
        N.lib().tc_debug_pipe_trace(None, 0, C.byref(g))
        buf = np.zeros(64 * 3 * g.value, np.uint64)
        N.lib().tc_debug_pipe_trace(buf.ctypes.data, buf.size, C.byref(g))
        tr = buf.reshape(64, 3, g.value).astype(np.float64)
        for k in range(1, 12):
            a = tr[k]
            ok = a[0] > 0
            if not ok.any():
                break
            t0 = a[0][ok].min()
            prev_end = tr[k - 1][2][tr[k - 1][2] > 0].max() if k else 0
            print(f"  step {k}: gate spread {(a[0][ok].max() - t0) / 1e3:.2f} us, shipped "
                  f"min/max +{(a[1][ok].min() - t0) / 1e3:.2f}/+{(a[1][ok].max() - t0) / 1e3:.2f} us, "
                  f"frames min/med/max +{(a[2][ok].min() - t0) / 1e3:.2f}/"
                  f"+{(np.median(a[2][ok]) - t0) / 1e3:.2f}/+{(a[2][ok].max() - t0) / 1e3:.2f} us, "
                  f"gap after prev frames {(t0 - prev_end) / 1e3:.2f} us, "
                  f"period {(t0 - tr[k - 1][0][tr[k - 1][0] > 0].min()) / 1e3:.2f} us", flush=True)
    if pipeline:
        print(f"  released steps: release call {split[0]:.1f} us, wait for results {split[1]:.1f} us "
              f"({int(split[2])} steps); the rest is python", flush=True)
