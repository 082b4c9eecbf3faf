"""Host-side cost of batch_step_host with the native call stubbed out."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_19926_b200 as tc  # noqa: E402

spec = tc.make_env("my-way-home")
n, K = 4096, 300
acts = tc.policy_actions(spec, n, K + 5, 1)
bs = tc.batch_reset(spec, n, 1)
for s in range(3):
    bs, r, d = tc.batch_step_host(bs, acts[s], reuse=True)
torch.cuda.synchronize()
stg = bs._stage
real = stg.fn
stg.fn = lambda *a: 0
t0 = time.perf_counter()
for s in range(K):
    bs, r, d = tc.batch_step_host(bs, acts[s], reuse=True)
t1 = time.perf_counter()
print(f"batch_step_host python-only {1e6*(t1-t0)/K:.1f} us")
x = np.empty(n, np.int64)
t0 = time.perf_counter()
for s in range(K):
    stg.h_act[:] = acts[s]
t1 = time.perf_counter()
print(f"copy actions {1e6*(t1-t0)/K:.2f} us")
t0 = time.perf_counter()
for s in range(K):
    torch.cuda.current_device()
t1 = time.perf_counter()
print(f"current_device {1e6*(t1-t0)/K:.2f} us")
t0 = time.perf_counter()
for s in range(K):
    stg.h_rew.copy(); stg.h_done.copy()
t1 = time.perf_counter()
print(f"result copies {1e6*(t1-t0)/K:.2f} us")
t0 = time.perf_counter()
for s in range(K):
    float(r.sum())
t1 = time.perf_counter()
print(f"reward sum {1e6*(t1-t0)/K:.2f} us")
# the native pipelined call alone, with pipelining off (one launch per call)
key = next(iter(stg.calls))
cs = stg.calls[key][1]
cs.speculate = 0
stg.fn = real
tc.pipeline_drain()
t0 = time.perf_counter()
for s in range(K):
    real(stg.calls[key][0])
t1 = time.perf_counter()
print(f"native step call (not pipelined) {1e6*(t1-t0)/K:.1f} us")
