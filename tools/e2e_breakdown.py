"""Where the ~48 us of one mapped host step (C2) goes: launch + sync floor,
kernel alone, kernel + sync, mapped call."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2605_19926_b200 as tc  # noqa: E402
from paper_2605_19926_b200 import _native as N  # noqa: E402
from paper_2605_19926_b200.engine import stream_ptr  # noqa: E402

spec = tc.make_env("my-way-home")
n, K = 4096, 300
acts = tc.policy_actions(spec, n, K + 5, 1)
bs = tc.batch_reset(spec, n, 1)
for s in range(3):
    bs, r, d = tc.batch_step_host(bs, acts[s], reuse=True)
torch.cuda.synchronize()
stg = bs._stage
key = next(iter(stg.calls))
margs = stg.calls[key][0]
_, sb, sb2, ob = stg.calls[key]
lib = N.lib()
x = torch.zeros(1, device="cuda")


def wall(fn, k=K):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    return 1e6 * (time.perf_counter() - t0) / k


print(f"tiny torch op + synchronize      {wall(lambda: (x.add_(1), torch.cuda.synchronize())):6.1f} us")
dev_act = stg.dev[0]
dev_act.copy_(torch.from_numpy(acts[3]))
into = (bs._ds.handle, N.C.byref(sb.c_struct()), N.C.byref(sb2.c_struct()), dev_act.data_ptr(),
        N.C.byref(ob.c_struct()), n, 1, 0, N.ptr(bs._counters), stream_ptr(bs.device))
print(f"step_into + synchronize          {wall(lambda: (lib.tc_batch_step_into(*into), torch.cuda.synchronize())):6.1f} us")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
tot = 0.0
for _ in range(50):
    e0.record()
    lib.tc_batch_step_into(*into)
    e1.record()
    torch.cuda.synchronize()
    tot += e0.elapsed_time(e1)
print(f"step_into kernel, isolated (evt) {1e3 * tot / 50:6.1f} us")
print(f"mapped call                      {wall(lambda: lib.tc_batch_step_mapped(*margs)):6.1f} us")
tot = 0.0
for _ in range(50):
    e0.record()
    lib.tc_batch_step_mapped(*margs)
    e1.record()
    torch.cuda.synchronize()
    tot += e0.elapsed_time(e1)
print(f"mapped call, event span          {1e3 * tot / 50:6.1f} us")
