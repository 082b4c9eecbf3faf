"""Where the end-to-end batch_step time goes (host side)."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2605_19926_b200 as tc  # noqa: E402
from paper_2605_19926_b200 import batch as B  # noqa: E402

spec = tc.make_env("my-way-home")
n = 4096
acts = tc.policy_actions(spec, n, 300, 1)
bs = tc.batch_reset(spec, n, 1)
for s in range(5):
    bs, r, d = tc.batch_step(bs, acts[s], reuse=True, copy_outputs=False)
torch.cuda.synchronize()
K = 200
t0 = time.perf_counter()
for s in range(K):
    B._coerce_actions(bs, acts[s])
t1 = time.perf_counter()
print(f"_coerce_actions {1e6*(t1-t0)/K:.1f} us")
t0 = time.perf_counter()
for s in range(K):
    bs, r, d = tc.batch_step(bs, acts[s], reuse=True, copy_outputs=False)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"batch_step (async) {1e6*(t1-t0)/K:.1f} us/call; drain {1e6*(t2-t1):.0f} us")
t0 = time.perf_counter()
for s in range(K):
    bs, r, d = tc.batch_step(bs, acts[s], reuse=True, copy_outputs=False)
    tc.to_host(r, d)
t1 = time.perf_counter()
print(f"batch_step + to_host {1e6*(t1-t0)/K:.1f} us/step -> {n*K/(t1-t0)/1e6:.1f} M env-steps/s")
t0 = time.perf_counter()
for s in range(K):
    tc.to_host(r, d)
t1 = time.perf_counter()
print(f"to_host alone {1e6*(t1-t0)/K:.1f} us")
t0 = time.perf_counter()
for s in range(K):
    bs, rh, dh = tc.batch_step_host(bs, acts[s], reuse=True)
t1 = time.perf_counter()
print(f"batch_step_host {1e6*(t1-t0)/K:.1f} us/step -> {n*K/(t1-t0)/1e6:.1f} M env-steps/s")
from paper_2605_19926_b200 import _native as N
from paper_2605_19926_b200.engine import stream_ptr
stg = bs._stage
t0 = time.perf_counter()
for s in range(K):
    B._check_host_actions(bs, acts[s])
t1 = time.perf_counter()
print(f"_check_host_actions {1e6*(t1-t0)/K:.1f} us")
sb, ob = bs._retired
lib = N.lib()
args = (bs._ds.handle, N.C.byref(bs._sb.c_struct()), N.C.byref(sb.c_struct()), stg.h_act_ptr,
        stg.dev_ptr, N.C.byref(ob.c_struct()), bs.n, 1, 0, N.ptr(bs._counters), stg.h_rew_ptr,
        stg.h_done_ptr, stream_ptr(bs.device))
t0 = time.perf_counter()
for s in range(K):
    lib.tc_batch_step_host(*args)
t1 = time.perf_counter()
print(f"raw C call (H2D+kernel+D2H+sync) {1e6*(t1-t0)/K:.1f} us")
args2 = (bs._ds.handle, N.C.byref(bs._sb.c_struct()), N.C.byref(sb.c_struct()), stg.h_act_ptr,
         stg.dev_ptr, N.C.byref(ob.c_struct()), bs.n, 1, 0, N.ptr(bs._counters), None, None,
         stream_ptr(bs.device))
t0 = time.perf_counter()
for s in range(K):
    lib.tc_batch_step_host(*args2)
t1 = time.perf_counter()
print(f"raw C call without D2H {1e6*(t1-t0)/K:.1f} us")
args3 = (bs._ds.handle, N.C.byref(bs._sb.c_struct()), N.C.byref(sb.c_struct()), stg.h_act_ptr,
         N.C.byref(ob.c_struct()), bs.n, 1, 0, N.ptr(bs._counters), stg.h_rew_ptr,
         stg.h_flag_ptr, stream_ptr(bs.device))
t0 = time.perf_counter()
for s in range(K):
    lib.tc_batch_step_mapped(*args3)
t1 = time.perf_counter()
print(f"raw mapped C call (kernel reads actions / writes results over the bus + sync) "
      f"{1e6*(t1-t0)/K:.1f} us")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for s in range(K):
    lib.tc_batch_step_into(bs._ds.handle, N.C.byref(bs._sb.c_struct()), N.C.byref(sb.c_struct()),
                           stg.dev_ptr, N.C.byref(ob.c_struct()), bs.n, 1, 0, N.ptr(bs._counters),
                           stream_ptr(bs.device))
e1.record()
torch.cuda.synchronize()
print(f"kernel only (async launches) {1e3*e0.elapsed_time(e1)/K:.1f} us/step")
