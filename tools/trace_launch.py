"""Per-launch timeline of K back-to-back step launches (needs a TC_TRACE=1
build): CTA entry, map staged, past griddepcontrol.wait, CTA exit, per
launch, relative to the first CTA entry of launch 0 (globaltimer, us).

    TILECAST_B200_LIB=paper_2605_19926_b200/variant_trace.so python tools/trace_launch.py [c2] [K]
"""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_19926_b200 as tc  # noqa: E402
from paper_2605_19926_b200 import _native as N  # noqa: E402
from paper_2605_19926_b200 import layout as L  # noqa: E402
from paper_2605_19926_b200.engine import DeviceOut, launch_batch  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 6
n = bench.CONFIGS[cfg][2]
spec = bench.make_spec(cfg)
dev = torch.device("cuda", 0)
bs = tc.batch_reset(spec, n, 0, device=dev)
outs = [DeviceOut.alloc(n, spec.obs_height, spec.obs_width, dev) for _ in range(K + 3)]
acts = [tc.policy_actions_device(spec, s, n, 0, device=dev) for s in range(K + 3)]
lib = N.lib()
lib.tc_debug_trace_cta.argtypes = [C.c_void_p]
buf = torch.zeros((K + 3, 16384, 4), dtype=torch.int64, device=dev)
for s in range(3):
    launch_batch(bs._ds, bs._sb, acts[s], outs[s], n, L.MODE_STEP, True, False, bs._counters)
torch.cuda.synchronize()
# the K launches are captured into a CUDA graph like bench.py's timed region
# (a Python launch loop would be CPU-bound and hide the device-side gaps)
graph = torch.cuda.CUDAGraph()
cap = torch.cuda.Stream(dev)
cap.wait_stream(torch.cuda.current_stream(dev))
chained = len(sys.argv) > 3 and sys.argv[3] == "chained"
if chained:
    bsc = [tc.batch_steps(bs, torch.stack(acts[:3]), outs=outs[:3])]
    torch.cuda.synchronize()
with torch.cuda.stream(cap):
    with torch.cuda.graph(graph, stream=cap):
        if chained:
            bsc[0] = tc.batch_steps(bsc[0], torch.stack(acts[3:3 + K]), outs=outs[3:3 + K])
        else:
            for s in range(K):
                launch_batch(bs._ds, bs._sb, acts[3 + s], outs[3 + s], n, L.MODE_STEP, True,
                             False, bs._counters)
torch.cuda.synchronize()
N.check(lib.tc_debug_trace_cta(buf.data_ptr()), "trace_cta")
torch.cuda.synchronize()
graph.replay()
torch.cuda.synchronize()
t = buf.cpu().numpy()[:K].astype(np.int64)
used = (t[:, :, 3] > 0).all(axis=0)   # CTAs that ran an env in every launch
grid = int(used.sum())
t = t[:, used, :]
t0 = t[0, :, 0].min()
r = (t - t0) / 1000.0
print(f"{cfg} n={n} grid={grid} K={K} (us from the first CTA entry of launch 0)")
print("launch  entry[first,last]   staged[p50,last]   waited[first,last]   exit[p50,last]  "
      "span  gap(prev last exit -> first waited)")
prev_exit = None
for k in range(K):
    e, st, w, x = r[k, :, 0], r[k, :, 1], r[k, :, 2], r[k, :, 3]
    gap = "" if prev_exit is None else f"{w.min() - prev_exit:6.2f}"
    print(f"{k:5d}  [{e.min():7.2f},{e.max():7.2f}]  [{np.median(st):7.2f},{st.max():7.2f}]  "
          f"[{w.min():7.2f},{w.max():7.2f}]  [{np.median(x):7.2f},{x.max():7.2f}]  "
          f"{x.max() - w.min():6.2f}  {gap}")
    prev_exit = x.max()
print(f"mean launch period {(r[K - 1, :, 3].max() - r[0, :, 3].max()) / (K - 1):.2f} us")
