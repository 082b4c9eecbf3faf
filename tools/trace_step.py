"""Per-env phase timeline of one fused step (needs a TC_TRACE=1 build:
TILECAST_B200_LIB=paper_2605_19926_b200/variant_trace.so)."""
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
n = int(sys.argv[2]) if len(sys.argv) > 2 else bench.CONFIGS[cfg][2]
spec = bench.make_spec(cfg)
dev = torch.device("cuda", 0)
bs = tc.batch_reset(spec, n, 0, device=dev)
out = DeviceOut.alloc(n, spec.obs_height, spec.obs_width, dev)
tr = torch.zeros((n, 16), dtype=torch.int64, device=dev)
lib = N.lib()
lib.tc_debug_trace.argtypes = [C.c_void_p]
for s in range(4):
    a = tc.policy_actions_device(spec, s, n, 0, device=dev)
    if s == 3:
        torch.cuda.synchronize()
        N.check(lib.tc_debug_trace(tr.data_ptr()), "trace")
    launch_batch(bs._ds, bs._sb, a, out, n, L.MODE_STEP, True, False, bs._counters)
torch.cuda.synchronize()
t = tr.cpu().numpy().astype(np.int64)
t0 = t[:, 0].min()
rel = (t[:, :6] - t0) / 1000.0  # us
names = ["start", "loaded", "dyn", "walls", "sprites", "end"]
print(f"{cfg} n={n}: kernel span {rel[:, 5].max():.1f} us; first start {rel[:,0].min():.1f}, "
      f"last start {rel[:,0].max():.1f}")
for k in range(1, 6):
    d = rel[:, k] - rel[:, k - 1]
    print(f"  {names[k-1]:>8s}->{names[k]:<8s} mean {d.mean():7.2f} us  p50 {np.median(d):7.2f}  "
          f"p90 {np.percentile(d, 90):7.2f}  max {d.max():7.2f}")
tot = rel[:, 5] - rel[:, 0]
print(f"  env total mean {tot.mean():.2f} us p90 {np.percentile(tot, 90):.2f} max {tot.max():.2f}")
sm = t[:, 6] & 0xFFFF
cnt = np.bincount(sm)
print("  envs per SM: min", cnt[cnt > 0].min(), "max", cnt.max(), "SMs used", (cnt > 0).sum())
hist = np.histogram(rel[:, 0], bins=8)
print("  start-time histogram (us):", [f"{e:.0f}" for e in hist[1]], hist[0].tolist())
if (t[:, 8] > 0).all():
    rs = (t[:, 8] - t[:, 2]) / 1000.0
    mr = (t[:, 9] - t[:, 8]) / 1000.0
    cw = (t[:, 3] - t[:, 9]) / 1000.0
    for nm, d in (("dyn->raysetup", rs), ("march", mr), ("colwrite", cw)):
        print(f"  {nm:>17s}  mean {d.mean():7.2f} us  p50 {np.median(d):7.2f}  "
              f"p90 {np.percentile(d, 90):7.2f}  max {d.max():7.2f}")
hist = np.histogram(rel[:, 5], bins=8)
print("  end-time histogram (us):", [f"{e:.0f}" for e in hist[1]], hist[0].tolist())
info = t[:, 7]
m = info & 0xFF
px = info >> 8
print("  by sprites drawn (m): env total us mean / max, count")
for k in range(0, int(m.max()) + 1):
    sel = m == k
    if sel.any():
        print(f"    m={k}: {tot[sel].mean():6.2f} / {tot[sel].max():6.2f}  n={int(sel.sum())}"
              f"  sprite px mean {px[sel].mean():.0f}  compose+sprites mean "
              f"{(rel[sel, 5] - rel[sel, 4]).mean():.2f}  setup mean {(rel[sel, 4] - rel[sel, 3]).mean():.2f}")
slow = np.argsort(-tot)[:12]
print("  slowest envs: total, phases (load,dyn,walls,sprites,compose), m, px")
for i in slow:
    ph = np.diff(rel[i, :6])
    print(f"    env {i:5d}: {tot[i]:6.2f}  {np.round(ph, 2).tolist()}  m={int(m[i])} px={int(px[i])}")
