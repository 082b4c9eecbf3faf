"""Host-side split of the non-pipelined mapped host step (batch_step_host
with pipeline=False) at C2: Python around the call, the launch call, the
wait for the kernel's completion word. tools/pipe_probe.py covers the
pipelined step."""
import ctypes as C
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_19926_b200 as tc  # noqa: E402
from paper_2605_19926_b200 import _native as N  # noqa: E402

spec = tc.make_env("my-way-home")
n, K = 4096, 400
acts = tc.policy_actions(spec, n, K + 5, 1)
bs = tc.batch_reset(spec, n, 1)
for s in range(5):
    bs, r, d = tc.batch_step_host(bs, acts[s], reuse=True, pipeline=False)
torch.cuda.synchronize()
lib = N.lib()
lib.tc_debug_mapped_timing.argtypes = [C.c_void_p, C.c_int32]
out = np.zeros(3)
lib.tc_debug_mapped_timing(out.ctypes.data, 1)
t0 = time.perf_counter()
for s in range(K):
    bs, r, d = tc.batch_step_host(bs, acts[5 + s], reuse=True, pipeline=False)
torch.cuda.synchronize()
el = (time.perf_counter() - t0) / K * 1e6
lib.tc_debug_mapped_timing(out.ctypes.data, 1)
print(f"per step {el:.1f} us: launch call {out[0]:.1f} us, wait for results {out[1]:.1f} us, "
      f"rest (python, ctypes) {el - out[0] - out[1]:.1f} us  ({n / el:.1f} M env-steps/s)")
