"""Stress the mapped host step's result ordering: every step, the rewards /
dones batch_step_host returned (read from pinned host memory once the
completion word is up) must equal the device copies the same kernel wrote.
Runs the lean one-wave (c2), the batch one-wave (large map) and the
multi-wave (c3) mapped paths."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_19926_b200 as tc  # noqa: E402

sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def run(name, spec, n, steps):
    acts = tc.policy_actions(spec, n, steps, 7)
    bs = tc.batch_reset(spec, n, 3)
    bad = 0
    nd = 0
    for s in range(steps):
        bs, r, d = tc.batch_step_host(bs, acts[s])
        rd = bs._ob.rewards.cpu().numpy()
        dd = bs._ob.dones.cpu().numpy().astype(bool)
        nd += int(d.sum())
        if not (np.array_equal(r, rd) and np.array_equal(d, dd)):
            bad += 1
    print(f"{name}: n={n} steps={steps} dones={nd} mismatched steps={bad}", flush=True)
    return bad


bad = run("c2 lean one-wave", tc.make_env("my-way-home"), 4096, 3000)
bad += run("c3 multi-wave", tc.make_env("key-door"), 16384, 1000)
bad += run("large batch one-wave", bench.large_spec(), 4096, 1000)
sys.exit(1 if bad else 0)
