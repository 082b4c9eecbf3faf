"""Heterogeneous-map throughput (multimap.py) beside the homogeneous batch.

    python tools/bench_multimap.py [--maps 16] [--envs 131072] [--steps 50]

Synthetic random tile maps (conftest.random_tilemap semantics, 64x64 obs):
the same N envs as one homogeneous batch (map 0), as one homogeneous
batch on each map in turn (weighted by the group sizes: the maps' own
cost), and split over --maps different maps (one step launch per map group per step, one output
block). Actions pre-staged on the device; CUDA events on the launching
stream; frames (N x 12 KB) exceed L2. Prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import random
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_19926_b200 as tc  # noqa: E402
from paper_2605_19926_b200.synthetic import random_tilemap  # noqa: E402


def spec_for(k: int):
    return tc.EnvSpec(id=f"syn-mm{k}", map=random_tilemap(random.Random(5000 + k)),
                      action_set=tc.suite.STRAFE_ACTIONS,
                      goal_mode=tc.GoalMode.RANDOM_PER_EPISODE, max_steps=200,
                      living_reward=0.01, health_decay=1.0, health_restore=10.0)


def timed(step, steps: int, warmup: int) -> float:
    for s in range(warmup):
        step(s)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for s in range(steps):
        step(warmup + s)
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--maps", type=int, default=16)
    ap.add_argument("--envs", type=int, default=131072)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    n, m = args.envs, args.maps
    specs = [spec_for(k) for k in range(m)]
    counts = [n // m + (1 if k < n % m else 0) for k in range(m)]
    acts = torch.from_numpy(tc.policy_actions(specs[0], n, args.steps + args.warmup, 0)).to(dev)

    homo = [tc.batch_reset(specs[0], n, 0, device=dev)]

    def step_homo(s):
        homo[0], _, _ = tc.batch_step(homo[0], acts[s], reuse=True, copy_outputs=False)

    mm = [tc.multi_reset(specs, counts, 0, device=dev)]

    def step_multi(s):
        mm[0], _, _ = tc.multi_step(mm[0], acts[s], reuse=True)

    torch.cuda._sleep(int(2e-3 * 1.965e9))  # SM clock up before timing
    ms_h = timed(step_homo, args.steps, args.warmup)
    ms_m = timed(step_multi, args.steps, args.warmup)
    homo[0].check()
    # the same N envs homogeneously on each map in turn: the cost of the maps
    # themselves (random maps differ in size and ray length), without the split
    ms_each = []
    for k in range(m):
        one = [tc.batch_reset(specs[k], n, 0, device=dev)]

        def step_one(s, one=one):
            one[0], _, _ = tc.batch_step(one[0], acts[s], reuse=True, copy_outputs=False)

        ms_each.append(timed(step_one, max(10, args.steps // 4), args.warmup))
        one[0].check()
    ms_mix = sum(ms_each[k] * counts[k] / n for k in range(m))
    mm[0].check()
    print(json.dumps({
        "metric": "env steps/sec (rendered frames/sec)", "unit": "env-steps/s",
        "envs": n, "maps": m, "obs": [64, 64], "steps": args.steps, "warmup": args.warmup,
        "homogeneous": {"value": n / (ms_h * 1e-3), "ms_per_step": ms_h},
        "heterogeneous": {"value": n / (ms_m * 1e-3), "ms_per_step": ms_m,
                          "launches_per_step": (1 if os.environ.get("TILECAST_MULTI_LAUNCH", "1")
                                                != "0" and m <= 16 else m)},
        "homogeneous_per_map_weighted": {"value": n / (ms_mix * 1e-3), "ms_per_step": ms_mix,
                                         "per_map_ms": ms_each},
        "ratio": ms_h / ms_m, "ratio_vs_per_map": ms_mix / ms_m}))


if __name__ == "__main__":
    main()
