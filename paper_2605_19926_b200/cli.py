"""``python -m paper_2605_19926_b200.cli bench`` -- the reference's bench
report (/root/reference/pkg/src/tilecast/cli.py:56-100; schema_version 1
fields unchanged) measured on the GPU, plus GPU fields.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time
from pathlib import Path

import torch

SCHEMA_VERSION = 1


def _host_fingerprint() -> dict:
    from . import BACKEND_NAME, __version__
    dev = torch.cuda.get_device_properties(torch.cuda.current_device())
    return {"platform": platform.platform(), "machine": platform.machine(),
            "python": platform.python_version(), "cpu_count": os.cpu_count(),
            "backend": BACKEND_NAME, "tilecast": __version__,
            "gpu": dev.name, "gpu_sms": dev.multi_processor_count}


def bench(env_id: str, n: int, steps: int, seed: int, width: int, height: int) -> dict:
    from . import batch_reset, make_env, policy_actions, registered_ids, rollout
    from .batch import batch_step_host, pipeline_drain
    if env_id not in registered_ids():
        raise SystemExit(f"error: unknown environment {env_id!r}; valid ids: "
                         f"{', '.join(registered_ids())}")
    spec = make_env(env_id, obs_width=width, obs_height=height)
    # steps/sec the reference way (throughput_probe semantics, batch.py:156-179):
    # pre-drawn actions, 3 warm-up steps, host actions in / numpy results out
    acts = policy_actions(spec, n, steps + 3, seed)
    bs = batch_reset(spec, n, seed)
    for s in range(3):
        bs, _, _ = batch_step_host(bs, acts[s], reuse=True)
    pipeline_drain()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s in range(steps):
        bs, _, _ = batch_step_host(bs, acts[3 + s], reuse=True)
    pipeline_drain()
    torch.cuda.synchronize()
    rate = n * steps / (time.perf_counter() - t0)
    # untimed rollout for the reward accounting (cli.py:76-81)
    bs = batch_reset(spec, n, seed)
    res = rollout(bs, steps, seed, record=True)
    # summed step by step in the reference's order (cli.py:76-81): one numpy
    # sum per step, accumulated in a Python float
    reward_sum = 0.0
    for row in res["rewards"].cpu().numpy():
        reward_sum += float(row.sum())
    # device-resident fused rollout rate, for reference
    rb = batch_reset(spec, n, seed)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rollout(rb, steps, seed)
    torch.cuda.synchronize()
    fused = n * steps / (time.perf_counter() - t0)
    return {
        "schema_version": SCHEMA_VERSION, "kind": "bench",
        "config": {"env": env_id, "n": n, "steps": steps, "seed": seed, "width": width,
                   "height": height, "threads": 1},
        "results": {"steps_per_second": rate, "frames_per_second": rate,
                    "us_per_frame": 1e6 / rate, "reward_sum": reward_sum,
                    "fused_rollout_steps_per_second": fused},
        "host": _host_fingerprint(),
    }


def main(argv=None) -> None:
    ap = argparse.ArgumentParser(prog="paper_2605_19926_b200.cli")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench", help="Measure batched steps/sec under a uniform-random policy.")
    b.add_argument("--env", dest="env_id", required=True)
    b.add_argument("--n", type=int, default=1)
    b.add_argument("--steps", type=int, default=1000)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--width", type=int, default=64)
    b.add_argument("--height", type=int, default=64)
    b.add_argument("--json", dest="json_path", default=None)
    a = ap.parse_args(argv)
    if a.n < 1 or a.steps < 1:
        ap.error("--n and --steps must be >= 1")
    report = bench(a.env_id, a.n, a.steps, a.seed, a.width, a.height)
    text = json.dumps(report, indent=2)
    print(text)
    if a.json_path:
        Path(a.json_path).write_text(text + "\n")


if __name__ == "__main__":
    main(sys.argv[1:])
