"""The N>1 path through the CUDA kernel: two ranks (processes) on one GPU,
gloo for the plumbing (NCCL cannot put two ranks on one device), each rank
stepping its contiguous shard of a global batch with global env indices.
The gathered per-rank digests and state must equal one process stepping
the whole batch -- the reference's thread-count independence check
(pkg/tests/test_acceptance.py:243-277) with ranks in place of threads.

The ranks' kernels are independent launches (no rank waits on another's
kernel); the only collectives are gloo CPU reductions / gathers.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT  # noqa: F401  (sys.path setup)

pytestmark = pytest.mark.gpu

ENV, N_TOTAL, STEPS, SEED = "key-door", 1000, 40, 13


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(base: int, n: int, n_total: int, device):
    """Step envs [base, base + n) of the global batch on the device; returns
    the host state, final frames and per-step digests of rewards / dones."""
    import hashlib
    import torch
    import paper_2605_19926_b200 as tc
    spec = tc.make_env(ENV, max_steps=17)
    bs = tc.batch_reset(spec, n, SEED, device=device, base=base, n_total=n_total)
    acts = torch.empty(n, dtype=torch.int64, device=device)
    h = hashlib.blake2b(digest_size=16)
    rsum, dones = 0.0, 0
    for s in range(STEPS):
        tc.policy_actions_device(spec, s, n, SEED, base=base, n_total=n_total, out=acts)
        bs, r, d = tc.batch_step(bs, acts, reuse=True)
        rh, dh = r.cpu().numpy(), d.cpu().numpy()
        h.update(rh.tobytes())
        h.update(dh.tobytes())
        rsum += float(rh.sum())
        dones += int(dh.sum())
    bs.check()
    return bs.host_state(), bs.frames.cpu().numpy(), h.hexdigest(), rsum, dones


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_19926_b200.shard import reduce_episode_stats, shard_range
    sh = shard_range(N_TOTAL, world, rank)
    state, frames, digest, rsum, dones = _run(sh.base, sh.n, sh.n_total, "cuda:0")
    tot = reduce_episode_stats({"reward_sum": rsum, "episodes_done": dones,
                                "env_steps": sh.n * STEPS})
    digests = [None] * world
    dist.all_gather_object(digests, digest)
    q.put((rank, sh.base, sh.n, state, frames, tot, digests))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_one_gpu_equal_single_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    full_state, full_frames, _, rsum, dones = _run(0, N_TOTAL, N_TOTAL, "cuda:0")
    gathered = {k: np.concatenate([r[3][k] for r in res]) for k in full_state}
    for k, v in full_state.items():
        assert np.array_equal(gathered[k], v), k
    assert np.array_equal(np.concatenate([r[4] for r in res]), full_frames)
    for rank, base, n, state, frames, tot, digests in res:
        assert tot["env_steps"] == N_TOTAL * STEPS
        assert tot["episodes_done"] == dones
        assert abs(tot["reward_sum"] - rsum) < 1e-9
        assert digests == res[0][6]  # every rank gathered the same digests


def test_bench_two_ranks_one_gpu(tmp_path):
    """bench.py's torchrun path (process group, barriers, max-over-ranks
    timing, the stats reduction) with 2 ranks on one GPU over gloo: one JSON
    line from rank 0 with n_gpus = 2 and the whole-job value."""
    import json
    import subprocess
    import sys
    env = dict(os.environ, TILECAST_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(ROOT / "bench.py"), "--gpus", "2", "--steps", "5", "--warmup", "3",
           "--no-cpu-baseline", "--e2e-steps", "3"]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["config"]["envs_total"] == 2 * j["config"]["envs_per_gpu"]
    assert j["value"] > 0 and j["e2e"]["value"] > 0
    assert j["e2e"]["episode_stats"]["env_steps"] == 2 * j["config"]["envs_per_gpu"] * 3
