"""The N>1 path on CPU (gloo, world size 2): envs sharded by global index,
per-rank trajectories identical to the single-process batch, and the
episode-statistics all-reduce. The oracle is the stepping engine here (CPU
test); the GPU path uses the same Shard / base / n_total plumbing."""

from __future__ import annotations

import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT  # noqa: F401  (sys.path setup)

ENV, N_TOTAL, STEPS, SEED = "key-door", 48, 30, 5


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_shard(base: int, n: int, n_total: int):
    import paper_2605_19926_b200 as tc
    from paper_2605_19926_b200 import rng
    from oracle import oracle as orc
    spec = tc.make_env(ENV, max_steps=12)
    t = spec.tables
    state = orc.alloc_state(n, t.n_doors, t.n_entities)
    out = orc.alloc_out(n, t.obs_height, t.obs_width)
    orc.seed_streams(SEED, base, n, state)
    orc.batch_kernel(t, state, None, out, 0, n_threads=1)
    tags = np.array([int(a) for a in spec.action_set], np.int64)
    rsum, dones = 0.0, 0
    for s in range(STEPS):
        acts = orc.policy_actions(rng.policy_key(SEED), s, n_total, base, n, tags)
        orc.batch_kernel(t, state, acts, out, 1, auto_reset=True, n_threads=1)
        rsum += float(out["rewards"].sum())
        dones += int(out["dones"].sum())
    return state, out["frames"].copy(), rsum, dones


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_19926_b200.shard import reduce_episode_stats, shard_range
    sh = shard_range(N_TOTAL, world, rank)
    state, frames, rsum, dones = _run_shard(sh.base, sh.n, sh.n_total)
    tot = reduce_episode_stats({"reward_sum": rsum, "episodes_done": dones,
                                "env_steps": sh.n * STEPS})
    q.put((rank, sh.base, sh.n, {k: v.copy() for k, v in state.items()}, frames, tot))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_equal_single_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full_state, full_frames, rsum, dones = _run_shard(0, N_TOTAL, N_TOTAL)
    for rank, base, n, state, frames, tot in res:
        for k, v in state.items():
            assert np.array_equal(v, full_state[k][base:base + n]), (rank, k)
        assert np.array_equal(frames, full_frames[base:base + n])
        assert tot["env_steps"] == N_TOTAL * STEPS
        assert tot["episodes_done"] == dones
        assert abs(tot["reward_sum"] - rsum) < 1e-9
