"""Benchmark: env steps/sec (rendered frames/sec) of the fused B200 step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4|c5]
                    [--impl ours|reference]

One "step" = one launch of the fused step kernel over the whole per-GPU batch
(dynamics + auto-reset + ray cast + sprites + frame write), actions drawn by
the seeded uniform policy (batch.policy_actions) and staged in HBM before the
timed region, like the reference's throughput_probe pre-draws them
(/root/reference/pkg/src/tilecast/batch.py:156-179).

Default workload (BASELINE.json configs[1]): my-way-home, 4096 envs per GPU,
64x64 RGB, auto-reset on. Frames rotate over a ring of output blocks larger
than the 126 MB L2 so every step's frame bytes go to HBM.

Prints ONE JSON line (rank 0). Multi-GPU: launched by torchrun, one process
per GPU, envs sharded by global index (weak scaling), no collective on the hot
path; elapsed time is the max over ranks (NCCL all-reduce of one scalar).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (env, overrides, envs per GPU, description)
    "c2": ("my-way-home", {}, 4096, "my-way-home, 4096 envs/GPU, 64x64 RGB, auto-reset"),
    "c3": ("key-door", {}, 16384, "key-door, 16384 envs/GPU, 64x64 RGB, sprites/doors"),
    "c4": ("dmlab-static-03", {"obs_width": 128, "obs_height": 128}, 8192,
           "dmlab-static-03, 8192 envs/GPU, 128x128 RGB"),
    "c5": ("synthetic", {}, 1 << 20,
           "synthetic random 6-14 tile map, 64x64 RGB, 2^20 envs split over the GPUs"),
    # the large-map variant of SURVEY §8(d): 20,480 cells, beyond the 4,096
    # staged as u32 codes -- u8 stop codes staged per CTA by one TMA bulk copy
    "large": ("large", {}, 4096,
              "synthetic large map 160x128 tiles (20,480 cells, TMA-staged u8 stop codes), "
              "4096 envs/GPU, 64x64 RGB"),
}
METRIC = "env steps/sec (rendered frames/sec) at 4096+ envs/GPU on 1/2/4/8 B200"
L2_BYTES = 126 * 2**20


def synthetic_spec(obs=(64, 64)):
    import random
    import paper_2605_19926_b200 as tc
    from paper_2605_19926_b200.synthetic import random_tilemap
    tmap = random_tilemap(random.Random(20260518))
    return tc.EnvSpec(id="synthetic-c5", map=tmap, action_set=tc.suite.STRAFE_ACTIONS,
                      goal_mode=tc.GoalMode.RANDOM_PER_EPISODE, max_steps=500,
                      obs_width=obs[0], obs_height=obs[1], living_reward=0.01,
                      health_decay=0.25, health_restore=10.0)


def clock_warm(stream, ms: float = 2.0) -> None:
    """A short device spin (torch.cuda._sleep: one busy thread, no env work)
    on `stream`, so the SM clock is at its under-load value when the timed
    region starts."""
    import torch
    with torch.cuda.stream(stream):
        torch.cuda._sleep(int(ms * 1e-3 * 1.965e9))


def physical_cores() -> int:
    """Physical cores of this host (the CPU reference runs
    one OpenMP thread per physical core)."""
    try:
        import psutil
        n = psutil.cpu_count(logical=False)
        if n:
            return int(n)
    except Exception:
        pass
    return os.cpu_count() or 1


def totals(cfg: str, world: int) -> tuple[int, str]:
    """(envs in the whole job, scaling): c2-c4 fix the envs per GPU (weak
    scaling); c5 splits 2^20 envs over the GPUs at every N (strong)."""
    if CONFIGS[cfg][0] == "synthetic":
        return 1 << 20, "strong"
    return CONFIGS[cfg][2] * world, "weak"


def config_dict(cfg: str, spec, n: int, n_total: int, world: int) -> dict:
    """The `config` object both arms print (identical keys and values)."""
    return {"workload": CONFIGS[cfg][3], "env": spec.id, "envs_per_gpu": n,
            "envs_total": n_total, "obs": [spec.obs_width, spec.obs_height],
            "auto_reset": True, "parallelism": f"env-shard x{world}"}


def source_sha16() -> str:
    import hashlib
    src = ROOT / "paper_2605_19926_b200" / "csrc" / "tilecast_b200.cu"
    return hashlib.sha256(src.read_bytes()).hexdigest()[:16]


def large_spec():
    """The 160x128-tile map of tests/golden (large-160x128, make_golden_r2.py)."""
    import random
    import paper_2605_19926_b200 as tc
    from paper_2605_19926_b200.synthetic import large_tilemap
    tmap = large_tilemap(random.Random(13), 160, 128, n_doors=4, n_entities=16, n_spawns=16,
                         doors_at_spawns=True)
    return tc.EnvSpec(id="large-160x128", map=tmap, action_set=tc.suite.STRAFE_ACTIONS,
                      goal_mode=tc.GoalMode.RANDOM_PER_EPISODE, max_steps=500,
                      living_reward=0.01, health_decay=0.25, health_restore=10.0)


def make_spec(cfg):
    import paper_2605_19926_b200 as tc
    env, ov, n, _ = CONFIGS[cfg]
    if env == "synthetic":
        return synthetic_spec()
    if env == "large":
        return large_spec()
    return tc.make_env(env, **ov)


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def measure_write_peak(dev) -> float | None:
    """Write-only HBM bandwidth on this GPU: an int64 fill_ (vectorised
    stores; a uint8 fill_ / memset reaches only ~3.9 TB/s) of a 2 GiB buffer
    (16x L2), best of 5, CUDA events on the current stream."""
    import torch
    try:
        buf = torch.empty(2 * 2**30 // 8, dtype=torch.int64, device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = None
        for k in range(6):
            torch.cuda.synchronize(dev)
            e0.record()
            buf.fill_(k + 1)
            e1.record()
            torch.cuda.synchronize(dev)
            if k:
                ms = e0.elapsed_time(e1)
                best = ms if best is None else min(best, ms)
        del buf
        return buf_bytes_gbs(2 * 2**30, best)
    except Exception:
        return None


def buf_bytes_gbs(nbytes: int, ms: float) -> float:
    return nbytes / (ms / 1e3) / 1e9


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.25)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(cfg, budget_s=12.0):
    """The reference's own CPU kernel (oracle/_ref, Cython+OpenMP) -- or the
    oracle port when _ref is absent -- on this host's cores, over a bounded
    sample of the workload (same spec, same env count, a few steps)."""
    import paper_2605_19926_b200 as tc
    spec = make_spec(cfg)
    n = CONFIGS[cfg][2] if CONFIGS[cfg][0] != "synthetic" else 131072
    cores = physical_cores()
    ref_dir = ROOT / "oracle" / "_ref"
    kind = "port"
    if (ref_dir / "tilecast" / "backend").exists() and CONFIGS[cfg][0] not in ("synthetic", "large"):
        try:
            sys.path.insert(0, str(ref_dir))
            import tilecast as ref
            from tilecast import backend as rb
            from tilecast.batch import batch_reset, batch_step
            rb.set_backend("compiled")
            os.environ["TILECAST_NUM_THREADS"] = str(cores)
            kind = "reference"
        except Exception:
            kind = "port"
        finally:
            if str(ref_dir) in sys.path:
                sys.path.remove(str(ref_dir))
    max_steps = 6000
    acts_all = tc.policy_actions(spec, n, max_steps + 1, 0)
    if kind == "reference":
        rspec = ref.make_env(*([CONFIGS[cfg][0]]), **CONFIGS[cfg][1])
        bs = batch_reset(rspec, n, 0, n_threads=cores)
        bs, _, _ = batch_step(bs, acts_all[0], n_threads=cores, reuse=True)
        steps, t0 = 0, time.perf_counter()
        while steps < max_steps and (steps < 3 or time.perf_counter() - t0 < budget_s):
            bs, _, _ = batch_step(bs, acts_all[1 + steps], n_threads=cores, reuse=True)
            steps += 1
        el = time.perf_counter() - t0
    else:
        from oracle import oracle as orc
        r = orc.Rollout(spec, n, 0, n_threads=cores)
        r.step(acts_all[0])
        steps, t0 = 0, time.perf_counter()
        while steps < max_steps and (steps < 3 or time.perf_counter() - t0 < budget_s):
            r.step(acts_all[1 + steps])
            steps += 1
        el = time.perf_counter() - t0
    return {"value": n * steps / el, "unit": "env-steps/s", "cores": cores, "kind": kind,
            "sample": f"{CONFIGS[cfg][3]}: {n} envs x {steps} batch_step calls "
                      f"({el:.1f} s wall, host threads={cores} = physical cores)"}


def run_reference(args, rank, world):
    """--impl reference: the reference CPU implementation on this host."""
    if rank != 0:
        return
    cfg = args.config
    import paper_2605_19926_b200 as tc
    spec = make_spec(cfg)
    n_total, scaling = totals(cfg, world)
    n = n_total // world if scaling == "strong" else CONFIGS[cfg][2]
    # the host steps the whole job's envs (a bounded 131072-env sample of the
    # 2^20-env c5 job: its rate is flat in N once N >> threads)
    n_run = min(n_total, 131072) if CONFIGS[cfg][0] == "synthetic" else n_total
    cores = physical_cores()
    ref_dir = ROOT / "oracle" / "_ref"
    acts = tc.policy_actions(spec, n_run, args.warmup + args.steps, 0)
    kind = "port"
    stepper = None
    if (ref_dir / "tilecast" / "backend").exists() and CONFIGS[cfg][0] not in ("synthetic", "large"):
        sys.path.insert(0, str(ref_dir))
        try:
            import tilecast as ref
            from tilecast import backend as rb
            from tilecast.batch import batch_reset, batch_step
            rb.set_backend("compiled")
            bs = [batch_reset(ref.make_env(CONFIGS[cfg][0], **CONFIGS[cfg][1]), n_run, 0,
                              n_threads=cores)]

            def stepper(a):
                bs[0], _, _ = batch_step(bs[0], a, n_threads=cores, reuse=True)
            kind = "reference"
        except Exception:
            stepper = None
    if stepper is None:
        from oracle import oracle as orc
        r = orc.Rollout(spec, n_run, 0, n_threads=cores)
        stepper = r.step
    for s in range(args.warmup):
        stepper(acts[s])
    t0 = time.perf_counter()
    for s in range(args.steps):
        stepper(acts[args.warmup + s])
    el = time.perf_counter() - t0
    v = n_run * args.steps / el
    line = {
        "metric": METRIC, "value": v, "unit": "env-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded uniform-random policy actions)", "impl": "reference",
        "config": config_dict(cfg, spec, n, n_total, world),
        "cpu_baseline": {"value": v, "unit": "env-steps/s", "cores": cores, "kind": kind,
                         "sample": f"{n_run} envs x {args.steps} timed batch_step calls on "
                                   f"{cores} host threads (one per physical core)"},
        "e2e": {"value": v, "unit": "env-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=50)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2605_19926_b200 as tc
    from paper_2605_19926_b200 import layout as L
    from paper_2605_19926_b200 import _native as N
    from paper_2605_19926_b200.engine import DeviceOut, launch_batch

    # one process per GPU; TILECAST_DIST_BACKEND=gloo lets a test run several
    # ranks on fewer GPUs (independent kernels, reductions on CPU tensors)
    backend = os.environ.get("TILECAST_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    rdev = dev if backend == "nccl" else torch.device("cpu")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    from paper_2605_19926_b200.shard import reduce_episode_stats, shard_range

    spec = make_spec(args.config)
    # c2-c4: fixed envs per GPU (weak scaling); c5: 2^20 envs in total split
    # over the GPUs at every N (strong scaling, 1 -> 8 on the same job)
    n_total, scaling = totals(args.config, world)
    sh = shard_range(n_total, world, rank)
    n, base = sh.n, sh.base
    H, W = spec.obs_height, spec.obs_width
    frame_bytes = n * H * W * 3
    ring = max(2, -(-2 * L2_BYTES // frame_bytes))  # >= 2x L2 of frame blocks

    seed = 0
    bs = tc.batch_reset(spec, n, seed, device=dev, base=base, n_total=n_total)
    total = args.warmup + args.steps
    acts = torch.empty((total, n), dtype=torch.int64, device=dev)
    for s in range(total):
        tc.policy_actions_device(spec, s, n, seed, base=base, n_total=n_total, out=acts[s])
    outs = [DeviceOut.alloc(n, H, W, dev) for _ in range(ring)]
    stream = torch.cuda.current_stream(dev)

    def step(s):
        launch_batch(bs._ds, bs._sb, acts[s], outs[s % ring], n, L.MODE_STEP, True, False,
                     bs._counters)

    # value: K steps through tc.batch_steps -- K launches of the step kernel,
    # each writing its own output block of the ring, chained per CTA (a
    # step's CTAs start as the previous step's CTAs free their slots; each
    # env waits only for its own state) -- captured once into a CUDA graph
    # (launch-bound at 4096 envs otherwise); replaying it runs exactly K steps
    bsc = [tc.batch_reset(spec, n, seed, device=dev, base=base, n_total=n_total)]
    bsc[0] = tc.batch_steps(bsc[0], acts[:args.warmup], outs=outs)
    for s in range(args.warmup):
        step(s)
    torch.cuda.synchronize(dev)
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream(dev)
    cap.wait_stream(stream)
    with torch.cuda.stream(cap):
        with torch.cuda.graph(graph, stream=cap):
            bsc[0] = tc.batch_steps(bsc[0], acts[args.warmup:args.warmup + args.steps], outs=outs)
    # the same K steps as K unchained launches (each waits for the whole
    # previous grid), reported beside it
    graph_u = torch.cuda.CUDAGraph()
    with torch.cuda.stream(cap):
        with torch.cuda.graph(graph_u, stream=cap):
            for k in range(args.steps):
                step(args.warmup + k)
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    with clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        # ~2 ms of device spin right before the timed region (no env work):
        # the sampler's start-up and the barrier leave the GPU idle long
        # enough for the SM clock to drop, and a 0.4 ms timed region would
        # otherwise run partly on the ramp
        clock_warm(stream)
        t_start.record(stream)
        graph.replay()
        t_end.record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        u0, u1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clock_warm(stream)
        u0.record(stream)
        graph_u.replay()
        u1.record(stream)
        torch.cuda.synchronize(dev)
    elapsed_ms = t_start.elapsed_time(t_end)
    unchained_ms = u0.elapsed_time(u1)
    if world > 1:
        t = torch.tensor([unchained_ms], dtype=torch.float64, device=rdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        unchained_ms = float(t.item())
    kern_ms = [elapsed_ms / args.steps]  # per-launch average over the graph replay
    if world > 1:
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device=rdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    bs.check()
    bsc[0].check()
    value = n_total * args.steps / (elapsed_ms / 1e3)

    # fused multi-step launch (tc_rollout: K steps, in-kernel policy) for context
    rb = tc.batch_reset(spec, n, seed, device=dev, base=base, n_total=n_total)
    rring = torch.empty((ring, n, H, W, 3), dtype=torch.uint8, device=dev)
    tc.rollout(rb, args.warmup, seed, frames=rring)
    torch.cuda.synchronize(dev)
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clock_warm(stream)
    r0.record(stream)
    tc.rollout(rb, args.steps, seed, step0=args.warmup, frames=rring)
    r1.record(stream)
    torch.cuda.synchronize(dev)
    rollout_ms = r0.elapsed_time(r1)
    if world > 1:
        t = torch.tensor([rollout_ms], dtype=torch.float64, device=rdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        rollout_ms = float(t.item())
    rollout_value = n_total * args.steps / (rollout_ms / 1e3)
    del rring

    # end-to-end through the public API: host actions (pinned H2D inside
    # batch_step) and a D2H read of each step's rewards + dones
    host_acts = tc.policy_actions(spec, n_total, args.e2e_steps + 3, seed + 1)[:, base:base + n]
    eb = tc.batch_reset(spec, n, seed + 1, device=dev, base=base, n_total=n_total)
    for s in range(3):
        eb, rh, dh = tc.batch_step_host(eb, host_acts[s], reuse=True)
    tc.pipeline_drain()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    rews = []  # each step's host rewards (summed after the timed region)
    clock_warm(torch.cuda.current_stream(dev))
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for s in range(args.e2e_steps):
        eb, rh, dh = tc.batch_step_host(eb, host_acts[3 + s], reuse=True)
        rews.append(rh)
    # the loop is over: cancel the step launched ahead of actions that will
    # not come (pipelined host step), then wait for the device
    tc.pipeline_drain()
    torch.cuda.synchronize(dev)
    e2e_s = time.perf_counter() - t0
    rsum = float(np.sum(rews))
    stats = reduce_episode_stats({"reward_sum": rsum, "env_steps": n * args.e2e_steps},
                                 device=rdev)  # the optional NCCL stats reduction
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=rdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = n_total * args.e2e_steps / e2e_s
    eb.check()

    peak, peak_src = load_peaks()
    write_peak = measure_write_peak(dev)
    mean_kernel_ms = float(np.mean(kern_ms))
    achieved = frame_bytes / (mean_kernel_ms / 1e3) / 1e9
    # DRAM bytes per launch from an ncu capture of THIS kernel source and
    # config (profiles/ncu_traffic.json, written by tools/ncu_traffic.py from
    # 8 consecutive ring-rotated launches with --cache-control none); null
    # when the capture was of another build
    traffic, traffic_src = None, "no capture of this build"
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():
        try:
            rec = json.loads(prof.read_text()).get(args.config)
            if rec and rec.get("source_sha16") == source_sha16() and rec.get("envs") == n:
                traffic = rec["dram_bytes_per_launch"]
                traffic_src = rec["capture"]
        except Exception:
            traffic = None

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "env-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded uniform-random policy actions; "
                    + ("generated random map" if args.config in ("c5", "large") else "shipped map")
                    + ")",
            "config": config_dict(args.config, spec, n, n_total, world),
            "l2_policy": f"frame ring of {ring} output blocks "
                         f"({ring * frame_bytes / 2**20:.0f} MiB > 2x L2)",
            "e2e": {"value": e2e_value, "unit": "env-steps/s",
                    "h2d_bytes_per_step": n * 8, "d2h_bytes_per_step": n * 9,
                    "api": "batch_step_host(numpy actions, reuse=True) -> numpy rewards,"
                           " dones per step: actions copied into pinned host memory and"
                           " read by the step kernel over the bus (H2D), rewards + dones"
                           " written back to pinned host memory by the kernel (D2H),"
                           " stream sync, numpy copies out",
                    "episode_stats": stats},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "kernel": N.lib().tc_step_kernel(bs._ds.handle, n).decode()
                                   + "; avg launch = graph replay / K",
                         "algorithmic_bytes_per_launch": frame_bytes,
                         "mean_kernel_ms": mean_kernel_ms, "peak_source": peak_src,
                         # the kernel only writes frames: its own ceiling is the
                         # write-only stream, measured here (2 GiB int64 fill_,
                         # best of 5; ~7.4 TB/s on B200, above the copy figure)
                         "write_peak_gbs": write_peak,
                         "frac_of_write_peak": achieved / write_peak if write_peak else None},
            "api": "tc.batch_steps (K step launches chained per CTA, tc_batch_steps)",
            "unchained": {"value": n_total * args.steps / (unchained_ms / 1e3),
                          "unit": "env-steps/s", "ms_per_step": unchained_ms / args.steps,
                          "api": "K tc_batch_kernel launches, each after the whole previous "
                                 "grid (griddepcontrol.wait)"},
            "rollout_fused": {"value": rollout_value, "unit": "env-steps/s",
                              "launches": 1, "steps_per_launch": args.steps},
            "gpu_launches": args.steps,
            "clocks": clocks.summary(),
        }
        if not args.no_cpu_baseline and world == 1:
            try:
                line["cpu_baseline"] = cpu_baseline(args.config)
            except Exception as exc:  # keep the bench line even if the host leg fails
                line["cpu_baseline"] = {"value": None, "error": repr(exc)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
