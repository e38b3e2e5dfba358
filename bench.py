#!/usr/bin/env python
"""Benchmark of the vectorised-rollout hot path (BASELINE.json metric:
"env-steps/sec (rollout incl. actor fwd) at 1/2/4/8 B200; GAE GB/s vs HBM peak").

One bench *step* = one pass of every SURVEY.md §8(a) row over one batch:
pod_rollout(T) (tcgen05 actor MLP + Gaussian sampling + env step + trajectory
writes, a CUDA graph of T x {actor, env-step}), pod_gae over the rollout's
[T, N] buffers, pod_env_fitness and pod_select_elite (NCCL fitness all-gather
+ elite slab moves).  Default workload: C3 (NASDAQ-100-shaped minute data,
8192 envs per GPU, actor 3x512, T = 256).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

Multi-GPU: launched by torchrun (one process per GPU, RANK/LOCAL_RANK/WORLD_SIZE
from the environment); envs and agents are sharded across ranks (weak
scaling), the only collectives are the per-step fitness all-gather / elite
moves.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# keep stdout to the one JSON line: NCCL's version banner must not reach it
os.environ["NCCL_DEBUG"] = os.environ.get("POD_BENCH_NCCL_DEBUG", "WARN")
# C-level prints (NCCL banners, driver messages) go to stderr; the JSON line goes to the real stdout
_JSON_FD = os.dup(1)
os.dup2(2, 1)


def emit(line: dict):
    os.write(_JSON_FD, (json.dumps(line) + "\n").encode())

METRIC = "env-steps/sec (rollout incl. actor fwd)"
UNIT = "env-steps/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="C3")
    p.add_argument("--T", type=int, default=None, help="override the rollout length")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--profile-stride", type=int, default=32,
                   help="bracket every k-th step's kernels with CUDA events (0 = off)")
    p.add_argument("--elite-k", type=int, default=None)
    p.add_argument("--tdata", type=int, default=None, help="truncate the market (profiling runs only)")
    p.add_argument("--agents", type=int, default=None, help="override agents per GPU (experiments)")
    p.add_argument("--envs", type=int, default=None, help="override envs per GPU (experiments)")
    return p.parse_args()


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region: the sampler is started (and its
    first line awaited) before the region, every line is stamped on arrival, and only the lines that arrive
    between mark_begin() and mark_end() (plus one sampling interval) are summarised."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    INTERVAL_MS = 50

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.t_begin = self.t_end = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.idx), "-lms", str(self.INTERVAL_MS)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
            t_wait = time.monotonic() + 5.0
            while not self.lines and time.monotonic() < t_wait and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def mark_begin(self):
        self.t_begin = time.monotonic()

    def mark_end(self):
        self.t_end = time.monotonic()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(2 * self.INTERVAL_MS / 1e3)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        lo = self.t_begin if self.t_begin is not None else float("-inf")
        hi = (self.t_end if self.t_end is not None else float("inf")) + self.INTERVAL_MS / 1e3
        sm, mx, reasons = [], [], set()
        names = ["active", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for t, ln in self.lines:
            if not lo <= t <= hi:
                continue
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names[1:], parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "interval_ms": self.INTERVAL_MS}


def actor_flops_per_env(obs_dim, n_hidden, hidden, n):
    """Algorithmic MLP FLOPs per env-step (unpadded dims): 2 sum d_in d_out."""
    macs = obs_dim * hidden + (n_hidden - 1) * hidden * hidden + hidden * n
    return 2 * macs


def env_bytes_per_env(n, f, obs_dim):
    """Algorithmic HBM bytes per env-step of the env-step kernel:
    a_t read 2n, holdings read+write 8n, cash/asset/disc read+write 48, reward 4,
    done 1, s_{t+1} write 2 obs_dim, plus the tile's market rows
    (p_t, p_{t+1}, p_0, feat: (3 + f) n x 4 B) shared by the 32 envs of a tile."""
    return 2 * n + 8 * n + 48 + 4 + 1 + 2 * obs_dim + (3 + f) * n * 4 / 32.0


def env_bytes_per_env_survey(n, f, obs_dim):
    """SURVEY.md §8(d)'s K2 byte model: a 2n + holdings r/w 8n + cash/asset r/w 32 + reward 4 + done 1 +
    s_{t+1} 2 obs_dim per env-step, plus (n + n f) 4 B per tile of 32 envs (2,089 B at n = 100)."""
    return 2 * n + 8 * n + 32 + 4 + 1 + 2 * obs_dim + (n + n * f) * 4 / 32.0


def gae_bytes_survey(T, N):
    """SURVEY.md §8(d)'s K3 byte model: 17 B per element (r, V, d read; A, R written) + 4 B per env."""
    return 17.0 * T * N + 4.0 * N


def gae_bytes(T, N):
    """r, V read 4+4, done 1, adv, ret written 4+4 per element; boot 4 per env; the per-buffer
    normalisation rereads and rewrites adv (+8 per element; R#23)."""
    return 25.0 * T * N + 4.0 * N


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_step_sample(w, market, weights_flat, n_envs, T, nthreads, starts, critic):
    """One bounded oracle pass of the hot path (rollout incl. actor and critic, GAE on the critic's
    values with V(s_T) as bootstrap, fitness, select)."""
    import numpy as np

    import oracle

    env = oracle.Env(market.close, market.feat, n_envs, horizon=w.horizon, h_max=w.h_max, C0=w.C0, cost=w.cost,
                     scale=w.reward_scale, gamma=w.gamma, seed=w.seed, env_offset=0, n_agents=1)
    env.reset(starts[:n_envs])
    t0 = time.perf_counter()
    out = env.rollout(T, "sample", weights=weights_flat[None, :], n_hidden=w.n_hidden, hidden=w.hidden,
                      nthreads=nthreads, want=("rew", "done", "val"), critic=critic[None, :])
    adv, _, _ = oracle.gae(out["rew"], out["val"][:T], out["done"], out["val"][T], w.gamma, w.lam)
    oracle.gae_normalize(adv)
    J = oracle.fitness(env.ep_ret, 1)
    oracle.select_elite(J, 1)
    return time.perf_counter() - t0


def c1_full_oracle(cores):
    """configs[0] (C1) run in full by the oracle on the host: 16 envs x T = 64 steps of the whole step
    (actor 2x128 + critic, env step, GAE, fitness, select), all cores and one thread."""
    import numpy as np

    import oracle
    from paper_2111_05188_b200 import configs, synth

    w1 = configs.preset("C1")
    m1 = synth.make_market(w1.n_stocks, w1.T_data, w1.dt, w1.seed, n_feat=w1.n_feat)
    aw = synth.make_actor(w1.obs_dim, w1.n_hidden, w1.hidden, w1.n_stocks, w1.seed * 1000)
    wf = oracle.actor_flat(aw.W, aw.b, aw.log_std)
    wcr = np.append(aw.w_v.astype(np.float64), aw.b_v)
    st = np.repeat(synth.tile_starts(1, w1.T_data, w1.horizon, w1.seed + 1), 32)
    out = {}
    for th in (cores, 1):
        tt = oracle_step_sample(w1, m1, wf, w1.n_envs, w1.T, th, st, wcr)
        out["all_cores" if th == cores else "one_thread"] = {"value": w1.n_envs * w1.T / tt, "unit": UNIT,
                                                              "cores": th, "seconds": tt}
    out["sample"] = "C1 in full: 16 envs x 64 steps (whole step incl. actor 2x128 + critic, GAE, fitness, select)"
    return out


def run_reference(args, w, rank, world):
    """--impl reference: the float64 oracle as it stands, on the host cores."""
    import numpy as np

    import oracle
    from paper_2111_05188_b200 import synth

    if rank != 0:
        return
    oracle.build()
    T_data = min(w.T_data, 200_000)
    market = synth.make_market(w.n_stocks, T_data, w.dt, w.seed, n_feat=w.n_feat)
    aw = synth.make_actor(w.obs_dim, w.n_hidden, w.hidden, w.n_stocks, w.seed * 1000)
    wf = oracle.actor_flat(aw.W, aw.b, aw.log_std)
    wcr = np.append(aw.w_v.astype(np.float64), aw.b_v)
    H = min(w.horizon, T_data - 2)
    starts = np.repeat(synth.tile_starts((4096 + 31) // 32, T_data, H, w.seed + 1), 32)
    cores = cpu_cores()
    # size one step to ~3 s of wall time: calibrate on one step of `cores` envs
    Ts = min(w.T, 8)
    t1 = oracle_step_sample(w, market, wf, cores, 1, cores, starts, wcr)
    per_env_step = t1 / cores * cores  # wall s per (env-step) x cores
    n_envs = int(max(cores, min(4096, (3.0 / max(per_env_step, 1e-9)) * cores / Ts)))
    n_envs = max(cores, n_envs // cores * cores)
    for _ in range(args.warmup):
        oracle_step_sample(w, market, wf, n_envs, Ts, cores, starts, wcr)
    times = [oracle_step_sample(w, market, wf, n_envs, Ts, cores, starts, wcr) for _ in range(args.steps)]
    tot = sum(times)
    value = n_envs * Ts * args.steps / tot
    sample = (f"{n_envs} envs x {Ts} steps of workload {w.name} per step (market truncated to {T_data} rows; "
              f"actor {w.n_hidden}x{w.hidden} + critic float64, "
              f"env step, GAE on the critic values + normalisation, fitness, select), {cores} OpenMP threads")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(w, T=Ts), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def workload_config(w, T=None, world=1):
    return {"workload": f"{w.name}: {w.description}", "n_stocks": w.n_stocks, "n_feat": w.n_feat,
            "T_data": w.T_data, "envs_per_gpu": w.n_envs, "T": T or w.T, "horizon": w.horizon,
            "actor": f"{w.n_hidden}x{w.hidden} MLP, bf16 tcgen05, fp32 accumulate", "agents_per_gpu": w.n_agents,
            "ledger": "float64", "parallelism": f"env-sharded x{world}",
            "l2": "inputs/outputs larger than L2 (trajectory writes per step >> 126 MB), no flush needed"}


def relaunch_distributed(n: int) -> int:
    """`--gpus N` without a torchrun environment: start N ranks of this same command under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1); rank 0 prints the line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, POD_BENCH_CHILD="1")
    # the JSON line of rank 0 goes to the real stdout; everything else to stderr
    r = subprocess.run(cmd, env=env, stdout=_JSON_FD, stderr=2)
    return r.returncode


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
                         f"(torchrun --nproc-per-node {args.gpus}) or drop --gpus")
    from paper_2111_05188_b200 import configs

    over = {}
    if args.T:
        over["T"] = args.T
    if args.tdata:
        over["T_data"] = args.tdata
    if args.agents:
        over["n_agents"] = args.agents
    if args.envs:
        over["n_envs"] = args.envs
    w = configs.preset(args.config, **over)
    if args.impl == "reference":
        run_reference(args, w, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2111_05188_b200 import _build, api, synth

    _build.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    api.load()
    peaks = load_peaks()

    # ---- inputs: market data (rank 0 generates, broadcast over NCCL), env shards, agents
    if rank == 0:
        market = synth.make_market(w.n_stocks, w.T_data, w.dt, w.seed, n_feat=w.n_feat)
        close = torch.from_numpy(market.close).to(dev)
        feat = torch.from_numpy(market.feat).to(dev)
    else:
        market = None
        close = torch.empty((w.T_data, w.n_stocks), dtype=torch.float32, device=dev)
        feat = torch.empty((w.T_data, w.n_feat, w.n_stocks), dtype=torch.float32, device=dev)
    if world > 1:
        dist.broadcast(close, 0)
        dist.broadcast(feat, 0)
    N, T, n = w.n_envs, w.T, w.n_stocks
    cfg = api.config_from_workload(w, env_offset=rank * N)
    env = api.Env(cfg, close, feat)
    n_tiles = env.n_tiles
    starts_all = synth.tile_starts(n_tiles * world, w.T_data, w.horizon, w.seed + 1)
    starts = starts_all[rank * n_tiles : (rank + 1) * n_tiles]
    P = w.n_agents
    agents = [synth.make_actor(env.obs_dim, w.n_hidden, w.hidden, n, w.seed * 1000 + rank * P + a) for a in range(P)]
    params = api.pack_actor_params(cfg, agents, w.n_hidden, w.hidden, device=dev)
    actor = api.make_actor(w.n_hidden, w.hidden, params)
    # the critic (head row n over the actor trunk, R#22) writes V(s_t) for t = 0..T during the rollout:
    # GAE consumes it on device, V(s_T) is the bootstrap
    traj = api.Trajectory.allocate(T, N, n, env.k_pad, device=dev, critic=True)
    val = traj.val[:T]
    boot = traj.val[T]
    adv = torch.empty_like(val)
    ret = torch.empty_like(val)
    adv_stats = torch.empty(2, dtype=torch.float64, device=dev)   # per-buffer advantage normalisation (R#23)
    fit = torch.empty(P, dtype=torch.float64, device=dev)
    comm = api.Comm(world, rank, P)
    k_elite = args.elite_k or max(1, (P * world) // 2)
    stream = torch.cuda.current_stream()
    env.reset(starts)
    env.profile(0)   # the headline is timed with no event nodes inside the rollout graph

    def step():
        env.rollout(T, traj, actor=actor)
        api.pod_gae(traj.rew, val, traj.done, boot, w.gamma, w.lam, adv, ret, normalize=True, stats=adv_stats)
        env.fitness(fit)
        comm.select_elite(fit, k_elite, params)

    for _ in range(args.warmup):
        step()
    # the rollout's own launches (one cached graph): 2T + 3 kernels as separate actor / env-step launches,
    # 3 with the fused rollout kernel (obs_0, the T steps, the step-counter bump)
    torch.cuda.synchronize()
    k0 = api.kernel_launches()
    env.rollout(T, traj, actor=actor)
    rollout_kernels = api.kernel_launches() - k0
    fused = rollout_kernels < T
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    launches0 = api.kernel_launches()
    clocks.mark_begin()
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    clocks.mark_end()
    gpu_launches = api.kernel_launches() - launches0   # every libpod kernel launched in the timed region
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ck = clocks.stop()
    ms = t0.elapsed_time(t1)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    env_steps = world * N * T * args.steps
    value = env_steps / (ms_max / 1e3)
    env.check()

    # ---- per-kernel durations: a separate pass of the same steps with CUDA events recorded inside the
    # rollout graph around the actor / env-step launches of every k-th step (on the stream each launch runs
    # on), and around the GAE launches; nothing of this pass enters `value`
    acc = {"actor_ms": 0.0, "actor_n": 0, "env_ms": 0.0, "env_n": 0, "gae_ms": 0.0, "gae_n": 0, "step_ms": 0.0,
           "roll_ms": 0.0, "roll_n": 0, "roll_step_ms": 0.0}
    if fused:
        # the fused rollout kernel as the headline runs it: CUDA events on the stream around each rollout
        # graph launch (obs_0 launch + the fused kernel + the counter bump: the bracket overstates the
        # fused kernel by those two small launches), the rest of the step outside the brackets
        rev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        q0 = torch.cuda.Event(enable_timing=True)
        q1 = torch.cuda.Event(enable_timing=True)
        q0.record(stream)
        for i in range(args.steps):
            rev[i][0].record(stream)
            env.rollout(T, traj, actor=actor)
            rev[i][1].record(stream)
            api.pod_gae(traj.rew, val, traj.done, boot, w.gamma, w.lam, adv, ret, normalize=True, stats=adv_stats)
            env.fitness(fit)
            comm.select_elite(fit, k_elite, params)
        q1.record(stream)
        torch.cuda.synchronize()
        acc["roll_step_ms"] = q0.elapsed_time(q1)
        for r0, r1 in rev:
            acc["roll_ms"] += r0.elapsed_time(r1)
            acc["roll_n"] += 1
    if args.profile_stride > 0:
        env.profile(args.profile_stride)
        gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        p0 = torch.cuda.Event(enable_timing=True)
        p1 = torch.cuda.Event(enable_timing=True)
        env.rollout(T, traj, actor=actor)   # capture the profiled graph outside the timed pass
        env.profile_read()
        p0.record(stream)
        for i in range(args.steps):
            env.rollout(T, traj, actor=actor)
            gev[i][0].record(stream)
            api.pod_gae(traj.rew, val, traj.done, boot, w.gamma, w.lam, adv, ret, normalize=True, stats=adv_stats)
            gev[i][1].record(stream)
            env.fitness(fit)
            comm.select_elite(fit, k_elite, params)
            am, an, em, en = env.profile_read()
            acc["actor_ms"] += am
            acc["actor_n"] += an
            acc["env_ms"] += em
            acc["env_n"] += en
        p1.record(stream)
        torch.cuda.synchronize()
        acc["step_ms"] = p0.elapsed_time(p1)
        for g0, g1 in gev:
            acc["gae_ms"] += g0.elapsed_time(g1)
            acc["gae_n"] += 1
        env.profile(0)

    # ---- end to end through the public API: pinned host inputs in, result out, every step
    e2e = None
    if not args.no_e2e:
        env.profile(0)
        h_params = params.cpu().pin_memory()
        h_fit = torch.empty(P, dtype=torch.float64).pin_memory()
        bi = h_params.numel() * h_params.element_size()
        bo = h_fit.numel() * 8

        def e2e_step():
            params.copy_(h_params, non_blocking=True)
            env.rollout(T, traj, actor=actor)
            api.pod_gae(traj.rew, val, traj.done, boot, w.gamma, w.lam, adv, ret, normalize=True, stats=adv_stats)
            env.fitness(fit)
            comm.select_elite(fit, k_elite, params)
            h_fit.copy_(fit, non_blocking=True)
            torch.cuda.current_stream().synchronize()

        for _ in range(2):
            e2e_step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e2e = {"value": env_steps / (float(ems.item()) / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(bi),
               "d2h_bytes_per_step": int(bo)}

    if rank == 0:
        # ---- per-kernel rooflines (algorithmic work per launch / live CUDA-event duration of the launch)
        # tensor peak: the burst figure when the run held its clocks with no power cap (the kernel's own
        # conditions), else the sustained one; both fractions are reported
        capped = "sw_power_cap" in (ck.get("reasons") or []) or (
            ck.get("sm_mhz") and ck.get("sm_max_mhz") and ck["sm_mhz"] < 0.95 * ck["sm_max_mhz"])
        tpeak = peaks["bf16_tflops_sustained"] if capped else peaks["bf16_tflops"]
        tpeak_kind = "sustained (power-capped clocks)" if capped else "burst (full clocks, no power cap)"
        pstep = acc["step_ms"] if acc["step_ms"] > 0 else ms
        kern = {}
        if acc["roll_n"]:
            r_ms = acc["roll_ms"] / acc["roll_n"]
            fpe = actor_flops_per_env(env.obs_dim, w.n_hidden, w.hidden, n)
            tf = N * T * fpe / (r_ms / 1e3) / 1e12
            ebytes = N * T * env_bytes_per_env(n, w.n_feat, env.obs_dim)
            kern["rollout_fused"] = {
                "bound": "tensor", "achieved": tf, "peak": tpeak, "peak_kind": tpeak_kind, "unit": "TFLOP/s",
                "frac": tf / tpeak, "frac_burst": tf / peaks["bf16_tflops"],
                "frac_sustained": tf / peaks["bf16_tflops_sustained"],
                "flop_per_env_step": fpe, "launch": f"T = {T} steps of actor + env step per launch",
                "avg_launch_us_full_n": r_ms * 1e3, "launch_units_timed": acc["roll_n"],
                "share_of_step": acc["roll_ms"] / acc["roll_step_ms"],
                "env_gbs_over_launch": ebytes / (r_ms / 1e3) / 1e9,
                "note": "one launch runs the T steps; achieved counts the actor MLP flops only, over the whole "
                        "launch (the env step's float64 ledger shares the SMs serially with it)"}

        if acc["actor_n"]:
            a_ms = acc["actor_ms"] / acc["actor_n"]
            flops = N * actor_flops_per_env(env.obs_dim, w.n_hidden, w.hidden, n)
            tf = flops / (a_ms / 1e3) / 1e12
            kern["actor_mlp"] = {"bound": "tensor", "achieved": tf, "peak": tpeak, "peak_kind": tpeak_kind,
                                 "unit": "TFLOP/s", "frac": tf / tpeak,
                                 "frac_burst": tf / peaks["bf16_tflops"],
                                 "frac_sustained": tf / peaks["bf16_tflops_sustained"],
                                 "flop_per_env_step": actor_flops_per_env(env.obs_dim, w.n_hidden, w.hidden, n),
                                 "avg_launch_us_full_n": a_ms * 1e3, "launch_units_timed": acc["actor_n"],
                                 "share_of_step": a_ms * T * args.steps / pstep,
                                 "path": "separate launches (profiling pass)" if fused else "headline"}
        if acc["env_n"]:
            e_ms = acc["env_ms"] / acc["env_n"]
            b_bench = env_bytes_per_env(n, w.n_feat, env.obs_dim)
            b_survey = env_bytes_per_env_survey(n, w.n_feat, env.obs_dim)
            gbs = N * b_bench / (e_ms / 1e3) / 1e9
            kern["env_step"] = {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                "frac": gbs / peaks["hbm_gbs"], "bytes_per_env_step": b_bench,
                                "bytes_per_env_step_survey": b_survey,
                                "frac_survey_bytes": N * b_survey / (e_ms / 1e3) / 1e9 / peaks["hbm_gbs"],
                                "avg_launch_us_full_n": e_ms * 1e3,
                                "launch_units_timed": acc["env_n"], "share_of_step": e_ms * T * args.steps / pstep,
                                "path": "separate launches (profiling pass)" if fused else "headline"}
        if acc["gae_n"]:
            g_ms = acc["gae_ms"] / acc["gae_n"]
            gbs = gae_bytes(T, N) / (g_ms / 1e3) / 1e9
            kern["gae"] = {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                           "frac": gbs / peaks["hbm_gbs"], "bytes_per_element": 25,
                           "bytes_per_element_survey": 17,
                           "frac_survey_bytes": gae_bytes_survey(T, N) / (g_ms / 1e3) / 1e9 / peaks["hbm_gbs"],
                           "avg_launch_us_full_n": g_ms * 1e3, "launch_units_timed": acc["gae_n"],
                           "share_of_step": acc["gae_ms"] / pstep}
        # the event-bracketed launches of the profiled pass run slower than in the plain graph (the record
        # nodes break the kernel-to-kernel launch path), so `achieved` keeps the bracketed (conservative)
        # duration; the rollout kernels' `share_of_step` is their bracketed proportion of the rollout's part
        # of the headline step (step minus GAE), `bracket_inflation` = bracketed (actor + env) time per step
        # over that part
        if "actor_mlp" in kern and "env_step" in kern:
            ra, re_ = kern["actor_mlp"], kern["env_step"]
            roll = max(0.0, 1.0 - kern["gae"]["share_of_step"]) if "gae" in kern else 1.0
            tot = ra["avg_launch_us_full_n"] + re_["avg_launch_us_full_n"]
            infl = (ra["share_of_step"] + re_["share_of_step"]) / roll if roll > 0 else None
            for k in (ra, re_):
                k["share_of_step"] = roll * k["avg_launch_us_full_n"] / tot
                k["bracket_inflation"] = infl
        # the dominant kernel of the headline step (with the fused rollout, the separate actor / env-step
        # launches of the profiling pass are not part of it)
        head = {k: v for k, v in kern.items() if not (fused and k in ("actor_mlp", "env_step"))}
        dom = max(head, key=lambda k: head[k]["share_of_step"]) if head else None
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if dom and os.path.exists(tpath):
            try:
                tj = json.load(open(tpath))
                traffic = tj.get(args.config, {}).get(dom)
            except Exception:
                traffic = None
        roofline = None
        if dom:
            k = kern[dom]
            roofline = {"kernel": dom, "bound": k["bound"], "achieved": k["achieved"], "peak": k["peak"],
                        "unit": k["unit"], "frac": k["frac"], "traffic": traffic, "peak_source": peaks["source"]}
            if "peak_kind" in k:
                roofline["peak_kind"] = k["peak_kind"]
                roofline["frac_burst"] = k["frac_burst"]
                roofline["frac_sustained"] = k["frac_sustained"]
        # ---- CPU baseline: the oracle as it stands, bounded sample, rank 0 at N=1 only
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            import oracle

            oracle.build()
            cores = cpu_cores()
            wf = oracle.actor_flat(agents[0].W, agents[0].b, agents[0].log_std)
            wcr = np.append(agents[0].w_v.astype(np.float64), agents[0].b_v)
            env_starts = np.repeat(starts, 32)[:N]
            t1s = oracle_step_sample(w, market, wf, cores, 1, cores, env_starts, wcr)
            # ~10 s of all-core work: all N envs if they fit, for as many steps (4..T) as fit
            per_env_step = t1s / cores   # wall seconds per env-step with `cores` threads
            n_s = int(min(N, max(cores, 10.0 / max(per_env_step, 1e-9) / 4)))
            n_s = max(cores, n_s // cores * cores)
            Ts = int(min(T, max(4, 10.0 / max(per_env_step * n_s, 1e-9))))
            tt = oracle_step_sample(w, market, wf, n_s, Ts, cores, env_starts, wcr)
            cpu = {"value": n_s * Ts / tt, "unit": UNIT, "cores": cores, "kind": "oracle",
                   "sample": f"{n_s} envs x {Ts} steps of {w.name} (float64 actor {w.n_hidden}x{w.hidden} + critic + "
                             f"env step + GAE on the critic values + normalisation + fitness + select), OpenMP over "
                             f"envs, {tt:.1f} s"}
            # the same oracle on one thread (a bounded sample of ~5 s)
            n_1 = int(min(N, max(1, 5.0 / max(t1s, 1e-9) / Ts)))   # one thread: t1s per env-step
            t_1 = oracle_step_sample(w, market, wf, n_1, Ts, 1, env_starts, wcr)
            cpu["single_thread"] = {"value": n_1 * Ts / t_1, "unit": UNIT, "cores": 1,
                                    "sample": f"{n_1} envs x {Ts} steps of {w.name}, 1 thread, {t_1:.1f} s"}
            # configs[0] (C1) in full: 16 envs x 64 steps, Dow-30 daily, actor 2x128 (the oracle-scale case)
            cpu["c1_full"] = c1_full_oracle(cores)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": workload_config(w, world=world), "roofline": roofline, "kernels": kern,
                "gae_gbs": kern.get("gae", {}).get("achieved"), "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": gpu_launches, "rollout_kernels": rollout_kernels, "clocks": ck,
                "precision": "actor bf16 x bf16 -> fp32 (tcgen05); sampling fp32; cash ledger float64; GAE fp32"}
        emit(line)
    comm.destroy()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
