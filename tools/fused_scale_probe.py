"""Diagnostics: the fused rollout's time per step at C3 shapes as the number of clusters (envs / 128) varies —
a per-cluster-latency-bound kernel keeps its step time; contention in the shared weight stream would not."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2111_05188_b200 import api, configs, synth  # noqa: E402

for N in [int(x) for x in (sys.argv[1:] or ["8192", "4096", "2048", "1024", "512"])]:
    w = configs.preset("C3", T_data=20000, n_envs=N)
    m = synth.make_market(w.n_stocks, w.T_data, w.dt, w.seed, n_feat=w.n_feat)
    cfg = api.config_from_workload(w)
    env = api.Env(cfg, torch.from_numpy(m.close).cuda(), torch.from_numpy(m.feat).cuda())
    aw = synth.make_actor(env.obs_dim, w.n_hidden, w.hidden, w.n_stocks, 1)
    params = api.pack_actor_params(cfg, [aw], w.n_hidden, w.hidden)
    actor = api.make_actor(w.n_hidden, w.hidden, params)
    T = 128
    tr = api.Trajectory.allocate(T, N, w.n_stocks, env.k_pad)
    env.reset(synth.tile_starts(env.n_tiles, w.T_data, min(w.horizon, w.T_data - 2), 1))
    for _ in range(3):
        env.rollout(T, tr, actor=actor)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        env.rollout(T, tr, actor=actor)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"N={N} clusters={N // 128}: {ms * 1e3 / T:.2f} us/step", flush=True)
    env.close_handle()
