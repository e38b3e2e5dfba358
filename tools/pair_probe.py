"""Rollout time at C3 without the critic output, for comparing actor variants (POD_PAIR / POD_MULTICAST)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2111_05188_b200 import api, configs, synth  # noqa: E402

w = configs.preset("C3", T_data=20000)
m = synth.make_market(w.n_stocks, w.T_data, w.dt, w.seed, n_feat=w.n_feat)
cfg = api.config_from_workload(w)
env = api.Env(cfg, torch.from_numpy(m.close).cuda(), torch.from_numpy(m.feat).cuda())
aw = synth.make_actor(env.obs_dim, w.n_hidden, w.hidden, w.n_stocks, 1)
params = api.pack_actor_params(cfg, [aw], w.n_hidden, w.hidden)
actor = api.make_actor(w.n_hidden, w.hidden, params)
T = 128
tr = api.Trajectory.allocate(T, w.n_envs, w.n_stocks, env.k_pad)
env.reset(synth.tile_starts(env.n_tiles, w.T_data, min(w.horizon, w.T_data - 2), 1))
for _ in range(3):
    env.rollout(T, tr, actor=actor)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    env.rollout(T, tr, actor=actor)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 5 / T * 1e3
print(f"per step {us:.2f} us  ->  {w.n_envs / us * 1e6:.3e} env-steps/s")
