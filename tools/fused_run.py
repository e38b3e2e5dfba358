"""Profiling driver: a few rollouts of a preset through the fused rollout kernel (ncu target)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2111_05188_b200 import api, configs, synth  # noqa: E402

w = configs.preset(sys.argv[1] if len(sys.argv) > 1 else "C3", T_data=20000)
T = int(sys.argv[2]) if len(sys.argv) > 2 else 32
m = synth.make_market(w.n_stocks, w.T_data, w.dt, w.seed, n_feat=w.n_feat)
cfg = api.config_from_workload(w)
env = api.Env(cfg, torch.from_numpy(m.close).cuda(), torch.from_numpy(m.feat).cuda())
aw = synth.make_actor(env.obs_dim, w.n_hidden, w.hidden, w.n_stocks, 1)
params = api.pack_actor_params(cfg, [aw] * w.n_agents, w.n_hidden, w.hidden)
actor = api.make_actor(w.n_hidden, w.hidden, params)
tr = api.Trajectory.allocate(T, w.n_envs, w.n_stocks, env.k_pad, critic=True)
env.reset(synth.tile_starts(env.n_tiles, w.T_data, min(w.horizon, w.T_data - 2), 1))
for _ in range(3):
    env.rollout(T, tr, actor=actor)
torch.cuda.synchronize()
env.check()
print("ok")
