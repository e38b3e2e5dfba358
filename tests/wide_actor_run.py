"""Subprocess helper for test_wide_actor_matches_column_split: one deterministic-noise rollout step at a
shape the opt-in wide actor (POD_WIDE=1) accepts; writes mu, V and logp of step 0 to argv[1] (.npz)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_05188_b200 import api, synth  # noqa: E402

n, f, N, T_data = 30, 3, 512, 400
m = synth.make_market(n, T_data, 1.0 / 252, 77, n_feat=f)
cfg = api.make_config(N, n, f, 100, 1, 100, 0, 1e6, 0.002, 1.0, 0.99, 77)
env = api.Env(cfg, torch.from_numpy(m.close).cuda(), torch.from_numpy(m.feat).cuda())
H = int(sys.argv[2]) if len(sys.argv) > 2 else 512
aw = synth.make_actor(env.obs_dim, 3, H, n, 78)
params = api.pack_actor_params(cfg, [aw], 3, H)
actor = api.make_actor(3, H, params)
tr = api.Trajectory.allocate(1, N, n, env.k_pad, mu=True, critic=True)
env.reset(synth.tile_starts(env.n_tiles, T_data, 100, 79))
env.rollout(1, tr, actor=actor)
torch.cuda.synchronize()
np.savez(sys.argv[1], mu=tr.mu[0].cpu().numpy(), val=tr.val[0].cpu().numpy(), logp=tr.logp[0].cpu().numpy())
