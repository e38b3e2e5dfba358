"""Diagnostics (needs the POD_EXP_GTIME build as libpod.so): per-step globaltimer spans of the actor
and env-step grids inside one rollout graph, and the gaps between them."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_05188_b200 import _lib, api, configs, synth  # noqa: E402

w = configs.preset(sys.argv[1] if len(sys.argv) > 1 else "C3", T_data=20000)
m = synth.make_market(w.n_stocks, w.T_data, w.dt, w.seed, n_feat=w.n_feat)
cfg = api.config_from_workload(w)
env = api.Env(cfg, torch.from_numpy(m.close).cuda(), torch.from_numpy(m.feat).cuda())
aw = synth.make_actor(env.obs_dim, w.n_hidden, w.hidden, w.n_stocks, 1)
params = api.pack_actor_params(cfg, [aw] * w.n_agents, w.n_hidden, w.hidden)
actor = api.make_actor(w.n_hidden, w.hidden, params)
T = 64
tr = api.Trajectory.allocate(T, w.n_envs, w.n_stocks, env.k_pad)
env.reset(synth.tile_starts(env.n_tiles, w.T_data, min(w.horizon, w.T_data - 2), 1))
L = _lib.load()
for _ in range(3):
    env.rollout(T, tr, actor=actor)
torch.cuda.synchronize()
L.pod_debug_gtime(None, 1)
env.rollout(T, tr, actor=actor)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (1024 * 4))()
L.pod_debug_gtime(buf, 0)
g = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 4)[:T].astype(np.float64)
g -= g[0, 0]
actor_dur = g[:, 1] - g[:, 0]
env_dur = g[:, 3] - g[:, 2]
gap_ae = g[:, 2] - g[:, 1]
gap_ea = g[1:, 0] - g[:-1, 3]
step = np.diff(g[:, 0])
print(f"per step (ns, median over {T}): step {np.median(step):.0f}  actor {np.median(actor_dur):.0f}  env {np.median(env_dur):.0f}"
      f"  gap actor->env {np.median(gap_ae):.0f}  gap env->actor {np.median(gap_ea):.0f}")
