"""Diagnostics (needs the POD_EXP_GTIME build, selected with POD_LIB_PATH): per-step globaltimer phases of
CTA 0 inside the fused rollout kernel — obs landed -> head accumulator ready (the actor's layers),
-> both CTAs' heads written, -> env step done, -> next obs landed (s_{t+1} round trip)."""
import sys

import ctypes as C
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
T = 128
tr = api.Trajectory.allocate(T, w.n_envs, w.n_stocks, env.k_pad)
env.reset(synth.tile_starts(env.n_tiles, w.T_data, min(w.horizon, w.T_data - 2), 1))
L = _lib.load()
for _ in range(3):
    env.rollout(T, tr, actor=actor)
torch.cuda.synchronize()
L.pod_debug_gtime(None, 1)
env.rollout(T, tr, actor=actor)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (1024 * 12))()
L.pod_debug_ftime(buf)
g = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 12)[:T].astype(np.float64)
med = lambda x: float(np.median(x))
names = ["actor layers", "head compute", "head fence+exchange", "env loads", "env sells", "env buys",
         "env ledger sync", "env reward", "env obs rows", "env end", "env fence+exchange"]
order = [0, 1, 2, 3, 6, 11, 10, 7, 8, 9, 4, 5]   # stamp columns in time order
parts = [med(g[:, order[k + 1]] - g[:, order[k]]) for k in range(len(order) - 1)]
obs = med(g[1:, 0] - g[:-1, 5])
step = med(np.diff(g[:, 0]))
print(f"{w.name} per step (ns, median over {T}): step {step:.0f}  " +
      "  ".join(f"{n} {p:.0f}" for n, p in zip(names, parts)) + f"  -> next obs landed {obs:.0f}")
