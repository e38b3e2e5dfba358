"""Diagnostics: per-phase clock64 timeline of the actor kernel at the C3 shape."""
import sys
import numpy as np
import torch
import ctypes as C
sys.path.insert(0, ".")
from paper_2111_05188_b200 import api, synth, configs, _lib

w = configs.preset(sys.argv[1] if len(sys.argv) > 1 else "C3", T_data=20000)
m = synth.make_market(w.n_stocks, w.T_data, w.dt, w.seed, n_feat=w.n_feat)
cfg = api.config_from_workload(w)
env = api.Env(cfg, torch.from_numpy(m.close).cuda(), torch.from_numpy(m.feat).cuda())
aw = synth.make_actor(env.obs_dim, w.n_hidden, w.hidden, w.n_stocks, 1)
params = api.pack_actor_params(cfg, [aw] * w.n_agents, w.n_hidden, w.hidden)
actor = api.make_actor(w.n_hidden, w.hidden, params)
T = 4
tr = api.Trajectory.allocate(T, w.n_envs, w.n_stocks, env.k_pad)
grid = 2 * ((w.n_envs // w.n_agents + 127) // 128) * w.n_agents
buf = torch.zeros(grid * 64, dtype=torch.int64, device="cuda")
ebuf = torch.zeros(env.n_tiles * 8, dtype=torch.int64, device="cuda")
_lib.load().pod_debug_trace(env.h, C.c_void_p(buf.data_ptr()), C.c_void_p(ebuf.data_ptr()))
env.reset(synth.tile_starts(env.n_tiles, w.T_data, min(w.horizon, w.T_data - 2), 1))
# argv[2]: rollouts of T = 4 steps before the traced one (the trace keeps the last launch): a few dozen put the
# envs in an episode's steady state (cash spent within the first buys of each step)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    env.rollout(T, tr, actor=actor)
torch.cuda.synchronize()
b = buf.view(grid, 64).cpu().numpy().astype(np.int64)
rel = b - b[:, :1]
names = {1: "obs", 26: "end", 24: "head_acc", 25: "head_done"}
for j in range(4):
    names[16 + 2 * j] = f"L1 atom{j} tmem"
    names[17 + 2 * j] = f"L1 atom{j} sent"
for j in range(2):
    names[27 + 2 * j] = f"L1 atom{j} stored"
    names[28 + 2 * j] = f"L1 atom{j} all arrived"
for l in range(w.n_hidden + 1):
    names[2 + 4 * l] = f"L{l}_mma_start"
    names[3 + 4 * l] = f"L{l}_mma_issued"
    if l < w.n_hidden:
        names[4 + 4 * l] = f"L{l}_acc_ready"
        names[5 + 4 * l] = f"L{l}_epi_done"
for k in sorted(names):
    col = rel[:, k]
    print(f"{names[k]:16s} median {int(np.median(col)):8d}  min {int(col.min()):8d}  max {int(col.max()):8d}")

eb = ebuf.view(env.n_tiles, 8).cpu().numpy().astype(np.int64)
erel = eb - eb[:, :1]
for k, nm in enumerate(["start", "staged", "sells_done", "buys_done", "ledger_done", "rows_staged", "end"]):
    col = erel[:, k]
    print(f"env {nm:14s} median {int(np.median(col)):8d}  min {int(col.min()):8d}  max {int(col.max()):8d}")
print("env trace slot 7: median", int(np.median(eb[:, 7])), "max", int(eb[:, 7].max()))

lead = rel[0::2] if rel[1::2, 1].max() == 0 and rel[0::2, 1].max() > 0 else rel
print("L0 stage ready (MMA side):", [int(np.median(lead[:, 32 + q])) for q in range(16)])
print("producer issue times      :", [int(np.median(rel[:, 48 + q])) for q in range(16)])
