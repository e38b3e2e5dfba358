"""A bounded rollout + GAE + fitness case for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): `python tools/sanitize_case.py c1|persist3` runs the hot path once through the C ABI with
graphs off (POD_NO_GRAPH=1 is set by the caller so every kernel launch is visible to the tool).

  c1       configs[0]: Dow-30 daily, 16 envs, actor 2x128, T = 8 (ragged single tile)
  persist3 n = 100, 3x512 actor, 3 agents, 34,560 envs: 270 M-tiles on 74 persistent clusters (multi-tile
           phase wrap-around, agent switches inside a cluster), 1,080 env tiles (dense PDL launch), T = 2
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_05188_b200 import api, synth  # noqa: E402


def main(case: str):
    torch.cuda.set_device(0)
    api.load()
    if case == "c1":
        n, f, N, H, T, nh, hid, P, Td = 30, 3, 16, 64, 8, 2, 128, 1, 2611
    else:
        n, f, N, H, T, nh, hid, P, Td = 100, 3, 34560, 500, 2, 3, 512, 3, 3000
    m = synth.make_market(n, Td, 1 / 252, 5189, n_feat=f)
    cfg = api.make_config(N, n, f, H, P, 100, 0, 1e6, 0.002, 1.0, 0.99, 5189)
    env = api.Env(cfg, torch.from_numpy(m.close).cuda(), torch.from_numpy(m.feat).cuda())
    aws = [synth.make_actor(env.obs_dim, nh, hid, n, 3 + a) for a in range(P)]
    params = api.pack_actor_params(cfg, aws, nh, hid)
    actor = api.make_actor(nh, hid, params)
    tr = api.Trajectory.allocate(T, N, n, env.k_pad, critic=True)
    env.reset(synth.tile_starts(env.n_tiles, Td, H, 1))
    env.rollout(T, tr, actor=actor)
    adv, ret = api.pod_gae(tr.rew, tr.val[:T].contiguous(), tr.done, tr.val[T].contiguous(), 0.99, 0.95,
                           normalize=True)
    fit = torch.empty(P, dtype=torch.float64, device="cuda")
    env.fitness(fit)
    env.check()
    torch.cuda.synchronize()
    assert torch.isfinite(adv).all() and torch.isfinite(tr.val).all()
    print(f"sanitize case {case}: ok ({N} envs, T={T}, fitness {fit.cpu().numpy()})")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c1")
