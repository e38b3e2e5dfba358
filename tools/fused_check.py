"""Diagnostics: the fused rollout kernel (POD_FUSED=1, the default where eligible) against the
separate actor / env-step launches (POD_FUSED=0) on the same inputs — every trajectory output and the
final env state must be bit-identical — and the device time of both per rollout.

    python tools/fused_check.py [C2|C3|C4 ...]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_05188_b200 import api, configs, synth  # noqa: E402


def run(w, fused: bool, T: int, horizon: int, deterministic: bool, reps: int = 0):
    os.environ["POD_FUSED"] = "1" if fused else "0"
    m = synth.make_market(w.n_stocks, w.T_data, w.dt, w.seed, n_feat=w.n_feat)
    cfg = api.config_from_workload(w)
    cfg.horizon = horizon
    env = api.Env(cfg, torch.from_numpy(m.close).cuda(), torch.from_numpy(m.feat).cuda())
    aws = [synth.make_actor(env.obs_dim, w.n_hidden, w.hidden, w.n_stocks, 1 + a) for a in range(w.n_agents)]
    params = api.pack_actor_params(cfg, aws, w.n_hidden, w.hidden)
    actor = api.make_actor(w.n_hidden, w.hidden, params)
    tr = api.Trajectory.allocate(T, w.n_envs, w.n_stocks, env.k_pad, debug=True, critic=True, equity=True)
    env.reset(synth.tile_starts(env.n_tiles, w.T_data, min(horizon, w.T_data - 2), 7))
    outs = []
    for _ in range(2):   # two rollouts: the second starts from the state the first left
        env.rollout(T, tr, actor=actor, deterministic=deterministic)
        torch.cuda.synchronize()
        outs.append({k: v.clone() for k, v in vars(tr).items() if v is not None})
    st = env.read_state()
    env.check()
    ms = None
    if reps:
        trb = api.Trajectory.allocate(T, w.n_envs, w.n_stocks, env.k_pad)
        for _ in range(3):
            env.rollout(T, trb, actor=actor)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            env.rollout(T, trb, actor=actor)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
    env.close_handle()
    return outs, st, ms


def main():
    time_only = "--time-only" in sys.argv
    names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["C2", "C3", "C4"]
    bad = 0
    for name in names:
        w = configs.preset(name, T_data=20000)
        if time_only:
            _, _, mf = run(w, True, w.T, w.horizon, False, reps=20)
            print(f"{name} T={w.T}: fused {mf:.3f} ms/rollout ({mf * 1e3 / w.T:.2f} us/step)", flush=True)
            continue
        for horizon, det in ((w.horizon, False), (40, False), (40, True)):
            T = 64
            t0 = time.time()
            a, sa, _ = run(w, True, T, horizon, det)
            b, sb, _ = run(w, False, T, horizon, det)
            diffs = []
            for r in range(2):
                for k in b[r]:
                    x, y = a[r][k], b[r][k]
                    if not torch.equal(x.view(torch.uint8) if x.dtype == torch.bfloat16 else x,
                                       y.view(torch.uint8) if y.dtype == torch.bfloat16 else y):
                        if x.is_floating_point():
                            nd = int((x != y).sum())
                        else:
                            nd = int((x != y).sum())
                        diffs.append(f"rollout {r} {k}: {nd} differ")
            for k, (x, y) in enumerate(zip(sa, sb)):
                if not torch.equal(x, y):
                    diffs.append(f"state {k}: {int((x != y).sum())} differ")
            bad += len(diffs)
            print(f"{name} H={horizon} det={det}: {'IDENTICAL' if not diffs else 'DIFF ' + '; '.join(diffs[:8])}"
                  f" ({time.time() - t0:.1f} s)", flush=True)
        _, _, mf = run(w, True, w.T, w.horizon, False, reps=10)
        _, _, mu = run(w, False, w.T, w.horizon, False, reps=10)
        print(f"{name} T={w.T}: fused {mf:.3f} ms/rollout ({mf * 1e3 / w.T:.2f} us/step), separate {mu:.3f} ms "
              f"({mu * 1e3 / w.T:.2f} us/step)", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
