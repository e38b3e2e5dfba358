"""End-to-end generational training on one GPU through the public API (paper Fig. 2 on one box):

  for each generation:
      for each agent's K pods (population slots): rollout (actor + critic + env) -> GAE (normalised)
          -> PPO update of the pod (learner)
      K-pod fusion of every agent (pod_fuse_pods)
      evaluation: deterministic rollout of one episode per env -> fitness; backtest metrics of the curve
      selection: top-k agents keep their weights, the rest take the elites' (pod_select_elite)
      early stop on the best fitness history (pod_early_stop)

Usage: python tools/train_loop.py [--config C2] [--agents 2] [--pods 2] [--gens 3] [--T 64]
Prints one line per generation (fitness per agent, best, Sharpe / max drawdown of the best agent's envs).
"""
import argparse
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_05188_b200 import api, configs, synth  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="C2")
    p.add_argument("--agents", type=int, default=2)
    p.add_argument("--pods", type=int, default=2)
    p.add_argument("--gens", type=int, default=3)
    p.add_argument("--T", type=int, default=64)
    p.add_argument("--envs", type=int, default=1024)
    p.add_argument("--patience", type=int, default=5)
    args = p.parse_args()

    w = configs.preset(args.config)
    A, K = args.agents, args.pods
    P = A * K                                   # population slots: agent a's pods are slots a*K .. a*K+K-1
    N = args.envs * P                           # every slot gets its own envs for its rollouts
    cfg = api.make_config(N, w.n_stocks, w.n_feat, min(w.horizon, 512), P, w.h_max, 0, w.C0, w.cost,
                          w.reward_scale, w.gamma, w.seed)
    m = synth.make_market(w.n_stocks, w.T_data, w.dt, w.seed, n_feat=w.n_feat)
    close, feat = torch.from_numpy(m.close).cuda(), torch.from_numpy(m.feat).cuda()
    env = api.Env(cfg, close, feat)
    starts = synth.tile_starts(env.n_tiles, w.T_data, min(w.horizon, 512), w.seed + 1)
    # each pod of an agent starts from the same weights (different noise streams via the env ids)
    aws = [synth.make_actor(env.obs_dim, w.n_hidden, w.hidden, w.n_stocks, w.seed * 1000 + s // K) for s in range(P)]
    params = api.pack_actor_params(cfg, aws, w.n_hidden, w.hidden)
    actor = api.make_actor(w.n_hidden, w.hidden, params)
    T = args.T
    tr = api.Trajectory.allocate(T, N, w.n_stocks, env.k_pad, critic=True)
    learners = [api.PPOLearner(cfg, w.n_hidden, w.hidden, params[s : s + 1], batch=1024) for s in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    comm = api.Comm(1, 0, P)
    fit = torch.empty(P, dtype=torch.float64, device="cuda")
    prev = torch.empty((A, int(api.actor_layout(cfg, w.n_hidden, w.hidden).n_elems)), dtype=torch.float32,
                       device="cuda")
    history = []
    rng = np.random.default_rng(0)
    env.reset(starts)
    for gen in range(args.gens):
        # ---- explore + learn: one rollout of all slots, then each pod learns from its own envs
        env.rollout(T, tr, actor=actor)
        adv, ret = api.pod_gae(tr.rew, tr.val[:T].contiguous(), tr.done, tr.val[T].contiguous(), w.gamma, w.lam,
                               normalize=True)
        per = N // P
        main = torch.cuda.current_stream()
        for s in range(P):   # the pods' learners run concurrently, one stream each
            rows = torch.arange(s * per, (s + 1) * per, device="cuda")
            sel = (torch.arange(T, device="cuda")[:, None] * N + rows[None, :]).reshape(-1)
            M = sel.numel()
            obs = tr.obs[:T].reshape(T * N, env.k_pad)[sel].contiguous()
            act = tr.act.reshape(T * N, w.n_stocks)[sel].contiguous()
            lpo = tr.logp.reshape(T * N)[sel].contiguous()
            a_s = adv.reshape(T * N)[sel].contiguous()
            r_s = ret.reshape(T * N)[sel].contiguous()
            n_mb = max(1, M // 1024)
            perm = torch.from_numpy(rng.permutation(M)[: n_mb * 1024].astype(np.int32)).cuda()
            streams[s].wait_stream(main)
            for t_ in (obs, act, lpo, a_s, r_s, perm):
                t_.record_stream(streams[s])
            learners[s].update(obs, act, lpo, a_s, r_s, perm, stream=streams[s])
        for s in range(P):
            main.wait_stream(streams[s])
        # ---- K-pod fusion (hard adoption of the mean, tau = 1)
        api.fuse_pods(cfg, w.n_hidden, w.hidden, params, K, tau=1.0, prev=prev)
        for s in range(P):   # learners continue from the fused parameters
            api.fuse_pods(cfg, w.n_hidden, w.hidden, params[s : s + 1], 1, tau=1.0,
                          prev=learners[s].master.view(1, -1))
        # ---- evaluation: one deterministic episode from reset, equity curve for the backtest metrics
        env.reset(starts)
        _, _, v0, _ = env.read_state()
        H = cfg.horizon
        ev = api.Trajectory.allocate(H, N, w.n_stocks, env.k_pad, equity=True)
        env.rollout(H, ev, actor=actor, deterministic=True, fitness_out=fit)
        metrics = api.backtest_metrics(v0, ev.equity, 252.0 if args.config in ("C1", "C2") else 252.0 * 390)
        # ---- selection across the population slots (pods of an agent have identical fused weights)
        plan = comm.select_elite(fit, max(1, P // 2), params)
        f = fit.cpu().numpy()
        best = int(np.argmax(f))
        history.append(float(f.max()))
        stop, best_gen = api.early_stop(history, args.patience)
        mb = metrics[:, best * per : (best + 1) * per].cpu().numpy()
        print(f"gen {gen}: fitness {np.round(f, 4).tolist()}  best slot {best}  plan {plan.tolist()}  "
              f"Sharpe(mean) {np.nanmean(mb[3]):.3f}  maxDD(mean) {mb[4].mean():.3f}  early-stop {stop}")
        for s in range(P):   # the selected slabs become the learners' masters
            api.fuse_pods(cfg, w.n_hidden, w.hidden, params[s : s + 1], 1, tau=1.0,
                          prev=learners[s].master.view(1, -1))
        env.reset(starts)
        if stop:
            break
    torch.cuda.synchronize()
    print("train loop OK")


if __name__ == "__main__":
    main()
