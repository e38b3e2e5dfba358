"""Thin Python binding over libpod.so (same names as the C ABI).

PyTorch supplies device memory, streams and process groups; every step of the
hot path runs in libpod's CUDA kernels.  Nothing here computes the method:
functions allocate or lay out buffers and marshal pointers.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import check, load

ENV_TILE = 32


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def kernel_launches() -> int:
    """Kernels libpod has launched in this process (cached graphs count their kernel nodes)."""
    return int(load().pod_kernel_launches())


def make_config(n_envs, n_stocks, n_feat, horizon, n_agents=1, h_max=100, env_offset=0, initial_capital=1e6,
                cost_rate=0.002, reward_scale=1.0, gamma=0.99, seed=0) -> _lib.EnvConfig:
    return _lib.EnvConfig(n_envs, n_stocks, n_feat, n_agents, horizon, h_max, env_offset, initial_capital, cost_rate,
                          reward_scale, gamma, seed)


def config_from_workload(w, n_envs=None, env_offset=0) -> _lib.EnvConfig:
    return make_config(n_envs or w.n_envs, w.n_stocks, w.n_feat, w.horizon, w.n_agents, w.h_max, env_offset, w.C0,
                       w.cost, w.reward_scale, w.gamma, w.seed)


def actor_layout(cfg: _lib.EnvConfig, n_hidden: int, hidden: int) -> _lib.ActorLayout:
    L = _lib.ActorLayout()
    check(load().pod_actor_layout_get(C.byref(cfg), n_hidden, hidden, C.byref(L)), "pod_actor_layout_get")
    return L


def pod_env_workspace_size(cfg: _lib.EnvConfig) -> int:
    b = C.c_size_t(0)
    check(load().pod_env_workspace_size(C.byref(cfg), C.byref(b)), "pod_env_workspace_size")
    return int(b.value)


def pack_actor_params(cfg: _lib.EnvConfig, agents: Sequence, n_hidden: int, hidden: int,
                      device="cuda") -> torch.Tensor:
    """Lay out per-agent weights (synth.ActorWeights: W[l] [out, in] bf16-representable float32,
    b[l], log_std) in the slab format of pod_actor_layout: returns uint8 [P, param_bytes]."""
    L = actor_layout(cfg, n_hidden, hidden)
    pb = int(L.param_bytes)
    slab = np.zeros((len(agents), pb), dtype=np.uint8)
    for a, w in enumerate(agents):
        for l in range(L.n_layers):
            rows, cols = L.w_rows[l], L.w_cols[l]
            Wp = torch.zeros((rows, cols), dtype=torch.bfloat16)
            Wl = torch.from_numpy(np.ascontiguousarray(w.W[l], dtype=np.float32))
            Wp[: Wl.shape[0], : Wl.shape[1]] = Wl.to(torch.bfloat16)
            raw = Wp.view(torch.uint8).numpy().ravel()
            o = int(L.w_offset[l])
            slab[a, o : o + raw.size] = raw
            if l == L.n_layers - 1 and getattr(w, "w_v", None) is not None:
                # critic: head row n (R#22)
                Wp[cfg.n_stocks, : w.w_v.size] = torch.from_numpy(np.ascontiguousarray(w.w_v, np.float32)).to(torch.bfloat16)
                raw = Wp.view(torch.uint8).numpy().ravel()
                o = int(L.w_offset[l])
                slab[a, o : o + raw.size] = raw
            bp = np.zeros(rows, dtype=np.float32)
            bp[: w.b[l].size] = w.b[l]
            if l == L.n_layers - 1 and getattr(w, "w_v", None) is not None:
                bp[cfg.n_stocks] = np.float32(w.b_v)
            o = int(L.b_offset[l])
            slab[a, o : o + 4 * rows] = bp.view(np.uint8)
        ls = np.zeros(L.n_out_pad, dtype=np.float32)
        ls[: w.log_std.size] = w.log_std
        o = int(L.log_std_offset)
        slab[a, o : o + 4 * L.n_out_pad] = ls.view(np.uint8)
    return torch.from_numpy(slab).to(device)


@dataclass
class Trajectory:
    obs: torch.Tensor                  # bf16 [T+1, N, k_pad]
    act: Optional[torch.Tensor]        # f32 [T, N, n]
    logp: Optional[torch.Tensor]       # f32 [T, N]
    rew: torch.Tensor                  # f32 [T, N]
    done: torch.Tensor                 # u8 [T, N]
    mu: Optional[torch.Tensor] = None
    dbg_aint: Optional[torch.Tensor] = None
    dbg_hold: Optional[torch.Tensor] = None
    dbg_cash: Optional[torch.Tensor] = None
    val: Optional[torch.Tensor] = None    # f32 [T+1, N] critic V(s_t) (R#22)
    equity: Optional[torch.Tensor] = None  # f64 [T, N] account value after each step (R#25)

    @staticmethod
    def allocate(T: int, N: int, n: int, k_pad: int, device="cuda", debug=False, mu=False, sampled=True,
                 critic=False, equity=False):
        z = dict(device=device)
        return Trajectory(
            obs=torch.empty((T + 1, N, k_pad), dtype=torch.bfloat16, **z),
            act=torch.empty((T, N, n), dtype=torch.float32, **z) if sampled else None,
            logp=torch.empty((T, N), dtype=torch.float32, **z) if sampled else None,
            rew=torch.empty((T, N), dtype=torch.float32, **z),
            done=torch.empty((T, N), dtype=torch.uint8, **z),
            mu=torch.empty((T, N, n), dtype=torch.float32, **z) if (mu or debug) and sampled else None,
            dbg_aint=torch.empty((T, N, n), dtype=torch.int16, **z) if debug else None,
            dbg_hold=torch.empty((T, N, n), dtype=torch.int32, **z) if debug else None,
            dbg_cash=torch.empty((T, N), dtype=torch.float64, **z) if debug else None,
            val=torch.empty((T + 1, N), dtype=torch.float32, **z) if critic and sampled else None,
            equity=torch.empty((T, N), dtype=torch.float64, **z) if equity else None,
        )

    def c(self) -> _lib.Traj:
        return _lib.Traj(*[None if x is None else x.data_ptr() for x in
                           (self.obs, self.act, self.logp, self.rew, self.done, self.mu, self.dbg_aint,
                            self.dbg_hold, self.dbg_cash, self.val, self.equity)])


class Env:
    """pod_env_t handle.  Owns (via torch) its workspace; the market tensors
    must stay alive as long as the Env (it keeps references)."""

    def __init__(self, cfg: _lib.EnvConfig, close: torch.Tensor, feat: Optional[torch.Tensor]):
        L = load()
        assert close.is_cuda and close.dtype == torch.float32 and close.is_contiguous()
        self.cfg = cfg
        self.close = close
        self.feat = feat
        self.T_data = int(close.shape[0])
        self.market = _lib.Market(close.data_ptr(), None if feat is None else feat.data_ptr(), self.T_data)
        self.ws = torch.empty(pod_env_workspace_size(cfg), dtype=torch.uint8, device=close.device)
        h = C.c_void_p()
        check(L.pod_env_create(C.byref(cfg), C.byref(self.market), _ptr(self.ws), self.ws.numel(), C.byref(h)),
              "pod_env_create")
        self.h = h
        self.N = cfg.n_envs
        self.n = cfg.n_stocks
        self.n_tiles = (self.N + ENV_TILE - 1) // ENV_TILE
        od = 1 + 2 * cfg.n_stocks + cfg.n_stocks * cfg.n_feat
        self.obs_dim = od
        self.k_pad = (od + 63) // 64 * 64

    def close_handle(self):
        if getattr(self, "h", None):
            load().pod_env_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close_handle()
        except Exception:
            pass

    def reset(self, tile_starts: Optional[np.ndarray] = None, obs0: Optional[torch.Tensor] = None, stream=None):
        st = None
        if tile_starts is not None:
            st = np.ascontiguousarray(tile_starts, dtype=np.int64)
            assert st.size == self.n_tiles
        check(load().pod_env_reset(self.h, None if st is None else st.ctypes.data_as(C.c_void_p), _ptr(obs0),
                                   _stream(stream)), "pod_env_reset")

    def rollout(self, T: int, traj: Trajectory, actor: Optional[_lib.Actor] = None,
                injected_u: Optional[torch.Tensor] = None, deterministic=False,
                fitness_out: Optional[torch.Tensor] = None, stream=None):
        check(load().pod_rollout(self.h, None if actor is None else C.byref(actor), int(T), C.byref(traj.c()),
                                 _ptr(injected_u), 1 if deterministic else 0, _ptr(fitness_out), _stream(stream)),
              "pod_rollout")

    def profile(self, stride: int):
        """Bracket the actor and env-step launches of every `stride`-th step with CUDA events (0 = off)."""
        check(load().pod_env_profile(self.h, int(stride)), "pod_env_profile")

    def profile_read(self, stream=None):
        am, em = C.c_double(0), C.c_double(0)
        al, el = C.c_double(0), C.c_double(0)
        check(load().pod_env_profile_read(self.h, C.byref(am), C.byref(al), C.byref(em), C.byref(el),
                                          _stream(stream)), "pod_env_profile_read")
        return am.value, al.value, em.value, el.value

    def fitness(self, out: torch.Tensor, stream=None):
        check(load().pod_env_fitness(self.h, _ptr(out), _stream(stream)), "pod_env_fitness")

    def read_state(self, stream=None):
        dev = self.close.device
        hold = torch.empty((self.N, self.n), dtype=torch.int32, device=dev)
        cash = torch.empty(self.N, dtype=torch.float64, device=dev)
        asset = torch.empty(self.N, dtype=torch.float64, device=dev)
        ep = torch.empty(self.N, dtype=torch.float64, device=dev)
        check(load().pod_env_read_state(self.h, _ptr(hold), _ptr(cash), _ptr(asset), _ptr(ep), _stream(stream)),
              "pod_env_read_state")
        return hold, cash, asset, ep

    def check(self, stream=None):
        check(load().pod_env_check(self.h, _stream(stream)), "pod_env_check")


def make_actor(n_hidden: int, hidden: int, params: torch.Tensor, act: int = 0) -> _lib.Actor:
    return _lib.Actor(n_hidden, hidden, act, 0, params.data_ptr(), params.shape[1] if params.dim() == 2 else params.numel())


def pod_gae(rew, val, done, boot, gamma, lam, adv=None, ret=None, stream=None, normalize=False, stats=None):
    """GAE over [T, N]; normalize=True also rewrites adv as (A - mean) / std over the buffer (R#23),
    with the float64 sums (sum A, sum A^2) left in `stats` (a [2] float64 device tensor, allocated if None)."""
    T, N = rew.shape
    adv = torch.empty_like(rew) if adv is None else adv
    ret = torch.empty_like(rew) if ret is None else ret
    if normalize and stats is None:
        stats = torch.empty(2, dtype=torch.float64, device=rew.device)
    check(load().pod_gae(_ptr(rew), _ptr(val), _ptr(done), _ptr(boot), T, N, float(gamma), float(lam), _ptr(adv),
                         _ptr(ret), _ptr(stats) if normalize else None, _stream(stream)), "pod_gae")
    return adv, ret


def pod_elite_plan(fitness: np.ndarray, k: int) -> np.ndarray:
    f = np.ascontiguousarray(fitness, dtype=np.float64)
    plan = np.zeros(f.size, dtype=np.int32)
    check(load().pod_elite_plan(f.ctypes.data_as(C.c_void_p), f.size, int(k), plan.ctypes.data_as(C.c_void_p)),
          "pod_elite_plan")
    return plan


def pod_elite_transfers(plan: np.ndarray, P_local: int, rank: int):
    p = np.ascontiguousarray(plan, dtype=np.int32)
    ops = (_lib.Transfer * (2 * p.size + 2))()
    n = C.c_int32(0)
    check(load().pod_elite_transfers(p.ctypes.data_as(C.c_void_p), p.size, int(P_local), int(rank), ops, len(ops),
                                     C.byref(n)), "pod_elite_transfers")
    return [(ops[i].kind, ops[i].peer, ops[i].src_local, ops[i].dst_local) for i in range(n.value)]


def fuse_pods(cfg: _lib.EnvConfig, n_hidden: int, hidden: int, params: torch.Tensor, K_local: int, tau: float = 1.0,
              prev: Optional[torch.Tensor] = None, comm: Optional["Comm"] = None, work: Optional[torch.Tensor] = None,
              stream=None):
    """K-pod ensemble fusion (pod_fuse_pods, R#24): params uint8 [P_local, param_bytes] (slots a*K_local + k are
    agent a's pods), prev float32 [P_local/K_local, n_elems] (in/out; optional when tau == 1)."""
    P_local = params.shape[0]
    check(load().pod_fuse_pods(comm.h if comm is not None else None, C.byref(cfg), n_hidden, hidden, _ptr(params),
                               params.shape[1], P_local, int(K_local), float(tau), _ptr(prev), _ptr(work),
                               _stream(stream)), "pod_fuse_pods")
    return prev


def fuse_pods_local_ranks(cfg: _lib.EnvConfig, n_hidden: int, hidden: int, params: Sequence[torch.Tensor],
                          K_local: int, tau: float = 1.0, prevs: Optional[Sequence[torch.Tensor]] = None, stream=None):
    """pod_fuse_pods_local_ranks: the fusion over R ranks' slab arrays on this device in one launch (block rows
    play the ranks and exchange partial sums as pod_fuse_pods' ranks do over peer memory)."""
    R = len(params)
    P_local = params[0].shape[0]
    nb = C.c_size_t(0)
    check(load().pod_fuse_workspace_size(C.byref(cfg), n_hidden, hidden, P_local, int(K_local), R, C.byref(nb)),
          "pod_fuse_workspace_size")
    ws = torch.empty(int(nb.value), dtype=torch.uint8, device=params[0].device)
    pp_arr = (C.c_void_p * R)(*[p.data_ptr() for p in params])
    pv_arr = (C.c_void_p * R)(*[p.data_ptr() for p in prevs]) if prevs is not None else None
    pp = C.cast(pp_arr, C.c_void_p)
    pv = C.cast(pv_arr, C.c_void_p) if pv_arr is not None else None
    check(load().pod_fuse_pods_local_ranks(C.byref(cfg), n_hidden, hidden, pp, params[0].shape[1], R, P_local,
                                           int(K_local), float(tau), pv, _ptr(ws), ws.numel(), _stream(stream)),
          "pod_fuse_pods_local_ranks")
    return ws


def backtest_metrics(v0: torch.Tensor, curve: torch.Tensor, periods_per_year: float, rf_per_period: float = 0.0,
                     stream=None) -> torch.Tensor:
    """Evaluator metrics per env (pod_backtest_metrics, R#25): returns f64 [5, N] = cumulative return, annual
    return, annual volatility, Sharpe (NaN if degenerate), max drawdown."""
    T, N = curve.shape
    out = torch.empty((5, N), dtype=torch.float64, device=curve.device)
    check(load().pod_backtest_metrics(_ptr(v0), _ptr(curve), T, N, float(periods_per_year), float(rf_per_period),
                                      _ptr(out), _stream(stream)), "pod_backtest_metrics")
    return out


def early_stop(history, patience: int):
    """(stop, best) of the evaluator's early-stop rule (pod_early_stop, R#25)."""
    h = np.ascontiguousarray(history, dtype=np.float64)
    stop, best = C.c_int32(0), C.c_int32(0)
    check(load().pod_early_stop(h.ctypes.data_as(C.c_void_p), h.size, int(patience), C.byref(stop), C.byref(best)),
          "pod_early_stop")
    return bool(stop.value), int(best.value)


class PPOLearner:
    """PPO clipped-surrogate learner of agent 0 (pod_ppo_update, R#26) on a float32 master copy of the rollout
    slab, with Adam moments; `update` runs minibatches over the flattened rollout buffers and refreshes the
    rollout slab (bf16) in place."""

    def __init__(self, cfg: _lib.EnvConfig, n_hidden: int, hidden: int, params: torch.Tensor, act: int = 0,
                 batch: int = 1024, ratio_clip=0.25, entropy_coef=0.02, value_coef=0.5, learning_rate=2.0 ** -14,
                 betas=(0.9, 0.999), adam_eps=1e-8, fp32: bool = False):
        """fp32=True runs the products on float32 operands (the reference mode: master weights, float32
        activations and deltas) instead of bf16 on the tensor cores."""
        self.cfg, self.n_hidden, self.hidden, self.act, self.batch = cfg, n_hidden, hidden, act, batch
        self.params = params
        L = actor_layout(cfg, n_hidden, hidden)
        self.n_elems = int(L.n_elems)
        dev = params.device
        self.master = torch.empty(self.n_elems, dtype=torch.float32, device=dev)
        # widen the rollout slab of agent 0 into the master copy (fusion with K = 1, tau = 1: slab unchanged)
        fuse_pods(cfg, n_hidden, hidden, params[:1], 1, tau=1.0, prev=self.master.view(1, -1))
        self.m = torch.zeros_like(self.master)
        self.v = torch.zeros_like(self.master)
        self.t = 0
        self.hp = _lib.PpoHparams(ratio_clip, entropy_coef, value_coef, learning_rate, betas[0], betas[1], adam_eps,
                                  1 if fp32 else 0)
        nb = C.c_size_t(0)
        check(load().pod_ppo_workspace_size(C.byref(cfg), n_hidden, hidden, batch, C.byref(nb)), "pod_ppo_workspace_size")
        self.ws = torch.empty(int(nb.value), dtype=torch.uint8, device=dev)
        self.losses = torch.zeros(4, dtype=torch.float64, device=dev)

    def set_hparams(self, **kw):
        """Change hyper-parameters between updates (schedules): ratio_clip, entropy_coef, value_coef,
        learning_rate, adam_beta1, adam_beta2, adam_eps.  They reach the captured minibatch loop through
        device memory, so the next update replays the same graph."""
        for k, v in kw.items():
            if not hasattr(self.hp, k) or k == "fp32_operands":
                raise ValueError(f"unknown PPO hyper-parameter {k!r}")
            setattr(self.hp, k, float(v))

    def update(self, obs: torch.Tensor, act_raw: torch.Tensor, logp_old: torch.Tensor, adv: torch.Tensor,
               ret: torch.Tensor, perm: torch.Tensor, grad_out: Optional[torch.Tensor] = None, stream=None):
        """obs bf16 [M, k_pad], act_raw f32 [M, n], logp_old/adv/ret f32 [M], perm i32 [n_mb * batch]."""
        M = obs.shape[0]
        n_mb = perm.numel() // self.batch
        if stream is not None:
            with torch.cuda.stream(stream):
                self.losses.zero_()
        else:
            self.losses.zero_()
        check(load().pod_ppo_update(C.byref(self.cfg), self.n_hidden, self.hidden, self.act, C.byref(self.hp),
                                    _ptr(self.master), _ptr(self.m), _ptr(self.v), self.t, _ptr(self.params),
                                    self.params.shape[1], _ptr(obs), _ptr(act_raw), _ptr(logp_old), _ptr(adv),
                                    _ptr(ret), M, _ptr(perm), self.batch, n_mb, _ptr(self.losses), _ptr(grad_out),
                                    _ptr(self.ws), self.ws.numel(), _stream(stream)), "pod_ppo_update")
        self.t += n_mb
        return self.losses

    def check(self, stream=None):
        """pod_ppo_check: raises PodError(POD_ERR_NONFINITE) if a minibatch loss was not finite."""
        check(load().pod_ppo_check(_ptr(self.ws), _stream(stream)), "pod_ppo_check")


class Comm:
    """NCCL communicator of libpod (one process per GPU).  The torch process
    group (if any) only broadcasts the 128-byte unique id."""

    def __init__(self, nranks: int, rank: int, max_agents_local: int, group=None):
        L = load()
        uid = np.zeros(128, dtype=np.uint8)
        if rank == 0:
            check(L.pod_comm_unique_id(uid.ctypes.data_as(C.c_void_p)), "pod_comm_unique_id")
        if nranks > 1:
            import torch.distributed as dist
            t = torch.from_numpy(uid.astype(np.int64))
            if dist.get_backend(group) == "nccl":
                t = t.cuda()
            dist.broadcast(t, 0, group=group)
            uid = t.cpu().numpy().astype(np.uint8)
        h = C.c_void_p()
        check(L.pod_comm_init(uid.ctypes.data_as(C.c_void_p), nranks, rank, max_agents_local, C.byref(h)),
              "pod_comm_init")
        self.h = h
        self.nranks, self.rank = nranks, rank

    def select_elite(self, fitness_local: torch.Tensor, k: int, params: torch.Tensor, stream=None) -> np.ndarray:
        P_local = fitness_local.numel()
        plan = np.zeros(P_local * self.nranks, dtype=np.int32)
        check(load().pod_select_elite(self.h, _ptr(fitness_local), P_local, int(k), _ptr(params), params.shape[1],
                                      plan.ctypes.data_as(C.c_void_p), _stream(stream)), "pod_select_elite")
        return plan

    def destroy(self):
        if getattr(self, "h", None):
            load().pod_comm_destroy(self.h)
            self.h = None
