"""Helpers for GPU-vs-oracle parity tests: seeded inputs, running both sides,
and the tolerance checks DESIGN.md §6 states.  The oracle side uses only
oracle/ (float64 C); the GPU side only paper_2111_05188_b200.api (libpod)."""
from __future__ import annotations

import numpy as np
import torch

import oracle
from paper_2111_05188_b200 import api, synth

OBS_RTOL = 2.0 ** -8       # bf16 RNE (2^-9) + fp32 evaluation
GAE_TOL = 1e-5             # x magnitude recurrence M_t
MU_ROW_RTOL = 2e-2         # north_star: actor logits within 2e-2 (bf16 MLP)


def bf16_to_f64(t: torch.Tensor) -> np.ndarray:
    return t.float().cpu().numpy().astype(np.float64)


class Case:
    """One env configuration on both sides."""

    def __init__(self, n, f, T_data, N, H, n_agents=1, C0=1e6, cost=0.002, scale=1.0, gamma=0.99, seed=7,
                 env_offset=0, h_max=100, market_seed=11, dt=1 / 252):
        self.market = synth.make_market(n, T_data, dt, market_seed, n_feat=f)
        self.n, self.f, self.N, self.H = n, f, N, H
        self.cfg = api.make_config(N, n, f, H, n_agents, h_max, env_offset, C0, cost, scale, gamma, seed)
        self.kw = dict(horizon=H, h_max=h_max, C0=C0, cost=cost, scale=scale, gamma=gamma, seed=seed,
                       env_offset=env_offset, n_agents=n_agents)
        self.n_tiles = (N + 31) // 32
        self.starts = synth.tile_starts(self.n_tiles, T_data, H, market_seed + 1)
        self.close_d = torch.from_numpy(self.market.close).cuda()
        self.feat_d = torch.from_numpy(self.market.feat).cuda()
        self.env = api.Env(self.cfg, self.close_d, self.feat_d)
        self.obs_dim = self.env.obs_dim
        self.k_pad = self.env.k_pad

    def env_starts(self):
        return np.repeat(self.starts, 32)[: self.N]

    def oracle_env(self):
        o = oracle.Env(self.market.close, self.market.feat, self.N, **self.kw)
        o.reset(self.env_starts())
        return o


def assert_obs_close(g_obs: torch.Tensor, o_obs: np.ndarray, obs_dim: int):
    g = bf16_to_f64(g_obs)
    assert np.all(g[..., obs_dim:] == 0.0), "obs pad columns must be zero"
    g = g[..., :obs_dim]
    err = np.abs(g - o_obs)
    bad = err > OBS_RTOL * np.abs(o_obs) + 1e-30
    assert not bad.any(), f"obs mismatch at {np.argwhere(bad)[:5]}: gpu {g[bad][:5]} oracle {o_obs[bad][:5]}"


def assert_env_exact(tr: api.Trajectory, out: dict, obs_dim: int):
    """Integer holdings, dones, cash ledger bit-identical; rewards = fp32(oracle)."""
    np.testing.assert_array_equal(tr.done.cpu().numpy(), out["done"])
    np.testing.assert_array_equal(tr.dbg_hold.cpu().numpy(), out["hold"])
    np.testing.assert_array_equal(tr.dbg_cash.cpu().numpy(), out["cash"])   # bit-identical float64 ledger
    np.testing.assert_array_equal(tr.rew.cpu().numpy(), out["rew"].astype(np.float32))
    assert_obs_close(tr.obs, out["obs"], obs_dim)


def gae_check(adv_g, ret_g, adv_o, ret_o, mag):
    ag = adv_g.cpu().numpy().astype(np.float64)
    rg = ret_g.cpu().numpy().astype(np.float64)
    tol = GAE_TOL * mag + 1e-6
    ea = np.abs(ag - adv_o)
    er = np.abs(rg - ret_o)
    assert (ea <= tol).all(), f"adv max err/tol {np.max(ea / tol)}"
    assert (er <= tol + 1e-6 * np.abs(ret_o)).all(), f"ret max err {np.max(er)}"


def mu_check(mu_g: np.ndarray, mu_o: np.ndarray):
    """Per-row relative L2 <= 2e-2 and elementwise |g-o| <= 2e-2 (|o| + rms_row(o))."""
    d = mu_g - mu_o
    rn = np.linalg.norm(d, axis=-1) / np.maximum(np.linalg.norm(mu_o, axis=-1), 1e-30)
    assert rn.max() <= MU_ROW_RTOL, f"mu row rel err {rn.max()}"
    rms = np.sqrt(np.mean(mu_o ** 2, axis=-1, keepdims=True))
    assert (np.abs(d) <= MU_ROW_RTOL * (np.abs(mu_o) + rms)).all()
    return float(rn.max())
