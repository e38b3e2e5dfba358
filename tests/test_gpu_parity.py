"""GPU parity: libpod's CUDA path vs the float64 oracle on the same seeded
inputs.  Every call goes through the C ABI (paper_2111_05188_b200.api).

Bars: integer holdings, dones and the float64 cash ledger bit-exact; rewards
equal the float32 rounding of the oracle's float64 reward; observations within
bf16 rounding; GAE within 1e-5 x the magnitude recurrence; actor means within
2e-2 (north_star); Gaussian noise, log-probs and the action map checked
against the oracle's Philox/Box–Muller and map.
"""
import math

import sys

import numpy as np
import pytest
import torch

import oracle
from paper_2111_05188_b200 import PodError, api, synth
from parity_helpers import Case, assert_env_exact, assert_obs_close, bf16_to_f64, gae_check, mu_check

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    api.load()
    torch.cuda.set_device(0)


def _actor(case, n_hidden, hidden, seed=3, n_agents=1, act=0):
    aws = [synth.make_actor(case.obs_dim, n_hidden, hidden, case.n, seed + a) for a in range(n_agents)]
    params = api.pack_actor_params(case.cfg, aws, n_hidden, hidden)
    return aws, params, api.make_actor(n_hidden, hidden, params, act)


# ----------------------------------------------------------------- injected
@pytest.mark.parametrize("kind", ["uniform", "all_buy", "all_sell", "sparse", "buy_then_sell"])
@pytest.mark.parametrize("N,H", [(16, 64), (100, 13)])
def test_injected_actions_exact(kind, N, H):
    c = Case(n=30, f=3, T_data=400, N=N, H=H)
    T = 40
    u = synth.injected_u(kind, T, N, c.n, 5)
    tr = api.Trajectory.allocate(T, N, c.n, c.k_pad, debug=True, sampled=False)
    c.env.reset(c.starts)
    c.env.rollout(T, tr, injected_u=torch.from_numpy(u).cuda())
    c.env.check()
    o = c.oracle_env()
    out = o.rollout(T, "inject", u=u, want=("obs", "rew", "done", "hold", "cash", "a_int"))
    np.testing.assert_array_equal(tr.dbg_aint.cpu().numpy(), out["a_int"])
    assert_env_exact(tr, out, c.obs_dim)
    hold, cash, asset, ep = c.env.read_state()
    np.testing.assert_array_equal(hold.cpu().numpy(), o.hold)
    np.testing.assert_array_equal(cash.cpu().numpy(), o.cash)
    np.testing.assert_array_equal(asset.cpu().numpy(), o.asset)
    np.testing.assert_array_equal(ep.cpu().numpy(), o.ep_ret)


def test_injected_end_of_data_and_continuation():
    # tiles starting near the end of the data end their episodes at t+1 == T_data-1;
    # state carries across two rollout calls
    c = Case(n=5, f=2, T_data=120, N=64, H=50, C0=2e4, cost=0.001)
    c.starts[:] = [69, 10]            # 69 + 50 = 119 = T_data - 1 -> ends by data exhaustion
    u = synth.injected_u("uniform", 70, 64, 5, 9)
    o = c.oracle_env()
    out = o.rollout(70, "inject", u=u, want=("obs", "rew", "done", "hold", "cash"))
    c.env.reset(c.starts)
    for lo, hi in ((0, 33), (33, 70)):
        T = hi - lo
        tr = api.Trajectory.allocate(T, 64, 5, c.k_pad, debug=True, sampled=False)
        c.env.rollout(T, tr, injected_u=torch.from_numpy(np.ascontiguousarray(u[lo:hi])).cuda())
        sub = {k: out[k][lo:hi] for k in ("rew", "done", "hold", "cash")}
        sub["obs"] = out["obs"][lo : hi + 1]
        assert_env_exact(tr, sub, c.obs_dim)


# ----------------------------------------------------------------- sampled
@pytest.mark.parametrize("shape", ["dow30_2x128", "nasdaq100_3x512"])
def test_sampled_rollout_parity(shape):
    if shape == "dow30_2x128":
        c = Case(n=30, f=3, T_data=500, N=160, H=24, seed=21, env_offset=1000)
        nh, hid, T = 2, 128, 30
    else:
        c = Case(n=100, f=3, T_data=3000, N=256, H=400, seed=22, dt=1 / (252 * 390))
        nh, hid, T = 3, 512, 6
    aws, params, actor = _actor(c, nh, hid)
    tr = api.Trajectory.allocate(T, c.N, c.n, c.k_pad, debug=True)
    c.env.reset(c.starts)
    c.env.rollout(T, tr, actor=actor)
    c.env.check()
    obs_g = bf16_to_f64(tr.obs)[..., : c.obs_dim]
    mu_g = tr.mu.cpu().numpy().astype(np.float64)
    raw_g = tr.act.cpu().numpy().astype(np.float64)
    logp_g = tr.logp.cpu().numpy().astype(np.float64)
    a_g = tr.dbg_aint.cpu().numpy()
    w = oracle.actor_flat(aws[0].W, aws[0].b, aws[0].log_std)
    ls = aws[0].log_std.astype(np.float64)
    sig = np.exp(ls)
    worst = 0.0
    for t in range(T):
        # actor mean: oracle float64 MLP on the GPU's own (bf16) observation
        mu_o = oracle.actor_mu(w, obs_g[t], nh, hid, c.n)
        worst = max(worst, mu_check(mu_g[t], mu_o))
        for e in range(c.N):
            z_o = oracle.normals(c.cfg.seed, c.cfg.env_offset + e, t, c.n)
            z_g = (raw_g[t, e] - mu_g[t, e]) / sig
            assert np.all(np.abs(z_g - z_o) <= 2e-5 * np.abs(z_o) + 5e-4), (t, e)
            lp_o = float(np.sum(-0.5 * z_o * z_o - ls - 0.5 * math.log(2 * math.pi)))
            terms = float(np.sum(0.5 * z_o * z_o + np.abs(ls) + 0.5 * math.log(2 * math.pi)))
            assert abs(logp_g[t, e] - lp_o) <= 1e-5 * terms + 1e-4, (t, e)
            # integer action = map(tanh(raw)) (R#6), except exactly at a rounding boundary
            u = np.tanh(raw_g[t, e])
            a_o = np.array([oracle.map_action(x, 100) for x in u])
            off = a_g[t, e] != a_o
            if off.any():
                frac = np.abs(np.abs(u[off]) * 100 - np.floor(np.abs(u[off]) * 100) - 0.5)
                assert (frac < 1e-4).all() and (np.abs(a_g[t, e][off] - a_o[off]) == 1).all()
    # the environment driven by the GPU's executed actions: exact replay
    o = c.oracle_env()
    out = o.rollout(T, "replay", a_rep=a_g, want=("obs", "rew", "done", "hold", "cash"))
    assert_env_exact(tr, out, c.obs_dim)
    print(f"{shape}: worst mu row rel err {worst:.3e}")


def test_deterministic_mode():
    c = Case(n=30, f=3, T_data=300, N=64, H=40)
    aws, params, actor = _actor(c, 2, 128)
    tr = api.Trajectory.allocate(5, 64, 30, c.k_pad, debug=True)
    c.env.reset(c.starts)
    c.env.rollout(5, tr, actor=actor, deterministic=True)
    np.testing.assert_array_equal(tr.act.cpu().numpy(), tr.mu.cpu().numpy())
    lp = float(np.float32(np.sum(-aws[0].log_std.astype(np.float64) - 0.5 * math.log(2 * math.pi))))
    np.testing.assert_allclose(tr.logp.cpu().numpy(), lp, rtol=1e-5)


def test_multi_agent_grouping_and_ragged_tiles():
    # 3 agents x 100 envs: tiles straddle agents (100 % 128 != 0) and env tiles are ragged
    c = Case(n=30, f=3, T_data=400, N=300, H=30, n_agents=3, seed=5)
    aws, params, actor = _actor(c, 2, 128, n_agents=3)
    tr = api.Trajectory.allocate(3, 300, 30, c.k_pad, debug=True)
    c.env.reset(c.starts)
    c.env.rollout(3, tr, actor=actor)
    obs_g = bf16_to_f64(tr.obs)[..., : c.obs_dim]
    mu_g = tr.mu.cpu().numpy().astype(np.float64)
    for a in range(3):
        w = oracle.actor_flat(aws[a].W, aws[a].b, aws[a].log_std)
        for t in range(3):
            mu_o = oracle.actor_mu(w, obs_g[t, a * 100 : (a + 1) * 100], 2, 128, 30)
            mu_check(mu_g[t, a * 100 : (a + 1) * 100], mu_o)


def test_rerun_bit_identical_and_env_offset_invariance():
    # reading R#14: noise keyed on global env ids -> the same global envs give
    # bit-identical outputs whatever the split across processes/GPUs
    full = Case(n=30, f=3, T_data=400, N=64, H=20, seed=9, env_offset=0)
    aws, params, actor = _actor(full, 2, 128)
    tr1 = api.Trajectory.allocate(8, 64, 30, full.k_pad, debug=True)
    full.env.reset(full.starts)
    full.env.rollout(8, tr1, actor=actor)
    tr2 = api.Trajectory.allocate(8, 64, 30, full.k_pad, debug=True)
    full.env.reset(full.starts)
    full.env.rollout(8, tr2, actor=actor)
    for name in ("obs", "act", "logp", "rew", "done", "dbg_hold", "dbg_cash"):
        assert torch.equal(getattr(tr1, name), getattr(tr2, name)), name
    half = Case(n=30, f=3, T_data=400, N=32, H=20, seed=9, env_offset=32)
    half.starts = full.starts[1:2].copy()
    tr3 = api.Trajectory.allocate(8, 32, 30, half.k_pad, debug=True)
    half.env.reset(half.starts)
    half.env.rollout(8, tr3, actor=actor)
    for name in ("obs", "act", "logp", "rew", "done", "dbg_hold", "dbg_cash"):
        assert torch.equal(getattr(tr1, name)[:, 32:], getattr(tr3, name)), name


def test_fitness_after_deterministic_episode():
    c = Case(n=30, f=3, T_data=400, N=128, H=16, n_agents=2, gamma=0.99)
    aws, params, actor = _actor(c, 2, 128, n_agents=2)
    tr = api.Trajectory.allocate(16, 128, 30, c.k_pad, debug=True)
    fit = torch.empty(2, dtype=torch.float64, device="cuda")
    c.env.reset(c.starts)
    c.env.rollout(16, tr, actor=actor, deterministic=True, fitness_out=fit)
    assert tr.done[-1].all() and not tr.done[:-1].any()
    o = c.oracle_env()
    o.rollout(16, "replay", a_rep=tr.dbg_aint.cpu().numpy(), want=("rew",))
    _, _, _, ep = c.env.read_state()
    np.testing.assert_array_equal(ep.cpu().numpy(), o.ep_ret)
    np.testing.assert_allclose(fit.cpu().numpy(), oracle.fitness(o.ep_ret, 2), rtol=1e-12)


# ----------------------------------------------------------------- GAE
@pytest.mark.parametrize("path", ["auto", "seq", "seg"])
@pytest.mark.parametrize("T,N", [(1, 32), (3, 1), (77, 100), (50, 48), (64, 4096), (256, 8192), (1000, 96), (33, 65536),
                                 (31, 16), (512, 32), (544, 64), (640, 256)])
def test_gae_parity(T, N, path, monkeypatch):
    """Both GAE kernels (single-warp sequential scan; time-segmented block scan) against the oracle."""
    if path != "auto":
        monkeypatch.setenv("POD_GAE_PATH", path)
    r, v, d, boot = synth.gae_inputs(T, N, seed=T * 7 + N)
    adv_o, ret_o, mag = oracle.gae(r, v, d, boot, 0.99, 0.95)
    adv, ret = api.pod_gae(*(torch.from_numpy(x).cuda() for x in (r, v, d, boot)), 0.99, 0.95)
    gae_check(adv, ret, adv_o, ret_o, mag)


@pytest.mark.parametrize("path", ["seq", "seg"])
@pytest.mark.parametrize("T,N", [(256, 8192), (77, 100), (33, 4096), (5, 3)])
def test_gae_normalized_parity(T, N, path, monkeypatch):
    """R#23: per-buffer advantage normalisation fused with the scan (float64 sums) + in-place rewrite."""
    monkeypatch.setenv("POD_GAE_PATH", path)
    r, v, d, boot = synth.gae_inputs(T, N, seed=T * 3 + N)
    adv_o, ret_o, mag = oracle.gae(r, v, d, boot, 0.99, 0.95)
    an_o = oracle.gae_normalize(adv_o)
    s_o = float(np.sqrt(((adv_o - adv_o.mean()) ** 2).mean()))
    adv, ret = api.pod_gae(*(torch.from_numpy(x).cuda() for x in (r, v, d, boot)), 0.99, 0.95, normalize=True)
    an_g = adv.cpu().numpy().astype(np.float64)
    # error of A (<= 1e-5 M_t, plus the float32 rounding of A) carried through (A - m) / s
    # (the mean and the standard deviation move by at most the mean error bound, hence the (1 + |A'|) factor)
    tol = (1e-5 * mag + 1e-6 + 1e-5 * mag.mean() + 1e-6) / s_o * (1.0 + np.abs(an_o)) + 2e-6 * np.abs(an_o)
    assert np.all(np.abs(an_g - an_o) <= tol)
    np.testing.assert_allclose(ret.cpu().numpy(), ret_o, rtol=0, atol=float((1e-5 * mag + 1e-6).max()))


def test_gae_worked_example_on_gpu():
    r = torch.tensor([[1.0], [0.0], [2.0]]).cuda()
    v = torch.tensor([[0.5], [0.2], [0.1]]).cuda()
    d = torch.zeros((3, 1), dtype=torch.uint8).cuda()
    adv, ret = api.pod_gae(r, v, d, torch.zeros(1).cuda(), 0.99, 0.95)
    np.testing.assert_allclose(adv[:, 0].cpu().numpy(), [2.283635975, 1.68595, 1.9], rtol=2e-7)
    np.testing.assert_allclose(ret[:, 0].cpu().numpy(), [2.783635975, 1.88595, 2.0], rtol=2e-7)


# ----------------------------------------------------------------- selection
def test_select_elite_single_rank():
    comm = api.Comm(1, 0, 8)
    fit = torch.tensor([1.2, 3.4, 2.0, -1.0, 3.4, 0.0], dtype=torch.float64, device="cuda")
    params = torch.arange(6, dtype=torch.uint8, device="cuda")[:, None].repeat(1, 4096).contiguous()
    plan = comm.select_elite(fit, 2, params)
    ref = oracle.select_elite(fit.cpu().numpy(), 2)
    np.testing.assert_array_equal(plan, ref)
    torch.cuda.synchronize()
    got = params[:, 0].cpu().numpy()
    np.testing.assert_array_equal(got, ref)   # each slot now holds its source agent's slab
    assert (params == params[:, :1]).all()
    comm.destroy()


# ----------------------------------------------------------------- errors
def test_error_paths():
    c = Case(n=30, f=3, T_data=200, N=32, H=50)
    with pytest.raises(PodError) as ei:
        c.env.reset(np.array([150]))          # 150 + 50 > 199
    assert ei.value.name == "POD_ERR_RANGE"
    bad = api.make_config(32, 30, 3, 50, cost_rate=1.5)
    with pytest.raises(PodError) as ei:
        api.Env(bad, c.close_d, c.feat_d)
    assert ei.value.name == "POD_ERR_ARG"
    tr = api.Trajectory.allocate(2, 32, 30, c.k_pad, sampled=False)
    with pytest.raises(PodError) as ei:
        c.env.rollout(2, tr)                    # neither actor nor injected actions
    assert ei.value.name == "POD_ERR_ARG"
    cfg = api.make_config(32, 30, 3, 50)
    for bad_close, bad_feat in ((0.0, None), (float("inf"), None), (float("nan"), None), (None, float("nan"))):
        close = c.close_d.clone()
        feat = c.feat_d.clone()
        if bad_close is not None:
            close[17, 3] = bad_close                # a zero / infinite price has no unit price reciprocal
        if bad_feat is not None:
            feat[5, 1, 2] = bad_feat
        with pytest.raises(PodError) as ei:
            api.Env(cfg, close, feat)
        assert ei.value.name == "POD_ERR_NONFINITE"
    api.Env(cfg, c.close_d, c.feat_d)           # the clean market is accepted


def test_degenerate_calls():
    """Empty and degenerate inputs: a rollout of T = 0 steps and a GAE over an empty buffer are argument
    errors (nothing launched); selection with k = P keeps every slot (identity plan, slabs untouched);
    a PPO update with no minibatches only re-narrows the master into the slab it came from (unchanged)."""
    c = Case(n=30, f=3, T_data=200, N=64, H=50, seed=31)
    aws, params, actor = _actor(c, 2, 128, n_agents=2)
    tr = api.Trajectory.allocate(1, 64, 30, c.k_pad)
    c.env.reset(c.starts)
    with pytest.raises(PodError) as ei:
        c.env.rollout(0, tr, actor=actor)
    assert ei.value.name == "POD_ERR_ARG"
    z = torch.zeros((0, 64), dtype=torch.float32, device="cuda")
    with pytest.raises(PodError) as ei:
        api.pod_gae(z, z, torch.zeros((0, 64), dtype=torch.uint8, device="cuda"),
                    torch.zeros(64, device="cuda"), 0.99, 0.95)
    assert ei.value.name == "POD_ERR_ARG"
    comm = api.Comm(1, 0, 2)
    before = params.clone()
    plan = comm.select_elite(torch.tensor([0.5, 0.25], dtype=torch.float64, device="cuda"), 2, params)
    torch.cuda.synchronize()
    assert plan.tolist() == [0, 1] and torch.equal(params, before)
    comm.destroy()
    learner = api.PPOLearner(c.cfg, 2, 128, params[:1], batch=64)
    M = 64
    empty_perm = torch.zeros(0, dtype=torch.int32, device="cuda")
    learner.update(tr.obs[:1].reshape(M, c.k_pad), torch.zeros((M, 30), device="cuda"), torch.zeros(M, device="cuda"),
                   torch.zeros(M, device="cuda"), torch.zeros(M, device="cuda"), empty_perm)
    torch.cuda.synchronize()
    assert torch.equal(params, before)


# ----------------------------------------------------------------- full size (bench launch config)
@pytest.mark.parametrize("agents", [1, 8])
def test_full_size_c3_sampled_rows(agents):
    """C3 launch configuration (8192 envs, n=100, 3x512, one agent) on sampled rows; with 8 agents, C4's
    (8 x 1,024 envs: agent switches between the clusters' tiles)."""
    c = Case(n=100, f=3, T_data=60_000, N=8192, H=2000, n_agents=agents, seed=5191, dt=1 / (252 * 390))
    aws, params, actor = _actor(c, 3, 512, n_agents=agents)
    T = 4
    tr = api.Trajectory.allocate(T, c.N, c.n, c.k_pad, debug=True)
    c.env.reset(c.starts)
    c.env.rollout(T, tr, actor=actor)
    c.env.check()
    rows = np.unique(np.concatenate([np.arange(0, 8192, 257), [8191, 127, 128, 1023, 1024, 4095, 4096]]))
    obs_g = bf16_to_f64(tr.obs)[..., : c.obs_dim]
    mu_g = tr.mu.cpu().numpy().astype(np.float64)
    raw_g = tr.act.cpu().numpy().astype(np.float64)
    logp_g = tr.logp.cpu().numpy().astype(np.float64)
    per = 8192 // agents
    for t in range(T):
        for a in range(agents):
            ra = rows[(rows >= a * per) & (rows < (a + 1) * per)]
            w = oracle.actor_flat(aws[a].W, aws[a].b, aws[a].log_std)
            mu_check(mu_g[t, ra], oracle.actor_mu(w, obs_g[t, ra], 3, 512, 100))
        # noise (Philox, drawn by the previous env step) and the log-prob (partials summed by the env step)
        for e in rows:
            ls = aws[int(e) // per].log_std.astype(np.float64)
            z_o = oracle.normals(c.cfg.seed, c.cfg.env_offset + int(e), t, 100)
            z_g = (raw_g[t, e] - mu_g[t, e]) / np.exp(ls)
            assert np.all(np.abs(z_g - z_o) <= 2e-5 * np.abs(z_o) + 5e-4), (t, e)
            lp_o = float(np.sum(-0.5 * z_o * z_o - ls - 0.5 * math.log(2 * math.pi)))
            terms = float(np.sum(0.5 * z_o * z_o + np.abs(ls) + 0.5 * math.log(2 * math.pi)))
            assert abs(logp_g[t, e] - lp_o) <= 1e-5 * terms + 1e-4, (t, e)
    # env replay on the sampled envs (envs are independent: batch equivalence)
    a_g = tr.dbg_aint.cpu().numpy()
    starts = c.env_starts()[rows]
    o = oracle.Env(c.market.close, c.market.feat, len(rows), **dict(c.kw, n_agents=1))
    o.reset(starts)
    out = o.rollout(T, "replay", a_rep=np.ascontiguousarray(a_g[:, rows]), want=("obs", "rew", "done", "hold", "cash"))
    np.testing.assert_array_equal(tr.dbg_hold.cpu().numpy()[:, rows], out["hold"])
    np.testing.assert_array_equal(tr.dbg_cash.cpu().numpy()[:, rows], out["cash"])
    np.testing.assert_array_equal(tr.rew.cpu().numpy()[:, rows], out["rew"].astype(np.float32))
    assert_obs_close(tr.obs[:, rows], out["obs"], c.obs_dim)
    # properties over all rows
    assert (tr.dbg_cash >= 0).all() and (tr.dbg_hold >= 0).all()


def test_full_size_c2_sampled_rows():
    """C2 launch configuration (Dow-30 daily, 4,096 envs, 2x128, H = 1,024: the env step launched as a
    programmatic dependent of the actor, whose 32 M-tiles leave most SMs idle) on sampled rows, T = 6."""
    c = Case(n=30, f=3, T_data=2611, N=4096, H=1024, seed=5190)
    aws, params, actor = _actor(c, 2, 128)
    T = 6
    tr = api.Trajectory.allocate(T, c.N, c.n, c.k_pad, debug=True, critic=True)
    c.env.reset(c.starts)
    c.env.rollout(T, tr, actor=actor)
    c.env.check()
    rows = np.unique(np.concatenate([np.arange(0, 4096, 131), [4095, 31, 32, 127, 128, 2047, 2048]]))
    obs_g = bf16_to_f64(tr.obs)[:, rows, : c.obs_dim]
    mu_g = tr.mu.cpu().numpy()[:, rows].astype(np.float64)
    val_g = tr.val.cpu().numpy()[:, rows].astype(np.float64)
    w = oracle.actor_flat(aws[0].W, aws[0].b, aws[0].log_std)
    for t in range(T):
        mu_check(mu_g[t], oracle.actor_mu(w, obs_g[t], 2, 128, 30))
        v_o = oracle.actor_value(aws[0].W, aws[0].b, aws[0].w_v, aws[0].b_v, obs_g[t], 2, 128)
        v_abs = np.abs(oracle.actor_value(aws[0].W, aws[0].b, np.abs(aws[0].w_v), abs(aws[0].b_v), obs_g[t], 2, 128))
        rms = math.sqrt(float(np.mean(v_o ** 2)))
        assert np.all(np.abs(val_g[t] - v_o) <= 2e-2 * (np.abs(v_o) + rms) + 1e-2 * v_abs + 1e-6), t
    a_g = tr.dbg_aint.cpu().numpy()
    o = oracle.Env(c.market.close, c.market.feat, len(rows), **c.kw)
    o.reset(c.env_starts()[rows])
    out = o.rollout(T, "replay", a_rep=np.ascontiguousarray(a_g[:, rows]), want=("obs", "rew", "done", "hold", "cash"))
    np.testing.assert_array_equal(tr.dbg_hold.cpu().numpy()[:, rows], out["hold"])
    np.testing.assert_array_equal(tr.dbg_cash.cpu().numpy()[:, rows], out["cash"])
    np.testing.assert_array_equal(tr.rew.cpu().numpy()[:, rows], out["rew"].astype(np.float32))
    np.testing.assert_array_equal(tr.done.cpu().numpy()[:, rows], out["done"])
    assert_obs_close(tr.obs[:, rows], out["obs"], c.obs_dim)


@pytest.mark.parametrize("agents", [1, 8])
def test_full_size_c5_sampled_rows(agents):
    """C5 launch configuration (65,536 envs, n = 100, 3x512, default switches): the dense programmatic-
    dependent env-step launch (2,048 tiles >= 7 per SM) and the persistent actor (512 M-tiles on 74 clusters,
    ~7 tiles per cluster: barrier phases and TMEM buffers wrap around) against the oracle on sampled rows from
    the first wave, the second wave and the last persistent tiles of each cluster; agents = 8 switches agent
    inside the persistent loop (C4's population shape)."""
    N = 65536
    c = Case(n=100, f=3, T_data=60_000, N=N, H=3000, n_agents=agents, seed=5193, dt=1 / (252 * 390))
    aws, params, actor = _actor(c, 3, 512, n_agents=agents)
    T = 4
    tr = api.Trajectory.allocate(T, c.N, c.n, c.k_pad, debug=True)
    c.env.reset(c.starts)
    c.env.rollout(T, tr, actor=actor)
    c.env.check()
    # M-tiles (128 envs): 0 and 73 (first wave), 74 and 147 (second wave), 438..511 (the last tile of every
    # persistent cluster), plus env tiles (32 envs) at both ends of the PDL grid
    mt = [0, 73, 74, 147, 148, 300, 438, 480, 510, 511]
    rows = np.unique(np.concatenate([[m * 128 + o for m in mt for o in (0, 45, 127)], [31, 32, 65503, 65535]]))
    obs_g = bf16_to_f64(tr.obs)[:, rows, : c.obs_dim]
    mu_g = tr.mu.cpu().numpy()[:, rows].astype(np.float64)
    raw_g = tr.act.cpu().numpy()[:, rows].astype(np.float64)
    logp_g = tr.logp.cpu().numpy()[:, rows].astype(np.float64)
    per_agent = N // agents
    for t in range(T):
        for k, e in enumerate(rows):
            aw = aws[int(e) // per_agent]
            w = oracle.actor_flat(aw.W, aw.b, aw.log_std)
            ls = aw.log_std.astype(np.float64)
            mu_check(mu_g[t, k][None, :], oracle.actor_mu(w, obs_g[t, k][None, :], 3, 512, 100))
            z_o = oracle.normals(c.cfg.seed, c.cfg.env_offset + int(e), t, 100)
            z_g = (raw_g[t, k] - mu_g[t, k]) / np.exp(ls)
            assert np.all(np.abs(z_g - z_o) <= 2e-5 * np.abs(z_o) + 5e-4), (t, e)
            lp_o = float(np.sum(-0.5 * z_o * z_o - ls - 0.5 * math.log(2 * math.pi)))
            terms = float(np.sum(0.5 * z_o * z_o + np.abs(ls) + 0.5 * math.log(2 * math.pi)))
            assert abs(logp_g[t, k] - lp_o) <= 1e-5 * terms + 1e-4, (t, e)
    a_g = tr.dbg_aint.cpu().numpy()
    o = oracle.Env(c.market.close, c.market.feat, len(rows), **dict(c.kw, n_agents=1))
    o.reset(c.env_starts()[rows])
    out = o.rollout(T, "replay", a_rep=np.ascontiguousarray(a_g[:, rows]), want=("obs", "rew", "done", "hold", "cash"))
    np.testing.assert_array_equal(tr.dbg_hold.cpu().numpy()[:, rows], out["hold"])
    np.testing.assert_array_equal(tr.dbg_cash.cpu().numpy()[:, rows], out["cash"])
    np.testing.assert_array_equal(tr.rew.cpu().numpy()[:, rows], out["rew"].astype(np.float32))
    np.testing.assert_array_equal(tr.done.cpu().numpy()[:, rows], out["done"])
    assert_obs_close(tr.obs[:, rows], out["obs"], c.obs_dim)
    assert (tr.dbg_cash >= 0).all() and (tr.dbg_hold >= 0).all()
    assert torch.isfinite(tr.mu).all() and torch.isfinite(tr.logp).all()


@pytest.mark.parametrize("where", ["head_bias", "hidden_weight"])
def test_nonfinite_weights_set_error_word(where):
    """S:L288 / §8(b): a non-finite actor mean sets the device error word; pod_env_check reports
    POD_ERR_NONFINITE (and clears it), and a later pod_rollout on the flagged state refuses to run with
    POD_ERR_NONFINITE until the word is cleared; pod_env_reset also clears it."""
    c = Case(n=30, f=3, T_data=400, N=256, H=50, seed=71)
    aws, params, actor = _actor(c, 2, 128)
    L = api.actor_layout(c.cfg, 2, 128)
    raw = params.view(torch.uint8)
    if where == "head_bias":
        off = L.b_offset[L.n_layers - 1] + 4 * 3   # b_L[3] = NaN: mu_3 of every env
        raw[0, off : off + 4] = torch.tensor([0, 0, 192, 127], dtype=torch.uint8)
    else:
        off = L.w_offset[1]   # W_1[0][0] = +inf (bf16 0x7F80): propagates to the mean through the head
        raw[0, off : off + 2] = torch.tensor([128, 127], dtype=torch.uint8)
    tr = api.Trajectory.allocate(3, c.N, c.n, c.k_pad)
    c.env.reset(c.starts)
    c.env.rollout(3, tr, actor=actor)
    with pytest.raises(PodError) as ei:
        c.env.check()
    assert ei.value.status == 7
    c.env.check()   # cleared
    # the next rollout after a flagged one (completed on the device) refuses to run
    c.env.rollout(1, tr, actor=actor)
    torch.cuda.synchronize()
    with pytest.raises(PodError) as ei:
        c.env.rollout(1, tr, actor=actor)
    assert ei.value.status == 7
    # reset clears the word; with finite weights the rollout is accepted again
    _, params2, actor2 = _actor(c, 2, 128)
    c.env.reset(c.starts)
    c.env.rollout(2, tr, actor=actor2)
    torch.cuda.synchronize()
    c.env.rollout(2, tr, actor=actor2)
    c.env.check()


def test_profile_events_in_graph():
    c = Case(n=30, f=3, T_data=300, N=256, H=40)
    aws, params, actor = _actor(c, 2, 128)
    tr = api.Trajectory.allocate(6, 256, 30, c.k_pad)
    c.env.reset(c.starts)
    for stride, marked in ((1, 6), (4, 2)):
        c.env.profile(stride)
        for _ in range(2):   # capture, then replay
            c.env.rollout(6, tr, actor=actor)
            am, an, em, en = c.env.profile_read()
            assert abs(an - marked) < 1e-9 and abs(en - marked) < 1e-9 and am > 0 and em > 0
        assert c.env.profile_read() == (0.0, 0.0, 0.0, 0.0)
    c.env.profile(0)


def test_env_groups_bit_identical(monkeypatch):
    """Running the envs as 1, 2 or 4 independent graph branches changes nothing."""
    outs = []
    for G in ("1", "2", "4"):
        monkeypatch.setenv("POD_GROUPS", G)
        c = Case(n=30, f=3, T_data=400, N=512, H=20, seed=12)
        aws, params, actor = _actor(c, 2, 128)
        tr = api.Trajectory.allocate(7, 512, 30, c.k_pad, debug=True)
        c.env.reset(c.starts)
        c.env.rollout(7, tr, actor=actor)
        c.env.check()
        outs.append(tr)
    for other in outs[1:]:
        for name in ("obs", "act", "logp", "rew", "done", "dbg_hold", "dbg_cash", "dbg_aint"):
            assert torch.equal(getattr(outs[0], name), getattr(other, name)), name


@pytest.mark.parametrize("n,N,nh,hid", [(30, 512, 2, 128), (100, 36864, 3, 512)])
def test_pdl_env_launch_bit_identical(n, N, nh, hid, monkeypatch):
    """The env step launched as a programmatic dependent of the actor (griddepcontrol; default where it
    pays: a small launch whose tiles fit the idle SMs, N = 512, or a dense one, >= 7 tiles per SM, N =
    36864 at the C3 actor shape) is bit-identical to the plain stream order (POD_PDL=0), including the
    critic values and the next-step noise the env step writes while the actor grid may still run."""
    outs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("POD_PDL", flag)
        c = Case(n=n, f=3, T_data=600, N=N, H=50, seed=14)
        aws, params, actor = _actor(c, nh, hid)
        tr = api.Trajectory.allocate(3, N, n, c.k_pad, debug=True, critic=True)
        c.env.reset(c.starts)
        c.env.rollout(3, tr, actor=actor)
        c.env.check()
        torch.cuda.synchronize()
        outs.append(tr)
    for name in ("obs", "act", "logp", "rew", "done", "dbg_hold", "dbg_cash", "dbg_aint", "val"):
        assert torch.equal(getattr(outs[0], name), getattr(outs[1], name)), name


@pytest.mark.parametrize("n,N,agents,nh,hid", [(30, 512, 2, 2, 128), (100, 256, 1, 3, 512), (100, 20480, 1, 3, 512)])
def test_weight_retile_bit_identical(n, N, agents, nh, hid, monkeypatch):
    """The actor weights re-tiled per rollout into ring-stage order and streamed by 1-D bulk copies (default)
    against the 2-D tensor-map boxes (POD_WT=0): every output bit-identical, in the fused kernel (N <= 9472 at
    these shapes) and in the separate persistent actor (N = 20480: 160 M-tiles)."""
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("POD_WT", flag)
        c = Case(n=n, f=3, T_data=600, N=N, H=6, n_agents=agents, seed=16)
        aws, params, actor = _actor(c, nh, hid, n_agents=agents)
        tr = api.Trajectory.allocate(4, N, n, c.k_pad, debug=True, critic=True)
        c.env.reset(c.starts)
        c.env.rollout(4, tr, actor=actor)
        c.env.check()
        torch.cuda.synchronize()
        outs.append(tr)
    for name in ("obs", "act", "logp", "mu", "rew", "done", "dbg_hold", "dbg_cash", "dbg_aint", "val"):
        x, y = getattr(outs[0], name), getattr(outs[1], name)
        if x.dtype == torch.bfloat16:
            x, y = x.view(torch.int16), y.view(torch.int16)
        assert torch.equal(x, y), name


@pytest.mark.parametrize("n,N,agents,nh,hid,det", [(1, 256, 1, 1, 128, False), (7, 384, 3, 1, 128, False),
                                                   (64, 512, 1, 2, 256, False),
                                                   (30, 512, 1, 2, 128, False), (30, 4096, 1, 2, 128, True),
                                                   (100, 8192, 1, 3, 512, False), (100, 8192, 8, 3, 512, False),
                                                   (100, 2048, 2, 3, 512, True)])
def test_fused_rollout_bit_identical(n, N, agents, nh, hid, det, monkeypatch):
    """The fused rollout kernel (one cluster per 128-env M-tile runs the actor and the env step of its envs for
    all T steps, rollout_fused_kernel; the default where it fits one wave) against the separate actor and
    env-step launches (POD_FUSED=0): every trajectory output — observations, actions, log-probs, mean
    actions, rewards, done flags, holdings, cash, equity, critic values including the bootstrap V(s_T) —
    and the env state left for the next rollout are bit-identical, over chained rollouts of 7, 7, 1 and 2 steps
    with episode resets inside them (H = 5)."""
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("POD_FUSED", flag)
        c = Case(n=n, f=3, T_data=600, N=N, H=5, n_agents=agents, seed=15)
        aws, params, actor = _actor(c, nh, hid, n_agents=agents)
        res = []
        c.env.reset(c.starts)
        # rollouts of 7, 1 and 2 steps, with and without the critic (the fused kernel's iteration T is the
        # bootstrap pass only with it)
        for T, critic in ((7, True), (7, True), (1, True), (2, False)):
            tr = api.Trajectory.allocate(T, N, n, c.k_pad, debug=True, critic=critic, equity=True)
            k0 = api.kernel_launches()
            c.env.rollout(T, tr, actor=actor, deterministic=det)
            torch.cuda.synchronize()
            if T == 7:   # the fused path is one launch for the steps (plus obs_0, the weight re-tiling, the bump)
                assert (api.kernel_launches() - k0 < T) == (flag == "1"), "unexpected rollout path"
            res.append({k: v.clone() for k, v in vars(tr).items() if v is not None})
        res.append(dict(zip(("hold", "cash", "asset", "ep_ret"), c.env.read_state())))
        c.env.check()
        outs.append(res)
    for a, b in zip(*outs):
        assert a.keys() == b.keys()
        for k in a:
            x, y = a[k], b[k]
            if x.dtype == torch.bfloat16:
                x, y = x.view(torch.int16), y.view(torch.int16)
            assert torch.equal(x, y), k


@pytest.mark.parametrize("cost", [0.0, 0.25, 0.002])
@pytest.mark.parametrize("kind", ["all_buy", "uniform", "buy_then_sell"])
def test_exact_quotient_ties(kind, cost):
    """Integer prices and capital make b/unit land exactly on integers: exercises the
    ledger's division fallback, the post-check and both exact shortcuts."""
    rng = np.random.default_rng(17)
    n, T_data, N, H, T = 8, 60, 64, 40, 40
    prices = rng.choice([1.0, 2.0, 4.0, 5.0, 8.0, 10.0, 20.0, 25.0, 50.0], size=(T_data, n))
    m = synth.make_flat_market(n, T_data, prices, n_feat=1)
    cfg = api.make_config(N, n, 1, H, 1, 100, 0, 1000.0, cost, 1.0, 0.99, 3)
    env = api.Env(cfg, torch.from_numpy(m.close).cuda(), torch.from_numpy(m.feat).cuda())
    starts = np.array([0, 7], np.int64)
    u = synth.injected_u(kind, T, N, n, 4)
    tr = api.Trajectory.allocate(T, N, n, env.k_pad, debug=True, sampled=False)
    env.reset(starts)
    env.rollout(T, tr, injected_u=torch.from_numpy(u).cuda())
    o = oracle.Env(m.close, m.feat, N, horizon=H, C0=1000.0, cost=cost, seed=3)
    o.reset(np.repeat(starts, 32)[:N])
    out = o.rollout(T, "inject", u=u, want=("obs", "rew", "done", "hold", "cash"))
    assert_env_exact(tr, out, env.obs_dim)


@pytest.mark.parametrize("mcg", ["1", "4"])
def test_weight_multicast_bit_identical(mcg, monkeypatch):
    """Opt-in clusters sharing weight tiles by TMA multicast (POD_MULTICAST=1: two M-tiles in 4-CTA
    clusters; 4: four M-tiles in 8-CTA clusters) give identical results."""
    outs = []
    for mc in ("0", mcg):
        monkeypatch.setenv("POD_MULTICAST", mc)
        c = Case(n=100, f=3, T_data=2000, N=512, H=300, seed=13, dt=1 / (252 * 390))
        aws, params, actor = _actor(c, 3, 512)
        tr = api.Trajectory.allocate(4, 512, 100, c.k_pad, debug=True)
        c.env.reset(c.starts)
        c.env.rollout(4, tr, actor=actor)
        c.env.check()
        outs.append(tr)
    for name in ("obs", "act", "logp", "rew", "done", "dbg_hold", "dbg_cash", "mu"):
        assert torch.equal(getattr(outs[0], name), getattr(outs[1], name)), name


@pytest.mark.parametrize("n,nh,hid", [(100, 3, 512), (30, 2, 128), (32, 2, 256)])
def test_critic_value_parity(n, nh, hid):
    """R#22: V(s_t) = head row n over the trunk, written per step; V(s_T) by the value-only pass.
    Compared with the oracle's float64 forward on the GPU's own bf16 observations (the actor bar);
    the actor's own outputs are bit-identical with and without the critic output."""
    outs = []
    for critic in (False, True):
        c = Case(n=n, f=3, T_data=600, N=256, H=7, seed=31)
        aws, params, actor = _actor(c, nh, hid)
        tr = api.Trajectory.allocate(9, c.N, c.n, c.k_pad, debug=True, critic=critic)
        c.env.reset(c.starts)
        c.env.rollout(9, tr, actor=actor)
        c.env.check()
        outs.append(tr)
    for name in ("obs", "act", "logp", "mu", "rew", "done", "dbg_hold"):
        assert torch.equal(getattr(outs[0], name), getattr(outs[1], name)), name
    tr = outs[1]
    obs_g = bf16_to_f64(tr.obs)[..., : c.obs_dim]
    val_g = tr.val.cpu().numpy().astype(np.float64)
    aw = aws[0]
    for t in range(10):
        v_o = oracle.actor_value(aw.W, aw.b, aw.w_v, aw.b_v, obs_g[t], nh, hid)
        rms = math.sqrt(float(np.mean(v_o ** 2)))
        assert np.all(np.abs(val_g[t] - v_o) <= 2e-2 * (np.abs(v_o) + rms)), t
    # the device values feed GAE directly (bootstrap = val[T])
    adv, ret = api.pod_gae(tr.rew, tr.val[:-1].contiguous(), tr.done, tr.val[-1].contiguous(), 0.99, 0.95)
    adv_o, ret_o, mag = oracle.gae(tr.rew.cpu().numpy(), val_g[:-1], tr.done.cpu().numpy(), val_g[-1], 0.99, 0.95)
    gae_check(adv, ret, adv_o, ret_o, mag)


def test_critic_deterministic_and_graph_reuse():
    """Critic output in deterministic mode, and across repeated (graph-cached) rollouts."""
    c = Case(n=30, f=3, T_data=400, N=96, H=50, seed=32)
    aws, params, actor = _actor(c, 2, 128)
    tr = api.Trajectory.allocate(4, c.N, c.n, c.k_pad, critic=True)
    c.env.reset(c.starts)
    vals = []
    for _ in range(3):
        c.env.rollout(4, tr, actor=actor, deterministic=True)
        vals.append(tr.val.clone())
    obs_g = bf16_to_f64(tr.obs)[..., : c.obs_dim]
    v_o = np.stack([oracle.actor_value(aws[0].W, aws[0].b, aws[0].w_v, aws[0].b_v, obs_g[t], 2, 128) for t in range(5)])
    rms = math.sqrt(float(np.mean(v_o ** 2)))
    assert np.all(np.abs(vals[-1].cpu().numpy() - v_o) <= 2e-2 * (np.abs(v_o) + rms))
    assert not torch.equal(vals[0], vals[1])   # the envs moved on between calls


def _slab_flat(slab: np.ndarray, L) -> np.ndarray:
    """Widen one parameter slab (bf16 weights, f32 biases / log-std) to the float64 flat vector of
    pod_actor_layout order (W_0..W_L, b_0..b_L, log_std)."""
    parts = []
    for l in range(L.n_layers):
        n = L.w_rows[l] * L.w_cols[l]
        raw = slab[L.w_offset[l] : L.w_offset[l] + 2 * n].view(np.uint16).astype(np.uint32) << 16
        parts.append(raw.view(np.float32).astype(np.float64))
    for l in range(L.n_layers):
        parts.append(slab[L.b_offset[l] : L.b_offset[l] + 4 * L.w_rows[l]].view(np.float32).astype(np.float64))
    parts.append(slab[L.log_std_offset : L.log_std_offset + 4 * L.n_out_pad].view(np.float32).astype(np.float64))
    return np.concatenate(parts)


@pytest.mark.parametrize("tau", [1.0, 0.3, 0.0])
def test_fuse_pods_parity(tau):
    """R#24: K_local = 4 pods of 2 agents on one GPU; every pod's slab <- narrow(tau mean + (1-tau) prev),
    prev <- the float32 fused vector; compared with the float64 oracle (bf16 weights within one bf16 ulp,
    float32 entries within 2 ulp), all pods of an agent bit-identical."""
    c = Case(n=30, f=3, T_data=300, N=64, H=20)
    nh, hid, K, A = 2, 128, 4, 2
    aws = [synth.make_actor(c.obs_dim, nh, hid, c.n, 100 + s) for s in range(K * A)]
    params = api.pack_actor_params(c.cfg, aws, nh, hid)
    L = api.actor_layout(c.cfg, nh, hid)
    E = int(L.n_elems)
    before = params.cpu().numpy()
    flats = np.stack([_slab_flat(before[s], L) for s in range(K * A)])
    prev0 = torch.from_numpy(np.random.default_rng(9).normal(size=(A, E)).astype(np.float32)).cuda()
    prev = prev0.clone() if tau != 1.0 else None
    api.fuse_pods(c.cfg, nh, hid, params, K, tau=tau, prev=prev)
    after = params.cpu().numpy()
    nw = sum(L.w_rows[l] * L.w_cols[l] for l in range(L.n_layers))
    for a in range(A):
        exp = oracle.fuse(flats[a * K : (a + 1) * K], prev0[a].cpu().numpy().astype(np.float64), tau)
        for k in range(K):
            assert np.array_equal(after[a * K + k], after[a * K]), (a, k)
        got = _slab_flat(after[a * K], L)
        # float32 sum + blend: a few roundings relative to the magnitudes involved; bf16: one more ulp
        mag = tau * np.abs(flats[a * K : (a + 1) * K]).mean(axis=0) + (1.0 - tau) * np.abs(prev0[a].cpu().numpy())
        tol32 = 8.0 * 2.0 ** -24 * mag
        assert np.all(np.abs(got[:nw] - exp[:nw]) <= np.abs(exp[:nw]) * 2.0 ** -8 + 2.0 * tol32[:nw]), a
        assert np.all(np.abs(got[nw:] - exp[nw:]) <= tol32[nw:]), a
        if prev is not None:
            assert np.all(np.abs(prev[a].cpu().numpy() - exp) <= tol32), a
    # the fused actor still runs
    actor = api.make_actor(nh, hid, params)
    tr = api.Trajectory.allocate(2, c.N, c.n, c.k_pad)
    c.env.reset(c.starts)
    c.env.rollout(2, tr, actor=actor)
    c.env.check()


@pytest.mark.parametrize("R,tau", [(2, 1.0), (4, 0.3), (3, 0.0)])
def test_fuse_pods_local_ranks_exchange(R, tau):
    """R#24, the cross-rank fusion kernel: R ranks' slab arrays (K_local = 2 pods of 2 agents each) fused in one
    launch whose block rows play the ranks and exchange partial sums through flags and staging buffers as
    pod_fuse_pods' ranks do over peer memory.  Every pod of an agent on every rank ends bit-identical, and equal
    to the float64 oracle over all R x K_local pods within the fusion bars; prev likewise."""
    c = Case(n=30, f=3, T_data=300, N=64, H=20)
    nh, hid, K, A = 2, 128, 2, 2
    L = api.actor_layout(c.cfg, nh, hid)
    E = int(L.n_elems)
    params = [api.pack_actor_params(c.cfg, [synth.make_actor(c.obs_dim, nh, hid, c.n, 300 + 10 * r + s)
                                            for s in range(K * A)], nh, hid) for r in range(R)]
    before = [p.cpu().numpy() for p in params]
    prev0 = torch.from_numpy(np.random.default_rng(19).normal(size=(A, E)).astype(np.float32)).cuda()
    prevs = [prev0.clone() for _ in range(R)] if tau != 1.0 else None
    api.fuse_pods_local_ranks(c.cfg, nh, hid, params, K, tau=tau, prevs=prevs)
    torch.cuda.synchronize()
    after = [p.cpu().numpy() for p in params]
    nw = sum(L.w_rows[l] * L.w_cols[l] for l in range(L.n_layers))
    for a in range(A):
        ref = after[0][a * K]
        for r in range(R):
            for k in range(K):
                assert np.array_equal(after[r][a * K + k], ref), (a, r, k)
        flats = np.stack([_slab_flat(before[r][a * K + k], L) for r in range(R) for k in range(K)])
        exp = oracle.fuse(flats, prev0[a].cpu().numpy().astype(np.float64), tau)
        got = _slab_flat(ref, L)
        mag = tau * np.abs(flats).mean(axis=0) + (1.0 - tau) * np.abs(prev0[a].cpu().numpy())
        tol32 = 8.0 * 2.0 ** -24 * mag
        assert np.all(np.abs(got[:nw] - exp[:nw]) <= np.abs(exp[:nw]) * 2.0 ** -8 + 2.0 * tol32[:nw]), a
        assert np.all(np.abs(got[nw:] - exp[nw:]) <= tol32[nw:]), a
        if prevs is not None:
            for r in range(R):
                np.testing.assert_array_equal(prevs[r][a].cpu().numpy(), prevs[0][a].cpu().numpy())
            assert np.all(np.abs(prevs[0][a].cpu().numpy() - exp) <= tol32), a
    if (R * K) & (R * K - 1):
        return
    # a second call (fresh flags) over identical pods: with a power-of-two pod count the float32 mean is exact
    snap = [p.clone() for p in params]
    api.fuse_pods_local_ranks(c.cfg, nh, hid, params, K, tau=1.0)
    torch.cuda.synchronize()
    for r in range(R):
        assert torch.equal(params[r], snap[r])


def test_equity_curve_exact_and_backtest_metrics():
    """R#25: traj.equity (v_{t+1} after each step) equals the oracle's float64 account value bit for bit;
    the device backtest metrics of those curves match the oracle's metric definitions."""
    c = Case(n=30, f=3, T_data=400, N=96, H=300, seed=41)
    T = 60
    u = synth.injected_u("uniform", T, c.N, c.n, 5)
    tr = api.Trajectory.allocate(T, c.N, c.n, c.k_pad, sampled=False, equity=True)
    c.env.reset(c.starts)
    _, _, v0, _ = c.env.read_state()
    c.env.rollout(T, tr, injected_u=torch.from_numpy(u).cuda())
    o = c.oracle_env()
    out = o.rollout(T, "inject", u=u, want=("asset",))
    np.testing.assert_array_equal(tr.equity.cpu().numpy(), out["asset"])
    m = api.backtest_metrics(v0, tr.equity, 252.0).cpu().numpy()
    curves = np.concatenate([v0.cpu().numpy()[None, :], out["asset"]], axis=0)
    for e in range(c.N):
        cv = curves[:, e]
        ann, vol = oracle.annual_return_volatility(cv, 252.0)
        exp = [oracle.cumulative_return(cv), ann, vol, oracle.sharpe(cv, 252.0), oracle.max_drawdown(cv)]
        np.testing.assert_allclose(m[:, e], exp, rtol=1e-11, atol=1e-13, equal_nan=True)
    # degenerate curve: constant value -> zero return / volatility / drawdown, Sharpe NaN
    flat = torch.full((5, 3), 7.0, dtype=torch.float64, device="cuda")
    mf = api.backtest_metrics(torch.full((3,), 7.0, dtype=torch.float64, device="cuda"), flat, 252.0).cpu().numpy()
    assert np.all(mf[[0, 1, 2, 4]] == 0.0) and np.all(np.isnan(mf[3]))


def _ppo_case(n, nh, hid, act, seed=51, N=256, T=8):
    c = Case(n=n, f=3, T_data=400, N=N, H=100, seed=seed)   # n = 64: the critic row in a fresh pad block
    aws, params, actor = _actor(c, nh, hid, act=act)
    tr = api.Trajectory.allocate(T, c.N, c.n, c.k_pad, critic=True)
    c.env.reset(c.starts)
    c.env.rollout(T, tr, actor=actor)
    adv, ret = api.pod_gae(tr.rew, tr.val[:T].contiguous(), tr.done, tr.val[T].contiguous(), 0.99, 0.95,
                           normalize=True)
    M = T * c.N
    args = (tr.obs[:T].reshape(M, c.k_pad), tr.act.reshape(M, c.n), tr.logp.reshape(M), adv.reshape(M), ret.reshape(M))
    return c, params, args, M


def _ppo_segments(L):
    segs, o = [], 0
    for l in range(L.n_layers):
        segs.append((o, o + L.w_rows[l] * L.w_cols[l]))
        o += L.w_rows[l] * L.w_cols[l]
    for l in range(L.n_layers):
        segs.append((o, o + L.w_rows[l]))
        o += L.w_rows[l]
    segs.append((o, o + L.n_out_pad))
    return segs


# PPO gradient bars (R#26/R#27), per parameter segment (W_l, b_l, log_std); m = the oracle's
# magnitude of each entry (the sum of the absolute values of the terms it is summed from):
#   float32 mode vs the float64 oracle:                 ||g-o|| <= 2e-4 ||o||, |g-o| <= 2e-3 (|o| + rms(o))
#   bf16 mode vs the oracle with bf16 operand rounding: ||g-o|| <= 2e-3 ||o||; |g-o| <= 1e-2 m for every entry
#                                                       with tanh; with ReLU for >= 97 % of a segment's entries
#                                                       and |g-o| <= 0.5 m for all
#   bf16 mode vs the plain float64 oracle:              ||g-o|| <= 3e-2 ||o||   (operand rounding moves rho)
# (ReLU: where a pre-activation lies within rounding of 0 the two sides can take opposite derivatives: the
# gradient entries of that unit pick up or lose a whole term — a large share of m for a rarely active unit —
# and the changed delta spreads, at a small scale, into every unit of the layers below; tanh has no such
# discontinuity, so its bar holds for every entry.  Measured at the C3 actor: <= 2.5 % of W_0's entries
# beyond 1e-2 m, the largest 0.24 m, in W_1.)
@pytest.mark.parametrize("fp32", [True, False])
@pytest.mark.parametrize("act,B,n,nh,hid", [(0, 512, 30, 2, 128), (1, 512, 30, 2, 128), (0, 1001, 30, 2, 128),
                                            (0, 512, 64, 1, 256), (1, 384, 30, 4, 128), (0, 1024, 100, 3, 512)])
def test_ppo_update_parity(act, B, n, nh, hid, fp32):
    """R#26: one PPO minibatch on the device buffers of a rollout (critic values, normalised GAE): the
    gradient of this library's learner (tcgen05 GEMMs in bf16 mode, the float32 core in fp32 mode, the same
    epilogues and reductions) vs the float64 oracle's analytic gradient at the same parameters on the same
    rows; the loss sums; the Adam step; the refreshed slab.  B = 1001 is ragged in every tile (128-row GEMM
    tiles, 8-sample head blocks); (100, 3, 512) is the C3 actor."""
    c, params, args, M = _ppo_case(n, nh, hid, act, N=256 if n < 100 else 512)
    obs, act_raw, lpo, A, R = args
    lr = 1e-3
    learner = api.PPOLearner(c.cfg, nh, hid, params, act=act, batch=B, learning_rate=lr, fp32=fp32)
    theta0 = learner.master.cpu().numpy().astype(np.float64)
    rows = np.random.default_rng(3).permutation(M)[:B].astype(np.int32)
    g_gpu = torch.empty(learner.n_elems, dtype=torch.float32, device="cuda")
    losses = learner.update(obs, act_raw, lpo, A, R, torch.from_numpy(rows).cuda(), grad_out=g_gpu)
    learner.check()
    L = api.actor_layout(c.cfg, nh, hid)
    dims = (L.k_pad, hid, nh, c.n, L.n_out_pad)
    oargs = (dims, bf16_to_f64(obs[rows]), act_raw[rows].cpu().numpy(), lpo[rows].cpu().numpy(),
             A[rows].cpu().numpy(), R[rows].cpu().numpy(), 0.25, 0.02, 0.5, act)
    _, g_o, (sobj, svl, H), m_o = oracle.ppo_loss_grad(theta0, *oargs, magnitudes=True)
    _, g_e, (sobj_e, svl_e, _), m_e = oracle.ppo_loss_grad(theta0, *oargs, bf16_operands=True, magnitudes=True)
    g_g = g_gpu.cpu().numpy().astype(np.float64)
    ref, mag, nb = (g_o, m_o, 2e-4) if fp32 else (g_e, m_e, 2e-3)
    for si, (a0, a1) in enumerate(_ppo_segments(L)):
        o = ref[a0:a1]
        d = g_g[a0:a1] - o
        rel = np.linalg.norm(d) / (np.linalg.norm(o) + 1e-30)
        assert rel <= nb, (a0, a1, rel)
        if not fp32:
            r = np.abs(d) / (mag[a0:a1] + 1e-30)
            r[np.abs(d) <= 1e-9] = 0.0
            frac = float((r > 1e-2).mean())
            assert frac <= (0.0 if act == 1 else 0.03), (si, frac, float(r.max()))
            assert r.max() <= 0.5, (si, float(r.max()))
        else:
            rms = np.sqrt(np.mean(o ** 2))
            bad = np.abs(d) > 2e-3 * (np.abs(o) + rms) + 1e-9
            assert not bad.any(), (a0, a1, float(np.max(np.abs(d) / (np.abs(o) + rms + 1e-30))))
        if not fp32:   # and against the plain float64 oracle: operand rounding moves rho by ~1e-2
            op = g_o[a0:a1]
            assert np.linalg.norm(g_g[a0:a1] - op) <= 3e-2 * np.linalg.norm(op) + 1e-9, (a0, a1)
    ls = losses.cpu().numpy()
    A_abs = float(np.abs(A[rows].cpu().numpy()).sum())
    so, sv = (sobj, svl) if fp32 else (sobj_e, svl_e)
    assert abs(ls[0] - so) <= (1e-4 if fp32 else 2e-3) * A_abs
    assert ls[1] == pytest.approx(sv, rel=1e-4 if fp32 else 2e-3)
    assert ls[2] == pytest.approx(H, rel=1e-6) and ls[3] == B
    # Adam, first step, on the device gradient
    th1, _, _ = oracle.adam_step(theta0, np.zeros_like(theta0), np.zeros_like(theta0), g_g, 1, lr)
    np.testing.assert_allclose(learner.master.cpu().numpy(), th1, rtol=0, atol=lr * 1e-4 + 1e-7 * np.abs(th1).max())
    # the rollout slab now holds the bf16 rounding of the updated master copy
    flat = _slab_flat(params.cpu().numpy()[0], L)
    m32 = learner.master.cpu().numpy()
    nw = sum(L.w_rows[l] * L.w_cols[l] for l in range(L.n_layers))
    np.testing.assert_array_equal(flat[:nw], bf16_to_f64(torch.from_numpy(m32[:nw]).to(torch.bfloat16)))
    np.testing.assert_array_equal(flat[nw:], m32[nw:].astype(np.float64))


def test_ppo_bf16_mode_tracks_fp32_mode():
    """The two learner modes on the same minibatch (C3 actor shape): they share every launch, layout and
    epilogue and differ only in the operand precision of the products, so their gradients agree to the bf16
    operand bar (a wrong operand layout in one core would show as an O(1) difference)."""
    c, params, args, M = _ppo_case(100, 3, 512, 0, seed=57, N=512)
    rows = torch.from_numpy(np.random.default_rng(8).permutation(M)[:1024].astype(np.int32)).cuda()
    g = {}
    for fp32 in (True, False):
        lr_ = api.PPOLearner(c.cfg, 3, 512, params.clone(), batch=1024, learning_rate=1e-3, fp32=fp32)
        g[fp32] = torch.empty(lr_.n_elems, dtype=torch.float32, device="cuda")
        lr_.update(*args, rows, grad_out=g[fp32])
    a, b = g[True].cpu().numpy().astype(np.float64), g[False].cpu().numpy().astype(np.float64)
    L = api.actor_layout(c.cfg, 3, 512)
    for a0, a1 in _ppo_segments(L):
        assert np.linalg.norm(a[a0:a1] - b[a0:a1]) <= 3e-2 * np.linalg.norm(a[a0:a1]) + 1e-9, (a0, a1)


def test_ppo_nonfinite_loss_is_flagged_and_not_applied():
    """a non-finite loss signals divergence.  A NaN advantage in the minibatch sets the learner's
    error word; the master, the moments and the slab are left as they were; pod_ppo_check reports
    POD_ERR_NONFINITE and clears it; until then the next update on the workspace refuses to run."""
    c, params, args, M = _ppo_case(30, 2, 128, 0, seed=58)
    obs, act_raw, lpo, A, R = args
    A = A.clone()
    A[5] = float("nan")
    learner = api.PPOLearner(c.cfg, 2, 128, params, batch=512, learning_rate=1e-3)
    m0, slab0 = learner.master.clone(), params.clone()
    rows = torch.arange(0, 512, dtype=torch.int32, device="cuda")
    learner.update(obs, act_raw, lpo, A, R, rows)
    torch.cuda.synchronize()
    assert torch.equal(learner.master, m0) and torch.equal(params, slab0)
    assert torch.count_nonzero(learner.m) == 0
    with pytest.raises(PodError) as ei:
        learner.update(obs, act_raw, lpo, A, R, rows)
    assert ei.value.status == 7
    with pytest.raises(PodError) as ei:
        learner.check()
    assert ei.value.status == 7
    learner.check()   # cleared
    learner.update(obs, act_raw, lpo, args[3], R, rows)   # finite data: applied
    learner.check()
    assert not torch.equal(learner.master, m0)


def test_ppo_learner_improves_surrogate():
    """A few passes of minibatch updates on fixed rollout data (surrogate only: no value or entropy term,
    which would move the shared trunk in directions unrelated to A) increase the clipped surrogate and
    keep every output finite (a smoke check of the full update loop, repeat_times x minibatches)."""
    c = Case(n=30, f=3, T_data=400, N=512, H=100, seed=52)
    aws, params, actor = _actor(c, 2, 128)
    T, B = 8, 1024
    tr = api.Trajectory.allocate(T, c.N, c.n, c.k_pad, critic=True)
    c.env.reset(c.starts)
    c.env.rollout(T, tr, actor=actor)
    adv, ret = api.pod_gae(tr.rew, tr.val[:T].contiguous(), tr.done, tr.val[T].contiguous(), 0.99, 0.95,
                           normalize=True)
    M = T * c.N
    args = (tr.obs[:T].reshape(M, c.k_pad), tr.act.reshape(M, c.n), tr.logp.reshape(M), adv.reshape(M), ret.reshape(M))
    learner = api.PPOLearner(c.cfg, 2, 128, params, batch=B, learning_rate=3e-4, value_coef=0.0, entropy_coef=0.0)
    rng = np.random.default_rng(5)
    objs = []
    for _ in range(4):
        perm = torch.from_numpy(rng.permutation(M).astype(np.int32)).cuda()
        ls = learner.update(*args, perm).cpu().numpy()
        assert np.all(np.isfinite(ls))
        objs.append(ls[0] / ls[3])
    assert objs[-1] > objs[0]
    assert torch.isfinite(learner.master).all()


def test_ppo_graph_replay_step_counter():
    """The minibatch loop is a cached CUDA graph replayed across calls; only the Adam step counter differs
    between calls (read from device memory).  Two calls of one minibatch through the same buffers (the
    second a replay at adam_t = 1) equal one call of two minibatches: a stale bias correction
    (1 - beta^step) on the replay would move the parameters by ~2x."""
    c = Case(n=30, f=3, T_data=400, N=256, H=100, seed=53)
    aws, params_a, actor = _actor(c, 2, 128)
    params_b = params_a.clone()
    T, B = 8, 512
    tr = api.Trajectory.allocate(T, c.N, c.n, c.k_pad, critic=True)
    c.env.reset(c.starts)
    c.env.rollout(T, tr, actor=actor)
    adv, ret = api.pod_gae(tr.rew, tr.val[:T].contiguous(), tr.done, tr.val[T].contiguous(), 0.99, 0.95,
                           normalize=True)
    M = T * c.N
    args = (tr.obs[:T].reshape(M, c.k_pad), tr.act.reshape(M, c.n), tr.logp.reshape(M), adv.reshape(M), ret.reshape(M))
    perm = torch.from_numpy(np.random.default_rng(9).permutation(M)[: 2 * B].astype(np.int32)).cuda()
    la = api.PPOLearner(c.cfg, 2, 128, params_a, batch=B, learning_rate=1e-3)
    lb = api.PPOLearner(c.cfg, 2, 128, params_b, batch=B, learning_rate=1e-3)
    m0 = la.master.cpu().numpy()
    buf = torch.empty(B, dtype=torch.int32, device="cuda")
    for k in range(2):
        buf.copy_(perm[k * B:(k + 1) * B])
        la.update(*args, buf)
    lb.update(*args, perm)
    torch.cuda.synchronize()
    ma, mb = la.master.cpu().numpy(), lb.master.cpu().numpy()
    assert np.isfinite(ma).all() and np.abs(mb - m0).max() > 1e-4
    # the learner is deterministic (fixed-order reductions, no float atomics in the gradient): bit-identical
    np.testing.assert_array_equal(ma, mb)


def test_ppo_hyperparameter_schedule_replays_graph():
    """Hyper-parameters reach the captured minibatch loop through device memory: a learner whose
    learning rate changes between calls (same buffers: a graph replay) takes exactly the step of a fresh
    learner constructed with that rate (same state, same kernels, deterministic data) — a stale, baked-in
    rate would give the first call's step."""
    c = Case(n=30, f=3, T_data=400, N=256, H=100, seed=55)
    aws, params, actor = _actor(c, 2, 128)
    T, B = 8, 512
    tr = api.Trajectory.allocate(T, c.N, c.n, c.k_pad, critic=True)
    c.env.reset(c.starts)
    c.env.rollout(T, tr, actor=actor)
    adv, ret = api.pod_gae(tr.rew, tr.val[:T].contiguous(), tr.done, tr.val[T].contiguous(), 0.99, 0.95,
                           normalize=True)
    M = T * c.N
    args = (tr.obs[:T].reshape(M, c.k_pad), tr.act.reshape(M, c.n), tr.logp.reshape(M), adv.reshape(M), ret.reshape(M))
    perm = torch.from_numpy(np.random.default_rng(4).permutation(M)[:B].astype(np.int32)).cuda()
    sched = api.PPOLearner(c.cfg, 2, 128, params.clone(), batch=B, learning_rate=1e-3, value_coef=0.0,
                           entropy_coef=0.0)
    sched.update(*args, perm)                       # capture at lr 1e-3
    sched.set_hparams(learning_rate=5e-3)
    sched.m.zero_()
    sched.v.zero_()
    sched.t = 0
    theta = sched.master.clone()
    slab = sched.params.clone()                     # the GEMMs read the bf16 slab narrowed from theta
    sched.update(*args, perm)                       # replay at lr 5e-3
    fresh = api.PPOLearner(c.cfg, 2, 128, slab, batch=B, learning_rate=5e-3, value_coef=0.0, entropy_coef=0.0)
    fresh.master.copy_(theta)
    fresh.update(*args, perm)
    torch.cuda.synchronize()
    a, b = sched.master.cpu().numpy(), fresh.master.cpu().numpy()
    moved = np.abs(b - theta.cpu().numpy()) > 0
    assert moved.mean() > 0.5
    np.testing.assert_array_equal(a, b)   # deterministic learner: the replayed step is the fresh one exactly


def test_ppo_concurrent_learners_on_streams():
    """Two learners (distinct buffers, all scratch inside their own workspaces) replayed concurrently on two
    streams reach exactly the parameters of each run alone (any sharing of scratch between the concurrent
    graphs would show)."""
    c = Case(n=30, f=3, T_data=400, N=256, H=100, seed=54)
    aws, params, actor = _actor(c, 2, 128)
    T, B = 8, 512
    tr = api.Trajectory.allocate(T, c.N, c.n, c.k_pad, critic=True)
    c.env.reset(c.starts)
    c.env.rollout(T, tr, actor=actor)
    adv, ret = api.pod_gae(tr.rew, tr.val[:T].contiguous(), tr.done, tr.val[T].contiguous(), 0.99, 0.95,
                           normalize=True)
    M = T * c.N
    args = (tr.obs[:T].reshape(M, c.k_pad), tr.act.reshape(M, c.n), tr.logp.reshape(M), adv.reshape(M), ret.reshape(M))
    perms = [torch.from_numpy(np.random.default_rng(20 + k).permutation(M)[: 4 * B].astype(np.int32)).cuda()
             for k in range(2)]

    def learners():
        return [api.PPOLearner(c.cfg, 2, 128, params.clone(), batch=B, learning_rate=1e-3) for _ in range(2)]

    solo = learners()
    for k in range(2):
        solo[k].update(*args, perms[k])
        torch.cuda.synchronize()
    conc = learners()
    streams = [torch.cuda.Stream() for _ in range(2)]
    main = torch.cuda.current_stream()
    for rep in range(2):   # the second round replays the captured graphs concurrently
        for k in range(2):
            streams[k].wait_stream(main)
            conc[k].update(*args, perms[k], stream=streams[k])
        for k in range(2):
            main.wait_stream(streams[k])
        if rep == 0:
            for k in range(2):
                solo[k].update(*args, perms[k])
    torch.cuda.synchronize()
    for k in range(2):
        a, b = conc[k].master.cpu().numpy(), solo[k].master.cpu().numpy()
        assert np.isfinite(a).all()
        np.testing.assert_array_equal(a, b)


# ----------------------------------------------------------------- shape sweep (edge configurations)
@pytest.mark.parametrize("n,f,N,nh,hid,act,agents,h_max,cost", [
    (1, 3, 1, 1, 128, 0, 1, 100, 0.002),      # one stock, one env (a 1-lane ragged tile)
    (102, 3, 64, 2, 256, 1, 1, 100, 0.002),   # the largest observation (obs_dim 511 of k_pad 512), tanh
    (30, 0, 96, 4, 128, 0, 1, 100, 0.0),      # no indicator channels, four hidden layers, zero cost
    (64, 3, 200, 1, 512, 1, 2, 7, 0.01),      # n % 32 == 0 (critic row in a fresh pad block), 2 agents, small h_max
    (5, 1, 33, 3, 128, 0, 1, 100, 0.002),     # one indicator channel, ragged second tile
    (127, 0, 160, 2, 512, 0, 1, 1000, 0.002), # the most stocks (n_out_pad 128: the widest head), h_max 1000
])
def test_shape_sweep(n, f, N, nh, hid, act, agents, h_max, cost):
    """Sampled rollout with critic on edge configurations: actor means and critic values vs the float64
    oracle on the GPU's observations, Gaussian noise and log-probs vs the oracle's Philox/Box-Muller, and
    the executed actions replayed through the oracle environment (holdings, cash, rewards bit-exact)."""
    c = Case(n=n, f=f, T_data=300, N=N, H=40, n_agents=agents, h_max=h_max, cost=cost, seed=60 + n)
    aws, params, actor = _actor(c, nh, hid, n_agents=agents, act=act)
    T = 5
    tr = api.Trajectory.allocate(T, c.N, c.n, c.k_pad, debug=True, critic=True)
    c.env.reset(c.starts)
    c.env.rollout(T, tr, actor=actor)
    c.env.check()
    obs_g = bf16_to_f64(tr.obs)[..., : c.obs_dim]
    mu_g = tr.mu.cpu().numpy().astype(np.float64)
    raw_g = tr.act.cpu().numpy().astype(np.float64)
    logp_g = tr.logp.cpu().numpy().astype(np.float64)
    val_g = tr.val.cpu().numpy().astype(np.float64)
    per = N // agents
    for a in range(agents):
        rows = slice(a * per, (a + 1) * per)
        aw = aws[a]
        w = oracle.actor_flat(aw.W, aw.b, aw.log_std)
        ls = aw.log_std.astype(np.float64)
        for t in range(T + 1):
            v_o = oracle.actor_value(aw.W, aw.b, aw.w_v, aw.b_v, obs_g[t, rows], nh, hid, act)
            rms = math.sqrt(float(np.mean(v_o ** 2)))
            # with one env the rms is V itself, and V can cancel to near 0: also allow 1e-2 of the
            # magnitude of its terms, sum |w_v| h + |b_v| (bf16 activations carry ~2^-8 of each term)
            v_abs = np.abs(oracle.actor_value(aw.W, aw.b, np.abs(aw.w_v), abs(aw.b_v), obs_g[t, rows], nh, hid, act))
            assert np.all(np.abs(val_g[t, rows] - v_o) <= 2e-2 * (np.abs(v_o) + rms) + 1e-2 * v_abs + 1e-6), (a, t)
            if t == T:
                break
            mu_o = oracle.actor_mu(w, obs_g[t, rows], nh, hid, n, act)
            mu_check(mu_g[t, rows], mu_o)
            for e in range(a * per, (a + 1) * per):
                z_o = oracle.normals(c.cfg.seed, c.cfg.env_offset + e, t, n)
                z_g = (raw_g[t, e] - mu_g[t, e]) / np.exp(ls)
                assert np.all(np.abs(z_g - z_o) <= 2e-5 * np.abs(z_o) + 5e-4), (t, e)
                lp_o = float(np.sum(-0.5 * z_o * z_o - ls - 0.5 * math.log(2 * math.pi)))
                terms = float(np.sum(0.5 * z_o * z_o + np.abs(ls) + 0.5 * math.log(2 * math.pi)))
                assert abs(logp_g[t, e] - lp_o) <= 1e-5 * terms + 1e-4, (t, e)
    o = c.oracle_env()
    out = o.rollout(T, "replay", a_rep=tr.dbg_aint.cpu().numpy(), want=("obs", "rew", "done", "hold", "cash"))
    assert_env_exact(tr, out, c.obs_dim)


@pytest.mark.parametrize("agents", [1, 3])
def test_persistent_actor_bit_identical(agents, monkeypatch):
    """Multi-wave batch (more M-tiles than SM pairs: each persistent cluster runs several tiles, and with
    several agents switches agents between tiles): every output equals the one-tile-per-cluster launch."""
    N = 128 * 90 * agents   # 90 M-tiles per agent > 74 clusters
    outs = []
    for ps in ("0", "1"):
        monkeypatch.setenv("POD_PERSIST", ps)
        c = Case(n=30, f=3, T_data=400, N=N, H=40, n_agents=agents, seed=70)
        aws, params, actor = _actor(c, 2, 128, n_agents=agents)
        tr = api.Trajectory.allocate(3, c.N, c.n, c.k_pad, debug=True, critic=True)
        c.env.reset(c.starts)
        c.env.rollout(3, tr, actor=actor)
        c.env.check()
        outs.append(tr)
    for name in ("obs", "act", "logp", "mu", "val", "rew", "done", "dbg_hold", "dbg_cash"):
        assert torch.equal(getattr(outs[0], name), getattr(outs[1], name)), name
    # and the persistent result itself against the oracle on sampled rows
    obs_g = bf16_to_f64(outs[1].obs)[..., : c.obs_dim]
    mu_g = outs[1].mu.cpu().numpy().astype(np.float64)
    per = N // agents
    for a in range(agents):
        rows = np.arange(a * per, (a + 1) * per, 997)
        w = oracle.actor_flat(aws[a].W, aws[a].b, aws[a].log_std)
        for t in range(3):
            mu_check(mu_g[t, rows], oracle.actor_mu(w, obs_g[t, rows], 2, 128, 30))
