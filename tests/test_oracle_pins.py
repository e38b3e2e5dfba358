"""Pins for the float64 oracle (oracle/oracle.c) against values the paper and
the mathematics fix: worked examples (tests/golden, each cited), closed forms,
invariants, library routines and brute force.  CPU only (`-m "not gpu"`).

Each check is chosen so that a plausible slip in the oracle (a dropped term,
a wrong sign or index, a transposed operand, a wrong order of sells/buys)
fails at least one of them.
"""
import math

import numpy as np
import pytest
from scipy import stats

import oracle
from conftest import golden
from paper_2111_05188_b200 import synth


# ---------------------------------------------------------------------------
# Philox4x32-10 and normals
# ---------------------------------------------------------------------------
def test_philox_known_answers():
    for v in golden("philox_kat.json")["vectors"]:
        ctr = [int(x, 16) for x in v["ctr"]]
        key = [int(x, 16) for x in v["key"]]
        out = oracle.philox4x32_10(ctr, key)
        assert [f"{x:08x}" for x in out] == v["out"]


def test_normals_statistics():
    # 2.5e5 draws x 4 components: mean 0, var 1, KS vs N(0,1)
    n = 100
    zs = np.concatenate([oracle.normals(1234, e, 7, n) for e in range(2500)])
    assert abs(zs.mean()) < 5 * (1 / math.sqrt(zs.size))
    assert abs(zs.var() - 1.0) < 5 * math.sqrt(2.0 / zs.size)
    assert stats.kstest(zs, "norm").pvalue > 1e-4
    # independence of the streams: different envs / steps / seeds differ
    a = oracle.normals(1, 0, 0, 8)
    assert not np.allclose(a, oracle.normals(1, 1, 0, 8))
    assert not np.allclose(a, oracle.normals(1, 0, 1, 8))
    assert not np.allclose(a, oracle.normals(2, 0, 0, 8))
    # components of the same quad are the Box-Muller pairs of one Philox call
    x = oracle.philox4x32_10([5, 9, 0, 0], [77, 0])
    u1 = (float(x[0]) + 1.0) * 2.0 ** -32
    u2 = float(x[1]) * 2.0 ** -32
    z = oracle.normals(77, 5, 9, 4)
    assert z[0] == pytest.approx(math.sqrt(-2 * math.log(u1)) * math.cos(2 * math.pi * u2), rel=1e-14)
    assert z[1] == pytest.approx(math.sqrt(-2 * math.log(u1)) * math.sin(2 * math.pi * u2), rel=1e-14)


# ---------------------------------------------------------------------------
# action map
# ---------------------------------------------------------------------------
def test_map_action_pins():
    for c in golden("map_pins.json")["cases"]:
        u = float(np.float32(c["u_f32"])) if "u_f32" in c else c["u"]
        assert oracle.map_action(u, c["h_max"]) == c["a"], c["cite"]


def test_map_action_properties():
    rng = np.random.default_rng(0)
    for u in rng.uniform(-1, 1, 2000):
        a = oracle.map_action(u, 100)
        assert abs(a) <= 100
        assert abs(a - u * 100) <= 0.5 + 1e-12
        assert oracle.map_action(-u, 100) == -a  # odd symmetry


# ---------------------------------------------------------------------------
# env step worked examples and derived cases
# ---------------------------------------------------------------------------
def _one_step(case):
    n = case["n"]
    prices = np.asarray(case["prices"] + [case["prices"][-1]], dtype=np.float32)  # 3 rows
    env = oracle.Env(prices, None, 1, horizon=10, C0=max(case["cash"], 1.0), cost=case["cost"])
    env.reset([0])
    env.cash[0] = case["cash"]
    env.hold[0] = case["hold"]
    env.asset[0] = case["cash"] + float(np.dot(prices[0].astype(np.float64), np.asarray(case["hold"], np.float64)))
    r, done, ties, hold_post, cash_post = env.step_env(0, np.asarray(case["a"], np.int32))
    v1 = cash_post + float(np.dot(prices[1].astype(np.float64), hold_post.astype(np.float64)))
    return r, hold_post, cash_post, v1


@pytest.mark.parametrize("case", golden("env_step_pins.json")["cases"], ids=lambda c: c["name"])
def test_env_step_pins(case):
    r, hold_post, cash_post, v1 = _one_step(case)
    assert list(hold_post) == case["hold_post"], case["cite"]
    atol = case["atol"]
    assert abs(cash_post - case["cash_post"]) <= atol, case["cite"]
    assert abs(v1 - case["value_post"]) <= atol + 1e-12, case["cite"]
    assert abs(r - case["reward"]) <= atol + 1e-12, case["cite"]


def test_account_value_pin():
    g = golden("env_step_pins.json")["account_value"]
    env = oracle.Env(np.asarray([g["price"], g["price"]], np.float32), None, 1, horizon=5, C0=1.0)
    env.reset([0])
    env.cash[0] = g["cash"]
    env.hold[0] = g["hold"]
    assert env.account_value(0) == g["value"]


# ---------------------------------------------------------------------------
# observation
# ---------------------------------------------------------------------------
def test_obs_pins():
    g = golden("obs_pins.json")
    env = oracle.Env(np.asarray([[5.0], [6.0]], np.float32), None, 1, horizon=1)
    env.reset([0])
    assert list(env.obs(0)) == g["fresh_reset_n1_f0"]["obs"]
    env2 = oracle.Env(np.ones((3, 2), np.float32), np.zeros((3, 3, 2), np.float32), 1, horizon=1)
    env2.reset([0])
    assert env2.obs(0).size == g["length_n2_f3"]["length"]
    h = g["holding_entry"]
    env3 = oracle.Env(np.asarray([[h["price"]], [h["price"]]], np.float32), None, 1, horizon=1, C0=h["C0"])
    env3.reset([0])
    env3.hold[0] = h["shares"]
    assert env3.obs(0)[1] == pytest.approx(h["value"], rel=1e-15)


def test_obs_layout_channel_major():
    T_data, n, f = 6, 3, 2
    close = (np.arange(T_data * n, dtype=np.float32).reshape(T_data, n) + 10.0)
    feat = np.arange(T_data * f * n, dtype=np.float32).reshape(T_data, f, n) / 100.0
    env = oracle.Env(close, feat, 1, horizon=4, C0=1000.0)
    env.reset([1])
    env.k[0] = 2  # t = 3
    env.hold[0] = [1, 2, 3]
    env.cash[0] = 250.0
    o = env.obs(0)
    assert o[0] == 0.25
    np.testing.assert_array_equal(o[1:4], np.array([1, 2, 3]) * close[3].astype(np.float64) / 1000.0)
    np.testing.assert_array_equal(o[4:7], close[3].astype(np.float64) / close[1].astype(np.float64))
    np.testing.assert_array_equal(o[7:10], feat[3, 0].astype(np.float64))
    np.testing.assert_array_equal(o[10:13], feat[3, 1].astype(np.float64))


# ---------------------------------------------------------------------------
# env invariants
# ---------------------------------------------------------------------------
def _market(n=5, T_data=400, seed=3):
    return synth.make_market(n, T_data, 1 / 252, seed)


@pytest.mark.parametrize("kind", ["uniform", "all_buy", "all_sell", "sparse", "buy_then_sell"])
def test_invariants_under_injected_actions(kind):
    m = _market()
    N, T, H = 6, 60, 25
    env = oracle.Env(m.close, m.feat, N, horizon=H, C0=1e4, cost=0.002)
    starts = synth.tile_starts(N, m.T_data, H, 1)
    env.reset(starts)
    u = synth.injected_u(kind, T, N, m.n, 2)
    for t in range(T):
        for e in range(N):
            tt = env.start[e] + env.k[e]
            pre_v = env.account_value(e)
            a = np.array([oracle.map_action(x, 100) for x in u[t, e]], np.int32)
            r, done, _, hp, cp = env.step_env(e, a)
            # cash and holdings non-negative (P:L222 b in R+, Eq. 4)
            assert cp >= 0.0 and (hp >= 0).all()
            # reward consistency: r = v_{t+1} - v_t
            v1 = cp + float(np.dot(m.close[tt + 1].astype(np.float64), hp.astype(np.float64)))
            assert r == pytest.approx(v1 - pre_v, rel=1e-12, abs=1e-9)
            # auto-reset semantics
            if done:
                assert env.k[e] == 0 and env.cash[e] == 1e4 and (env.hold[e] == 0).all()


def test_zero_cost_accounting_identity():
    # with cost 0, v_{t+1} - v_t = h_{t+1}^T (p_{t+1} - p_t)
    m = _market(seed=9)
    N = 4
    env = oracle.Env(m.close, m.feat, N, horizon=50, C0=1e5, cost=0.0)
    env.reset([3, 40, 100, 200])
    rng = np.random.default_rng(0)
    for t in range(40):
        for e in range(N):
            tt = env.start[e] + env.k[e]
            a = rng.integers(-100, 101, m.n).astype(np.int32)
            r, done, _, hp, cp = env.step_env(e, a)
            dp = m.close[tt + 1].astype(np.float64) - m.close[tt].astype(np.float64)
            assert r == pytest.approx(float(np.dot(hp.astype(np.float64), dp)), rel=1e-9, abs=1e-7)


def test_cost_monotonicity():
    # for the same state and action, raising the cost rate never raises the reward
    m = _market(seed=11)
    rng = np.random.default_rng(1)
    for trial in range(50):
        a = rng.integers(-100, 101, m.n).astype(np.int32)
        hold0 = rng.integers(0, 50, m.n).astype(np.int32)
        rs = []
        for c in (0.0, 0.001, 0.002, 0.01):
            env = oracle.Env(m.close, m.feat, 1, horizon=50, C0=2e4, cost=c)
            env.reset([10 + trial])
            env.hold[0] = hold0
            env.asset[0] = env.account_value(0)
            rs.append(env.step_env(0, a)[0])
        assert all(rs[i + 1] <= rs[i] + 1e-9 for i in range(len(rs) - 1))


def test_batch_equivalence_bit_identical():
    # S:L209 / S:L651: batched stepping == each env stepped alone, bit for bit
    m = _market(seed=4)
    N, T, H = 5, 30, 12
    starts = synth.tile_starts(N, m.T_data, H, 5)
    u = synth.injected_u("uniform", T, N, m.n, 6)
    batch = oracle.Env(m.close, m.feat, N, horizon=H, C0=1e4)
    batch.reset(starts)
    out = batch.rollout(T, "inject", u=u, want=("obs", "rew", "done", "hold", "cash"))
    for e in range(N):
        one = oracle.Env(m.close, m.feat, 1, horizon=H, C0=1e4)
        one.reset(starts[e : e + 1])
        o1 = one.rollout(T, "inject", u=np.ascontiguousarray(u[:, e : e + 1]), want=("obs", "rew", "done", "hold", "cash"))
        for key in ("obs", "rew", "done", "hold", "cash"):
            np.testing.assert_array_equal(out[key][:, e], o1[key][:, 0])
    # threads do not change anything
    again = oracle.Env(m.close, m.feat, N, horizon=H, C0=1e4)
    again.reset(starts)
    o2 = again.rollout(T, "inject", u=u, nthreads=4, want=("obs", "rew", "done", "hold", "cash"))
    for key in ("obs", "rew", "done", "hold", "cash"):
        np.testing.assert_array_equal(out[key], o2[key])


def test_rollout_matches_manual_stepping_and_done_rules():
    m = _market(n=3, T_data=60, seed=21)
    N, T, H = 3, 50, 7
    starts = np.array([0, 20, 50], np.int64)  # env 2 hits the end of data (t+1 == T_data-1) before H
    u = synth.injected_u("uniform", T, N, m.n, 7)
    env = oracle.Env(m.close, m.feat, N, horizon=H, C0=5e3)
    env.reset(starts)
    out = env.rollout(T, "inject", u=u, want=("obs", "rew", "done", "a_int"))
    man = oracle.Env(m.close, m.feat, N, horizon=H, C0=5e3)
    man.reset(starts)
    for t in range(T):
        for e in range(N):
            np.testing.assert_array_equal(out["obs"][t, e], man.obs(e))
            tt = man.start[e] + man.k[e]
            k_before = man.k[e]
            a = np.array([oracle.map_action(x, 100) for x in u[t, e]], np.int32)
            np.testing.assert_array_equal(out["a_int"][t, e], a)
            r, d, _, _, _ = man.step_env(e, a)
            assert out["rew"][t, e] == r
            assert bool(out["done"][t, e]) == d
            assert d == ((k_before + 1 == H) or (tt + 1 == m.T_data - 1))
    # env 2: start 50, T_data 60 -> t+1 == 59 after 9 steps, but H=7 comes first;
    # env 0 done every 7 steps exactly
    assert list(np.nonzero(out["done"][:, 0])[0][:3]) == [6, 13, 20]


def test_reward_scale_linear():
    m = _market(seed=13)
    u = synth.injected_u("uniform", 20, 2, m.n, 1)
    res = []
    for scale in (1.0, 0.25):
        env = oracle.Env(m.close, m.feat, 2, horizon=100, C0=1e4, scale=scale)
        env.reset([5, 9])
        res.append(env.rollout(20, "inject", u=u, want=("rew", "hold"))["rew"])
    np.testing.assert_array_equal(res[0] * 0.25, res[1])  # power-of-two scale: exact


# ---------------------------------------------------------------------------
# actor and sampler
# ---------------------------------------------------------------------------
def test_actor_zero_weights_give_bias():
    od, nh, H, n = 7, 2, 8, 3
    W = [np.zeros((H, od)), np.zeros((H, H)), np.zeros((n, H))]
    b = [np.ones(H), np.ones(H), np.array([0.5, -1.0, 2.0])]
    w = oracle.actor_flat(W, b, np.zeros(n))
    mu = oracle.actor_mu(w, np.random.default_rng(0).normal(size=(4, od)), nh, H, n)
    # h1 = relu(1) = 1, h2 = relu(0*1 + 1) = 1, mu = 0*h2 + b_out
    np.testing.assert_array_equal(mu, np.tile([0.5, -1.0, 2.0], (4, 1)))


@pytest.mark.parametrize("act", [0, 1])
def test_actor_matches_numpy_matmul(act):
    od, nh, H, n = 23, 3, 16, 5
    aw = synth.make_actor(od, nh, H, n, seed=3, bias_scale=0.3)
    w = oracle.actor_flat(aw.W, aw.b, aw.log_std)
    x = np.random.default_rng(1).normal(size=(9, od))
    mu = oracle.actor_mu(w, x, nh, H, n, act)
    h = x
    f = (lambda z: np.maximum(z, 0.0)) if act == 0 else np.tanh
    for l in range(nh):
        h = f(h @ aw.W[l].astype(np.float64).T + aw.b[l].astype(np.float64))
    ref = h @ aw.W[nh].astype(np.float64).T + aw.b[nh].astype(np.float64)
    np.testing.assert_allclose(mu, ref, rtol=1e-12, atol=1e-12)


def test_gae_normalize_pins():
    """R#23: zero mean / unit variance per buffer.  Worked example [1, 2, 3] -> m = 2,
    s = sqrt(2/3) -> [-sqrt(3/2), 0, sqrt(3/2)]; constant buffer -> zeros; the result has mean 0 and
    population variance 1, and is invariant to an affine change a A + b (a > 0) of the input."""
    np.testing.assert_allclose(oracle.gae_normalize(np.array([[1.0, 2.0, 3.0]])), [[-math.sqrt(1.5), 0.0, math.sqrt(1.5)]],
                               rtol=1e-15, atol=1e-15)
    np.testing.assert_array_equal(oracle.gae_normalize(np.full((4, 5), 2.5)), np.zeros((4, 5)))
    x = np.random.default_rng(3).normal(size=(64, 33)) * 3.0 + 1.7
    y = oracle.gae_normalize(x)
    assert abs(y.mean()) < 1e-13 and abs(y.var() - 1.0) < 1e-12
    np.testing.assert_allclose(oracle.gae_normalize(0.25 * x - 4.0), y, rtol=1e-12, atol=1e-12)


def test_fuse_pins():
    """R#24 pins: S:L371 fuse([0,0],[2,4], tau=1) = [1,2]; S:L310 soft update target [0,2], source [2,4],
    tau = 0.5 -> [1,3] (a single snapshot is its own mean); tau = 0 keeps prev; K identical snapshots with
    tau = 1 return the snapshot; the mean is symmetric in the pods."""
    np.testing.assert_array_equal(oracle.fuse([[0.0, 0.0], [2.0, 4.0]], [9.0, 9.0], 1.0), [1.0, 2.0])
    np.testing.assert_array_equal(oracle.fuse([[2.0, 4.0]], [0.0, 2.0], 0.5), [1.0, 3.0])
    x = np.random.default_rng(5).normal(size=(3, 7))
    p = np.random.default_rng(6).normal(size=7)
    np.testing.assert_array_equal(oracle.fuse(x, p, 0.0), p)
    np.testing.assert_array_equal(oracle.fuse(np.tile(x[0], (4, 1)), p, 1.0), x[0])
    np.testing.assert_allclose(oracle.fuse(x[::-1], p, 0.3), oracle.fuse(x, p, 0.3), rtol=1e-15)


def test_critic_value_pins():
    """R#22: V = w_v . h_L + b_v on the actor's trunk.  Pins: a zero trunk gives V = b_v exactly; a
    general trunk equals a numpy float64 forward; the actor mean is unaffected by the critic row."""
    od, nh, H, n = 9, 2, 8, 3
    W = [np.zeros((H, od)), np.zeros((H, H)), np.zeros((n, H))]
    b = [np.zeros(H), np.zeros(H), np.zeros(n)]
    x = np.random.default_rng(4).normal(size=(5, od))
    np.testing.assert_array_equal(oracle.actor_value(W, b, np.ones(H), -0.75, x, nh, H), np.full(5, -0.75))
    for act in (0, 1):
        aw = synth.make_actor(23, 3, 16, 5, seed=6, bias_scale=0.3)
        x = np.random.default_rng(7).normal(size=(6, 23))
        v = oracle.actor_value(aw.W, aw.b, aw.w_v, aw.b_v, x, 3, 16, act)
        h = x
        f = (lambda z: np.maximum(z, 0.0)) if act == 0 else np.tanh
        for l in range(3):
            h = f(h @ aw.W[l].astype(np.float64).T + aw.b[l].astype(np.float64))
        np.testing.assert_allclose(v, h @ aw.w_v.astype(np.float64) + aw.b_v, rtol=1e-12, atol=1e-12)
        mu = oracle.actor_mu(oracle.actor_flat(aw.W, aw.b, aw.log_std), x, 3, 16, 5, act)
        np.testing.assert_allclose(mu, h @ aw.W[3].astype(np.float64).T + aw.b[3].astype(np.float64),
                                   rtol=1e-12, atol=1e-12)


def test_rollout_critic_matches_standalone_value():
    """The rollout's trunk-sharing critic (orc_critic_value) equals the head-row evaluation of
    actor_value on the recorded observations, bit for bit, including the bootstrap V(s_T)."""
    m = _market(n=4, T_data=200, seed=5)
    od = 1 + 2 * 4 + 4 * 3
    aw = synth.make_actor(od, 3, 16, 4, seed=9)
    w = oracle.actor_flat(aw.W, aw.b, aw.log_std)[None, :]
    cr = np.append(aw.w_v.astype(np.float64), aw.b_v)[None, :]
    env = oracle.Env(m.close, m.feat, 3, horizon=4, C0=1e4, seed=11)
    env.reset([3, 50, 90])
    out = env.rollout(6, "sample", weights=w, n_hidden=3, hidden=16, want=("obs", "val"), critic=cr)
    for t in range(7):
        np.testing.assert_array_equal(out["val"][t], oracle.actor_value(aw.W, aw.b, aw.w_v, aw.b_v, out["obs"][t], 3, 16))


def test_sample_logprob_is_gaussian_density():
    # log_prob equals an independent evaluation of the Gaussian density
    rng = np.random.default_rng(2)
    n = 11
    mu = rng.normal(size=n)
    ls = rng.normal(size=n) * 0.3 - 0.7
    z = rng.normal(size=n)
    raw, u, lp = oracle.sample(mu, ls, z)
    np.testing.assert_allclose(raw, mu + np.exp(ls) * z, rtol=1e-15)
    np.testing.assert_allclose(u, np.tanh(raw), rtol=1e-15)
    ref = stats.norm.logpdf(raw, loc=mu, scale=np.exp(ls)).sum()
    assert lp == pytest.approx(ref, rel=1e-12, abs=1e-12)
    raw_d, _, lp_d = oracle.sample(mu, ls, z, deterministic=True)
    np.testing.assert_array_equal(raw_d, mu)  # S:L261 zero-variance limit -> mean
    assert lp_d == pytest.approx(stats.norm.logpdf(mu, loc=mu, scale=np.exp(ls)).sum(), rel=1e-12)


def test_sampled_rollout_uses_the_pieces():
    m = _market(n=4, T_data=200, seed=5)
    od = 1 + 2 * 4 + 4 * 3
    aw = synth.make_actor(od, 2, 16, 4, seed=8)
    w = oracle.actor_flat(aw.W, aw.b, aw.log_std)[None, :]
    env = oracle.Env(m.close, m.feat, 2, horizon=30, C0=1e4, seed=99, env_offset=40)
    env.reset([3, 50])
    out = env.rollout(5, "sample", weights=w, n_hidden=2, hidden=16, step0=17,
                      want=("obs", "mu", "raw", "logp", "a_int"))
    for t in range(5):
        for e in range(2):
            mu = oracle.actor_mu(w[0], out["obs"][t, e][None], 2, 16, 4)[0]
            np.testing.assert_array_equal(out["mu"][t, e], mu)
            z = oracle.normals(99, 40 + e, 17 + t, 4)
            raw, u, lp = oracle.sample(mu, aw.log_std, z)
            np.testing.assert_array_equal(out["raw"][t, e], raw)
            assert out["logp"][t, e] == lp
            assert list(out["a_int"][t, e]) == [oracle.map_action(x, 100) for x in u]


# ---------------------------------------------------------------------------
# GAE
# ---------------------------------------------------------------------------
def test_gae_worked_example():
    g = golden("gae_pins.json")
    adv, ret, _ = oracle.gae(np.array(g["r"])[:, None], np.array(g["v"])[:, None],
                             np.array(g["d"], np.uint8)[:, None], np.array([g["boot"]]), g["gamma"], g["lam"])
    np.testing.assert_allclose(adv[:, 0], g["adv"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(ret[:, 0], g["ret"], rtol=0, atol=1e-12)


def _gae_brute(r, v, d, boot, gamma, lam):
    T = r.shape[0]
    vn = np.concatenate([v[1:], [boot]])
    delta = r + gamma * (1 - d) * vn - v
    A = np.zeros(T)
    for t in range(T):
        s, w = 0.0, 1.0
        for l in range(T - t):
            s += w * delta[t + l]
            w *= gamma * lam * (1 - d[t + l])
        A[t] = s
    return A


def test_gae_brute_force_with_dones():
    T, N = 64, 6
    r, v, d, boot = synth.gae_inputs(T, N, seed=3, p_done=0.1)
    adv, ret, mag = oracle.gae(r, v, d, boot, 0.99, 0.95)
    for e in range(N):
        A = _gae_brute(r[:, e].astype(float), v[:, e].astype(float), d[:, e].astype(float), float(boot[e]), 0.99, 0.95)
        np.testing.assert_allclose(adv[:, e], A, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(ret, adv + v, rtol=1e-15, atol=1e-15)
    assert (mag >= np.abs(adv) - 1e-12).all()  # |A_t| <= M_t by the triangle inequality


def test_gae_closed_forms():
    T = 10
    r = np.arange(1, T + 1, dtype=float)[:, None]
    z = np.zeros((T, 1))
    d0 = np.zeros((T, 1), np.uint8)
    # lambda = gamma = 1, V = 0 -> suffix sums
    adv, _, _ = oracle.gae(r, z, d0, np.zeros(1), 1.0, 1.0)
    np.testing.assert_allclose(adv[:, 0], np.cumsum(r[::-1, 0])[::-1])
    # single step: A = r + gamma V' - V
    adv1, _, _ = oracle.gae(np.array([[2.0]]), np.array([[0.5]]), np.zeros((1, 1), np.uint8), np.array([3.0]), 0.9, 0.7)
    assert adv1[0, 0] == pytest.approx(2.0 + 0.9 * 3.0 - 0.5, rel=1e-15)
    # r == 1, V = 0, no dones -> A_t = (1 - (g l)^(T-t)) / (1 - g l)
    g, l = 0.99, 0.95
    adv2, _, _ = oracle.gae(np.ones((T, 1)), z, d0, np.zeros(1), g, l)
    ref = (1 - (g * l) ** (T - np.arange(T))) / (1 - g * l)
    np.testing.assert_allclose(adv2[:, 0], ref, rtol=1e-13)
    # gamma lambda = 0 -> A = delta
    rr, vv, dd, bb = synth.gae_inputs(T, 2, seed=1, p_done=0.3)
    adv3, _, _ = oracle.gae(rr, vv, dd, bb, 0.9, 0.0)
    vn = np.concatenate([vv[1:], bb[None]]).astype(float)
    np.testing.assert_allclose(adv3, rr + 0.9 * (1 - dd) * vn - vv, rtol=1e-12, atol=1e-12)
    # a done masks the bootstrap: the value after a terminal step never enters
    rr2, vv2 = np.ones((2, 1)), np.zeros((2, 1))
    adv4, _, _ = oracle.gae(rr2, vv2, np.array([[0], [1]], np.uint8), np.array([100.0]), 0.99, 0.95)
    np.testing.assert_allclose(adv4[:, 0], [1 + 0.99 * 0.95 * 1.0, 1.0])


# ---------------------------------------------------------------------------
# fitness and selection
# ---------------------------------------------------------------------------
def test_fitness_pin_via_env():
    g = golden("fitness_select_pins.json")["fitness"]
    # one stock whose price rises by 1 per step while holding 1 share, zero cost:
    # every reward is exactly 1 (Eq. 2), the episode lasts 3 steps (H = 3).
    close = np.array([[10.0], [11.0], [12.0], [13.0], [14.0]], np.float32)
    env = oracle.Env(close, None, 1, horizon=3, C0=100.0, cost=0.0, gamma=g["gamma"])
    env.reset([0])
    a = np.array([[[0]], [[0]], [[0]]], np.int16)
    env.hold[0] = [1]
    env.cash[0] = 90.0
    env.asset[0] = 100.0
    out = env.rollout(3, "replay", a_rep=a, want=("rew", "done"))
    np.testing.assert_array_equal(out["rew"][:, 0], g["rewards"])
    assert list(out["done"][:, 0]) == [0, 0, 1]
    assert env.ep_ret[0] == pytest.approx(g["J"], rel=1e-15)
    assert oracle.fitness(env.ep_ret, 1)[0] == pytest.approx(g["J"], rel=1e-15)


def test_fitness_is_group_mean():
    ep = np.arange(12, dtype=float) ** 1.5
    J = oracle.fitness(ep, 3)
    np.testing.assert_allclose(J, ep.reshape(3, 4).mean(1), rtol=1e-15)


def test_select_pins():
    for c in golden("fitness_select_pins.json")["select"]:
        assert list(oracle.select_elite(np.array(c["J"]), c["k"])) == c["plan"], c["cite"]


def test_select_brute_force_and_invariants():
    rng = np.random.default_rng(0)
    for trial in range(300):
        P = int(rng.integers(1, 20))
        J = rng.integers(-3, 4, P).astype(float)  # many ties
        k = int(rng.integers(1, P + 1))
        plan = oracle.select_elite(J, k)
        order = sorted(range(P), key=lambda g: (-J[g], g))
        elites = order[:k]
        elim = [g for g in range(P) if g not in elites]
        ref = list(range(P))
        for j, g in enumerate(elim):
            ref[g] = elites[j % k]
        assert list(plan) == ref
        # population conservation + survivor monotonicity
        assert len(plan) == P
        assert all(J[s] >= J[g] for s in elites for g in elim)
    with pytest.raises(ValueError):
        oracle.select_elite(np.array([1.0, np.nan]), 1)
    with pytest.raises(ValueError):
        oracle.select_elite(np.array([1.0]), 2)


# ---------------------------------------------------------------------------
# evaluator metrics (R#25)
# ---------------------------------------------------------------------------
def test_backtest_metric_pins():
    assert oracle.cumulative_return([1_000_000.0, 1_700_000.0, 2_495_530.0]) == pytest.approx(1.49553, abs=1e-12)
    assert oracle.cumulative_return([5.0, 5.0, 5.0]) == 0.0
    assert oracle.cumulative_return([10.0, 4.0, 0.0]) == -1.0
    # max drawdown vs an exhaustive peak-trough pair scan
    assert oracle.max_drawdown([100.0, 120.0, 90.0, 110.0]) == pytest.approx(-0.25, abs=1e-15)
    assert oracle.max_drawdown([100.0]) == 0.0
    assert oracle.max_drawdown(np.arange(1.0, 20.0)) == 0.0
    rng = np.random.default_rng(8)
    for _ in range(20):
        v = np.cumprod(1.0 + rng.normal(0, 0.05, size=30)) * 100.0
        brute = min([0.0] + [v[j] / v[i] - 1.0 for i in range(30) for j in range(i, 30)])
        assert oracle.max_drawdown(v) == pytest.approx(brute, abs=1e-15)
    # constant per-period return r with ppy = T: annual return (1 + r)^T - 1, volatility 0
    r, T = 0.01, 12
    curve = 100.0 * (1.0 + r) ** np.arange(T + 1)
    ann, vol = oracle.annual_return_volatility(curve, T)
    assert ann == pytest.approx((1 + r) ** T - 1, rel=1e-12) and vol == pytest.approx(0.0, abs=1e-12)
    ann, vol = oracle.annual_return_volatility([1.0, 2.0], 1)
    assert ann == pytest.approx(1.0, rel=1e-15)
    # Sharpe: zero-mean alternating returns -> 0; constant returns -> degenerate (NaN); S:L539 worked case
    alt = np.cumprod(np.r_[1.0, np.tile([1.01, 1.0 / 1.01], 5)])
    rho = oracle.period_returns(alt)
    assert oracle.sharpe(alt, 252) == pytest.approx(rho.mean() / rho.std(ddof=1) * math.sqrt(252), rel=1e-12)
    assert math.isnan(oracle.sharpe(2.0 ** np.arange(6.0), 252))   # returns exactly 1.0 each period
    c3 = np.cumprod([1.0, 1.01, 1.02, 0.995])
    rho3 = np.array([0.01, 0.02, -0.005])
    assert oracle.sharpe(c3, 252) == pytest.approx(rho3.mean() / np.std(rho3, ddof=1) * math.sqrt(252), rel=1e-10)


def test_early_stop_pins():
    # S:L446–448
    assert oracle.early_stop([1.0, 2.0, 1.5, 1.4, 1.3], 3) == (True, 1)
    assert oracle.early_stop([1.0, 2.0, 3.0, 4.0], 2) == (False, 3)
    assert oracle.early_stop([2.0, 2.0], 1)[1] == 0          # earliest wins
    assert oracle.early_stop([2.0, 2.0], 2) == (False, 0)
    with pytest.raises(ValueError):
        oracle.early_stop([], 1)


# ---------------------------------------------------------------------------
# PPO learner (R#26)
# ---------------------------------------------------------------------------
def _ppo_problem(seed, act=1, B=24):
    rng = np.random.default_rng(seed)
    dims = (8, 5, 2, 2, 4)   # k_pad, hidden, n_hidden, n, n_out_pad
    k_pad, hid, nh, n, nop = dims
    ne = hid * k_pad + hid * hid + nop * hid + hid + hid + nop + nop
    theta = rng.normal(size=ne) * 0.5
    obs = np.zeros((B, k_pad))
    obs[:, :6] = rng.normal(size=(B, 6))
    act_raw = rng.normal(size=(B, n))
    return rng, dims, theta, obs, act_raw


def test_ppo_gradient_matches_finite_differences():
    """the analytic gradient of the total loss matches central finite differences (here within 1e-6
    relative, float64), on a smooth (tanh) network with ratios away from the clip boundaries."""
    rng, dims, theta, obs, act_raw = _ppo_problem(1)
    B = obs.shape[0]
    adv = rng.normal(size=B)
    ret = rng.normal(size=B)
    # logp_old = current logp + offsets chosen so rho sits well inside or well outside [0.75, 1.25]
    k_pad, hid, nh, n, nop = dims
    Ws, bs, ls = oracle.ppo_unflatten(theta, k_pad, hid, nh, nop)
    h = obs
    for l in range(nh):
        h = np.tanh(h @ Ws[l].T + bs[l])
    mu = (h @ Ws[-1].T + bs[-1])[:, :n]
    z = (act_raw - mu) / np.exp(ls[:n])
    logp = (-0.5 * z * z - ls[:n] - 0.5 * math.log(2 * math.pi)).sum(axis=1)
    shift = rng.choice([-0.6, -0.05, 0.0, 0.05, 0.6], size=B)
    lpo = logp + shift
    args = (dims, obs, act_raw, lpo, adv, ret, 0.25, 0.02, 0.5, 1)
    L, g, _ = oracle.ppo_loss_grad(theta, *args)
    hstep = 1e-6
    idx = rng.choice(theta.size, size=60, replace=False)
    for i in idx:
        tp, tm = theta.copy(), theta.copy()
        tp[i] += hstep
        tm[i] -= hstep
        fd = (oracle.ppo_loss_grad(tp, *args)[0] - oracle.ppo_loss_grad(tm, *args)[0]) / (2 * hstep)
        assert abs(fd - g[i]) <= 1e-6 * max(1.0, abs(g[i])) + 1e-8, (i, fd, g[i])


def test_ppo_clip_pins():
    """rho = 1 everywhere -> the clipped surrogate's gradient equals the unclipped one.
    S:L291: rho = 2, A > 0, eps = 0.25 -> the contribution uses 1.25 A (and no policy gradient)."""
    rng, dims, theta, obs, act_raw = _ppo_problem(2)
    B = obs.shape[0]
    k_pad, hid, nh, n, nop = dims
    Ws, bs, ls = oracle.ppo_unflatten(theta, k_pad, hid, nh, nop)
    h = obs
    for l in range(nh):
        h = np.tanh(h @ Ws[l].T + bs[l])
    mu = (h @ Ws[-1].T + bs[-1])[:, :n]
    z = (act_raw - mu) / np.exp(ls[:n])
    logp = (-0.5 * z * z - ls[:n] - 0.5 * math.log(2 * math.pi)).sum(axis=1)
    adv = rng.normal(size=B)
    ret = rng.normal(size=B)
    _, g_clip, _ = oracle.ppo_loss_grad(theta, dims, obs, act_raw, logp, adv, ret, 0.25, 0.0, 0.0, 1)
    _, g_free, _ = oracle.ppo_loss_grad(theta, dims, obs, act_raw, logp, adv, ret, 1e9, 0.0, 0.0, 1)
    np.testing.assert_allclose(g_clip, g_free, rtol=1e-12, atol=1e-15)
    A = np.abs(adv) + 0.1
    L, g, (sobj, _, _) = oracle.ppo_loss_grad(theta, dims, obs, act_raw, logp - math.log(2.0), A, ret, 0.25, 0.0, 0.0, 1)
    assert sobj == pytest.approx(1.25 * A.sum(), rel=1e-12)
    nW = hid * k_pad + hid * hid + nop * hid
    np.testing.assert_array_equal(g[:nW][: hid * k_pad], 0.0)    # no policy gradient flows through the clip


def test_bf16_round_matches_torch_bfloat16():
    """R#27's rounding model: oracle.bf16_round (RNE of the float32 value to 8 significant bits) equals torch's
    float32 -> bfloat16 conversion (an independent library routine), including ties to even, negatives,
    subnormals, zero and the largest finite values."""
    import torch
    rng = np.random.default_rng(12)
    x = np.concatenate([rng.normal(size=4000) * 10.0 ** rng.integers(-30, 30, 4000),
                        [0.0, -0.0, 1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8, -(1.0 + 2.0 ** -8), 1e-40, -3e-39,
                         3.3895313892515355e38, 65504.0, 2.0 ** -133]]).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(oracle.bf16_round(x), ref)


def test_ppo_bf16_operand_emulation_exact_on_representable_values():
    """R#27: with every operand already bf16-representable (small integer observations and weights, ReLU,
    integer returns, c_v a power of two, A = 0 so only the value head trains) the rounding emulation changes
    nothing: the emulated gradient equals the plain float64 one exactly; with real-valued operands it
    differs (the rounding is applied)."""
    rng = np.random.default_rng(13)
    dims = (8, 5, 2, 2, 4)
    k_pad, hid, nh, n, nop = dims
    ne = hid * k_pad + hid * hid + nop * hid + hid + hid + nop + nop
    theta = rng.integers(-1, 2, size=ne).astype(np.float64) * 0.5   # activations stay small integers / halves
    theta[-nop:] = 0.0   # log-std 0
    B = 16
    obs = rng.integers(0, 2, size=(B, k_pad)).astype(np.float64)
    act_raw = rng.normal(size=(B, n))
    lpo = np.zeros(B)
    adv = np.zeros(B)
    ret = rng.integers(-4, 5, size=B).astype(np.float64)
    args = (dims, obs, act_raw, lpo, adv, ret, 0.25, 0.0, 4.0, 0)   # 2 c_v / B = 1/2
    _, g_plain, _ = oracle.ppo_loss_grad(theta, *args)
    _, g_emu, _ = oracle.ppo_loss_grad(theta, *args, bf16_operands=True)
    assert np.abs(g_plain).max() > 0
    np.testing.assert_array_equal(g_emu, g_plain)
    theta2 = theta + rng.normal(size=ne) * 1e-3
    _, g2p, _ = oracle.ppo_loss_grad(theta2, *args)
    _, g2e, _ = oracle.ppo_loss_grad(theta2, *args, bf16_operands=True)
    assert not np.array_equal(g2p, g2e)


def test_adam_first_step_is_normalised_gradient():
    """Bias-corrected Adam's first step: m_hat = g, v_hat = g^2, so the update is -lr g / (|g| + eps)."""
    g = np.array([1e-3, -2.0, 0.0, 5e-9])
    th, m, v = oracle.adam_step(np.zeros(4), np.zeros(4), np.zeros(4), g, 1, 0.01)
    np.testing.assert_allclose(th, -0.01 * g / (np.abs(g) + 1e-8), rtol=1e-12, atol=0.0)
