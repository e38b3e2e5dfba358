"""Python face of the float64 CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs — never by the product package
paper_2111_05188_b200/.  It shares no code with the CUDA path; both consume the
same seeded inputs from paper_2111_05188_b200/synth.py (which holds no
arithmetic of the method).

Everything here is argument marshalling (numpy <-> C) except ``actor_flat``,
which lays the per-layer weight matrices out in the oracle's own unpadded
float64 layout (documented in oracle.c, ``orc_actor_mu``).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE, "liboracle.so"])
    return _LIB_PATH


class _Cfg(C.Structure):
    _fields_ = [
        ("n_envs", C.c_int), ("n_stocks", C.c_int), ("n_feat", C.c_int), ("horizon", C.c_int),
        ("h_max", C.c_int), ("n_agents", C.c_int),
        ("C0", C.c_double), ("cost", C.c_double), ("scale", C.c_double), ("gamma", C.c_double),
        ("seed", C.c_uint64), ("env_offset", C.c_int64), ("T_data", C.c_int64),
    ]


class _State(C.Structure):
    _fields_ = [
        ("cash", C.c_void_p), ("asset", C.c_void_p), ("disc", C.c_void_p), ("gpow", C.c_void_p),
        ("ep_ret", C.c_void_p), ("hold", C.c_void_p), ("start", C.c_void_p), ("k", C.c_void_p),
    ]


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        vp, i, i64, u64, d = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double
        L.orc_philox4x32_10.argtypes = [vp, vp, vp]
        L.orc_normals.argtypes = [u64, i64, u64, i, vp]
        L.orc_map_action.argtypes = [d, i]
        L.orc_map_action.restype = i
        L.orc_reset.argtypes = [C.POINTER(_Cfg), C.POINTER(_State)]
        L.orc_obs.argtypes = [C.POINTER(_Cfg), vp, vp, C.POINTER(_State), i, vp]
        L.orc_env_step.argtypes = [C.POINTER(_Cfg), vp, C.POINTER(_State), i, vp, vp, vp, vp, vp, vp]
        L.orc_env_step.restype = i
        L.orc_actor_weight_count.argtypes = [i, i, i, i]
        L.orc_actor_weight_count.restype = i64
        L.orc_actor_mu.argtypes = [vp, i, i, i, i, i, vp, vp, vp]
        L.orc_sample.argtypes = [i, vp, vp, vp, i, vp, vp]
        L.orc_sample.restype = d
        L.orc_rollout.argtypes = [C.POINTER(_Cfg), vp, vp, C.POINTER(_State), i, i, vp, vp, vp, i, i, i,
                                  u64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i]
        L.orc_critic_value.argtypes = [vp, i, i, vp]
        L.orc_critic_value.restype = d
        L.orc_rollout.restype = i64
        L.orc_gae.argtypes = [i, i, vp, vp, vp, vp, d, d, vp, vp, vp]
        L.orc_fitness.argtypes = [i, i, vp, vp]
        L.orc_select_elite.argtypes = [i, vp, i, vp]
        L.orc_select_elite.restype = i
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------
def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def normals(seed: int, env_global: int, step: int, n: int) -> np.ndarray:
    z = np.zeros(n, dtype=np.float64)
    lib().orc_normals(seed, env_global, step, n, _p(z))
    return z


def map_action(u: float, h_max: int) -> int:
    return int(lib().orc_map_action(float(u), int(h_max)))


def actor_flat(W, b, log_std) -> np.ndarray:
    """Oracle weight layout: W_1, b_1, ..., W_out, b_out, log_std (float64)."""
    parts = []
    for Wl, bl in zip(W, b):
        parts.append(np.asarray(Wl, dtype=np.float64).ravel())
        parts.append(np.asarray(bl, dtype=np.float64).ravel())
    parts.append(np.asarray(log_std, dtype=np.float64).ravel())
    return np.ascontiguousarray(np.concatenate(parts))


def actor_mu(w_flat: np.ndarray, obs: np.ndarray, n_hidden: int, hidden: int, n: int, act: int = 0) -> np.ndarray:
    """mu for each row of obs [B, obs_dim] (float64)."""
    obs = np.ascontiguousarray(obs, dtype=np.float64)
    B, od = obs.shape
    assert w_flat.size == lib().orc_actor_weight_count(od, n_hidden, hidden, n)
    mu = np.zeros((B, n), dtype=np.float64)
    scratch = np.zeros(2 * hidden, dtype=np.float64)
    for r in range(B):
        lib().orc_actor_mu(_p(w_flat), od, n_hidden, hidden, n, act, _p(obs[r]), _p(mu[r]), _p(scratch))
    return mu


def actor_value(W, b, w_v, b_v, obs: np.ndarray, n_hidden: int, hidden: int, act: int = 0) -> np.ndarray:
    """Critic V(s) = w_v . h_L(s) + b_v on the actor's trunk h_L ("shared trunk -> actor head +
    critic head"; R#22), for each row of obs [B, obs_dim] (float64).  Evaluated by the same
    MLP routine as the actor mean, with the value row appended to the head."""
    n = int(np.asarray(W[-1]).shape[0])
    W_h = np.vstack([np.asarray(W[-1], dtype=np.float64), np.asarray(w_v, dtype=np.float64)[None, :]])
    b_h = np.append(np.asarray(b[-1], dtype=np.float64), float(b_v))
    flat = actor_flat(list(W[:-1]) + [W_h], list(b[:-1]) + [b_h], np.zeros(n + 1))
    return actor_mu(flat, obs, n_hidden, hidden, n + 1, act)[:, n]


def sample(mu, log_std, z, deterministic=False):
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    ls = np.ascontiguousarray(log_std, dtype=np.float64)
    z = np.ascontiguousarray(z, dtype=np.float64)
    n = mu.size
    raw = np.zeros(n)
    u = np.zeros(n)
    lp = lib().orc_sample(n, _p(mu), _p(ls), _p(z), int(deterministic), _p(raw), _p(u))
    return raw, u, lp


# ---------------------------------------------------------------------------
class Env:
    """Batched oracle environment: N independent envs stepped sequentially."""

    def __init__(self, close, feat, n_envs, horizon, h_max=100, C0=1e6, cost=0.002, scale=1.0,
                 gamma=0.99, seed=0, env_offset=0, n_agents=1):
        self.close = np.ascontiguousarray(close, dtype=np.float32)
        T_data, n = self.close.shape
        feat = np.zeros((T_data, 0, n), np.float32) if feat is None else feat
        self.feat = np.ascontiguousarray(feat, dtype=np.float32)
        f = self.feat.shape[1]
        self.n, self.f, self.N = n, f, n_envs
        self.obs_dim = 1 + 2 * n + n * f
        self.cfg = _Cfg(n_envs, n, f, horizon, h_max, n_agents, C0, cost, scale, gamma, seed,
                        env_offset, T_data)
        N = n_envs
        self.cash = np.zeros(N)
        self.asset = np.zeros(N)
        self.disc = np.zeros(N)
        self.gpow = np.zeros(N)
        self.ep_ret = np.zeros(N)
        self.hold = np.zeros((N, n), dtype=np.int32)
        self.start = np.zeros(N, dtype=np.int64)
        self.k = np.zeros(N, dtype=np.int64)
        self._st = _State(*[a.ctypes.data for a in (self.cash, self.asset, self.disc, self.gpow,
                                                    self.ep_ret, self.hold, self.start, self.k)])

    def reset(self, start_rows):
        self.start[:] = np.asarray(start_rows, dtype=np.int64)
        lib().orc_reset(C.byref(self.cfg), C.byref(self._st))

    def obs(self, e=None):
        if e is None:
            return np.stack([self.obs(i) for i in range(self.N)])
        o = np.zeros(self.obs_dim)
        lib().orc_obs(C.byref(self.cfg), _p(self.close), _p(self.feat), C.byref(self._st), int(e), _p(o))
        return o

    def step_env(self, e, a):
        a = np.ascontiguousarray(a, dtype=np.int32)
        r = np.zeros(1)
        nt = np.zeros(1, dtype=np.int64)
        hp = np.zeros(self.n, dtype=np.int32)
        cp = np.zeros(1)
        d = lib().orc_env_step(C.byref(self.cfg), _p(self.close), C.byref(self._st), int(e), _p(a),
                               _p(r), _p(nt), _p(hp), _p(cp), None)
        return float(r[0]), bool(d), int(nt[0]), hp, float(cp[0])

    def account_value(self, e):
        t = self.start[e] + self.k[e]
        return float(self.cash[e] + np.dot(self.close[t].astype(np.float64), self.hold[e].astype(np.float64)))

    def rollout(self, T, mode="inject", u=None, a_rep=None, weights=None, n_hidden=0, hidden=0, act=0,
                step0=0, nthreads=1, want=("obs", "rew", "done"), critic=None):
        """mode: inject (u [T,N,n] f32), replay (a_rep [T,N,n] i16), sample, deterministic.
        weights: [n_agents, count] float64 (actor_flat per agent).  critic: [n_agents, hidden+1] float64
        (w_v, b_v per agent, R#22); with "val" in want, V(s_t) for t = 0..T in sample/deterministic mode."""
        N, n, od = self.N, self.n, self.obs_dim
        modes = {"inject": 0, "replay": 1, "sample": 2, "deterministic": 3}
        out = {}

        def buf(name, shape, dt):
            if name in want:
                out[name] = np.zeros(shape, dtype=dt)
                return out[name]
            return None

        obs = buf("obs", (T + 1, N, od), np.float64)
        mu = buf("mu", (T, N, n), np.float64)
        raw = buf("raw", (T, N, n), np.float64)
        logp = buf("logp", (T, N), np.float64)
        rew = buf("rew", (T, N), np.float64)
        done = buf("done", (T, N), np.uint8)
        a_out = buf("a_int", (T, N, n), np.int32)
        hold_out = buf("hold", (T, N, n), np.int32)
        cash_out = buf("cash", (T, N), np.float64)
        val = buf("val", (T + 1, N), np.float64)
        asset = buf("asset", (T, N), np.float64)   # account value v_{t+1} after step t, before any reset
        cr = None if critic is None else np.ascontiguousarray(critic, dtype=np.float64)
        u = None if u is None else np.ascontiguousarray(u, dtype=np.float32)
        a_rep = None if a_rep is None else np.ascontiguousarray(a_rep, dtype=np.int16)
        w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
        ties = lib().orc_rollout(C.byref(self.cfg), _p(self.close), _p(self.feat), C.byref(self._st), int(T),
                                 modes[mode], _p(u), _p(a_rep), _p(w), int(n_hidden), int(hidden), int(act),
                                 int(step0), _p(obs), _p(mu), _p(raw), _p(logp), _p(rew), _p(done), _p(a_out),
                                 _p(hold_out), _p(cash_out), _p(cr), _p(val), _p(asset), int(nthreads))
        out["near_ties"] = int(ties)
        return out


# ---------------------------------------------------------------------------
def gae(r, v, d, boot, gamma, lam):
    r = np.ascontiguousarray(r, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    d = np.ascontiguousarray(d, dtype=np.uint8)
    boot = np.ascontiguousarray(boot, dtype=np.float64)
    T, N = r.shape
    adv = np.zeros((T, N))
    ret = np.zeros((T, N))
    mag = np.zeros((T, N))
    lib().orc_gae(T, N, _p(r), _p(v), _p(d), _p(boot), float(gamma), float(lam), _p(adv), _p(ret), _p(mag))
    return adv, ret, mag


def gae_normalize(adv):
    """Per-buffer advantage normalisation ("advantages then normalized to zero mean / unit variance
    per buffer"; R#23): (A - m) / s, m the mean, s the population standard deviation over the
    whole buffer; a constant buffer (s = 0) maps to zeros.  float64."""
    a = np.asarray(adv, dtype=np.float64)
    m = a.sum() / a.size
    s = math.sqrt(((a - m) ** 2).sum() / a.size)
    return np.zeros_like(a) if s == 0.0 else (a - m) / s


def fuse(snapshots, prev, tau):
    """K-pod fusion (S:L302–310 soft_update, S:L364–372 fuse; R#24):
    fused = tau * mean(snapshots) + (1 - tau) * prev, elementwise, float64.  snapshots [K, E]."""
    snap = np.asarray(snapshots, dtype=np.float64)
    mean = snap.sum(axis=0) / snap.shape[0]
    return tau * mean + (1.0 - tau) * np.asarray(prev, dtype=np.float64)


# ---------------------------------------------------------------------------
# evaluator: backtest metrics of an account-value curve and the early-stop rule (
# S:L441–449; R#25).  curve = [v_0, v_1, ..., v_T], float64.
def cumulative_return(curve):
    """S:L519 "subtracting the initial value from the final portfolio value, then dividing by the initial value"."""
    v = np.asarray(curve, dtype=np.float64)
    return (v[-1] - v[0]) / v[0]


def period_returns(curve):
    v = np.asarray(curve, dtype=np.float64)
    return v[1:] / v[:-1] - 1.0


def annual_return_volatility(curve, periods_per_year):
    """annual return (v_T/v_0)^(ppy/T) - 1; volatility = sample (n-1) std of the period returns * sqrt(ppy)."""
    v = np.asarray(curve, dtype=np.float64)
    T = v.size - 1
    rho = period_returns(v)
    ann = (v[-1] / v[0]) ** (periods_per_year / T) - 1.0
    vol = math.sqrt(((rho - rho.mean()) ** 2).sum() / (rho.size - 1)) * math.sqrt(periods_per_year) if rho.size > 1 else 0.0
    return ann, vol


def sharpe(curve, periods_per_year, rf_per_period=0.0):
    """(mean(rho) - rf) / std(rho) * sqrt(ppy), sample std; zero volatility -> NaN (degenerate)."""
    rho = period_returns(curve)
    if rho.size < 2:
        return float("nan")
    sd = math.sqrt(((rho - rho.mean()) ** 2).sum() / (rho.size - 1))
    return float("nan") if sd == 0.0 else (rho.mean() - rf_per_period) / sd * math.sqrt(periods_per_year)


def max_drawdown(curve):
    """min over t of (v_t / max_{s<=t} v_s - 1), single-pass running peak."""
    v = np.asarray(curve, dtype=np.float64)
    peak = -math.inf
    mdd = 0.0
    for x in v:
        peak = max(peak, x)
        mdd = min(mdd, x / peak - 1.0)
    return mdd


def early_stop(history, patience):
    """best = argmax (earliest wins); stop when the latest entry is at least `patience` entries
    after the best (the S:L446 example [1, 2, 1.5, 1.4, 1.3], patience 3 -> stop fixes ">= patience";
    DESIGN.md R#25)."""
    h = list(history)
    if not h:
        raise ValueError("empty history")
    best = max(range(len(h)), key=lambda i: (h[i], -i))
    return (len(h) - 1 - best) >= patience, best


# ---------------------------------------------------------------------------
# PPO learner (Table 3; R#26), float64, on the flat parameter vector in the
# documented slab order: W_0 [h][k_pad], W_1..W_{L-1} [h][h], W_L [n_out_pad][h], b_0.., b_L, log_std [n_out_pad].
def ppo_unflatten(theta, k_pad, hidden, n_hidden, n_out_pad):
    th = np.asarray(theta, dtype=np.float64)
    shapes = [(hidden, k_pad)] + [(hidden, hidden)] * (n_hidden - 1) + [(n_out_pad, hidden)]
    Ws, bs, o = [], [], 0
    for r, c in shapes:
        Ws.append(th[o : o + r * c].reshape(r, c))
        o += r * c
    for r, _ in shapes:
        bs.append(th[o : o + r])
        o += r
    ls = th[o : o + n_out_pad]
    assert o + n_out_pad == th.size
    return Ws, bs, ls


def bf16_round(x):
    """Round to bfloat16 (round to nearest, ties to even, on the float32 value: the precision model of a
    float32 result stored as a bf16 operand), returned as float64."""
    u = np.ascontiguousarray(np.asarray(x, dtype=np.float32)).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def ppo_loss_grad(theta, dims, obs, act_raw, logp_old, adv, ret, eps, c_ent, c_v, act=0, bf16_operands=False,
                  magnitudes=False):
    """Minibatch loss L = -mean(min(rho A, clip(rho, 1-eps, 1+eps) A)) - c_ent H + c_v mean((V - R)^2),
    H = sum_i (log sigma_i + (1 + ln 2 pi)/2), and its analytic gradient (backpropagation written out; the
    min's derivative is that of rho A when rho A <= clip(rho) A, else 0).  dims = (k_pad, hidden, n_hidden,
    n, n_out_pad).  Returns (L, grad [same layout as theta], (sum objective, sum (V-R)^2, H)).
    bf16_operands (DESIGN R#27): the same computation with the operands of every product rounded to bf16 as
    the tensor-core learner stores them — each hidden activation X_{l+1} after its nonlinearity, and each
    delta before it enters the weight- and input-gradient products (the bias gradients sum the unrounded
    delta; the head output Z stays unrounded).
    magnitudes: also return, in the layout of grad, the sums of the absolute values of the terms each
    gradient entry is summed from (|delta_l|^T |X_l|, sum |delta_l|, sum |coef (z^2 - 1)| + c_ent): the
    scale of an elementwise tolerance for a float implementation of the same sums."""
    k_pad, hidden, n_hidden, n, n_out_pad = dims
    Ws, bs, ls = ppo_unflatten(theta, k_pad, hidden, n_hidden, n_out_pad)
    rnd = bf16_round if bf16_operands else (lambda a: a)
    X = [np.asarray(obs, dtype=np.float64)]
    f = (lambda z: np.maximum(z, 0.0)) if act == 0 else np.tanh
    for l in range(n_hidden):
        X.append(rnd(f(X[-1] @ Ws[l].T + bs[l])))
    Z = X[-1] @ Ws[-1].T + bs[-1]
    B = Z.shape[0]
    mu, V = Z[:, :n], Z[:, n]
    sig = np.exp(ls[:n])
    raw = np.asarray(act_raw, dtype=np.float64)
    z = (raw - mu) / sig
    logp = (-0.5 * z * z - ls[:n] - 0.5 * math.log(2 * math.pi)).sum(axis=1)
    A = np.asarray(adv, dtype=np.float64)
    R = np.asarray(ret, dtype=np.float64)
    rho = np.exp(logp - np.asarray(logp_old, dtype=np.float64))
    s1 = rho * A
    s2 = np.clip(rho, 1.0 - eps, 1.0 + eps) * A
    active = s1 <= s2
    obj = np.where(active, s1, s2)
    H = float((ls[:n] + 0.5 * (1.0 + math.log(2 * math.pi))).sum())
    Lval = -obj.mean() - c_ent * H + c_v * ((V - R) ** 2).mean()
    coef = np.where(active, -A * rho / B, 0.0)                 # dL/dlogp per sample
    dZ = np.zeros_like(Z)
    dZ[:, :n] = coef[:, None] * z / sig
    dZ[:, n] = 2.0 * c_v * (V - R) / B
    g_ls = np.zeros(n_out_pad)
    g_ls[:n] = (coef[:, None] * (z * z - 1.0)).sum(axis=0) - c_ent
    m_ls = np.zeros(n_out_pad)
    m_ls[:n] = (np.abs(coef)[:, None] * np.abs(z * z - 1.0)).sum(axis=0) + c_ent
    gW, gb = [None] * (n_hidden + 1), [None] * (n_hidden + 1)
    mW, mb = [None] * (n_hidden + 1), [None] * (n_hidden + 1)
    d = dZ
    for l in range(n_hidden, -1, -1):
        dr = rnd(d)
        gW[l] = dr.T @ X[l]
        gb[l] = d.sum(axis=0)
        if magnitudes:
            mW[l] = np.abs(dr).T @ np.abs(X[l])
            mb[l] = np.abs(d).sum(axis=0)
        if l > 0:
            dx = dr @ Ws[l]
            d = dx * ((X[l] > 0.0) if act == 0 else (1.0 - X[l] ** 2))
    grad = np.concatenate([g.ravel() for g in gW] + [g.ravel() for g in gb] + [g_ls])
    sums = (float(obj.sum()), float(((V - R) ** 2).sum()), H)
    if magnitudes:
        mag = np.concatenate([m.ravel() for m in mW] + [m.ravel() for m in mb] + [m_ls])
        return Lval, grad, sums, mag
    return Lval, grad, sums


def adam_step(theta, m, v, g, t, lr, b1=0.9, b2=0.999, eps=1e-8):
    """Bias-corrected Adam (Kingma & Ba) for minimisation; t counts from 1.  Returns (theta, m, v)."""
    m = b1 * np.asarray(m, dtype=np.float64) + (1.0 - b1) * g
    v = b2 * np.asarray(v, dtype=np.float64) + (1.0 - b2) * g * g
    th = np.asarray(theta, dtype=np.float64) - lr * (m / (1.0 - b1 ** t)) / (np.sqrt(v / (1.0 - b2 ** t)) + eps)
    return th, m, v


def fitness(ep_ret, n_agents):
    ep = np.ascontiguousarray(ep_ret, dtype=np.float64)
    J = np.zeros(n_agents)
    lib().orc_fitness(ep.size, n_agents, _p(ep), _p(J))
    return J


def select_elite(J, k):
    J = np.ascontiguousarray(J, dtype=np.float64)
    plan = np.zeros(J.size, dtype=np.int32)
    rc = lib().orc_select_elite(J.size, _p(J), int(k), _p(plan))
    if rc != 0:
        raise ValueError("orc_select_elite rejected its arguments")
    return plan
