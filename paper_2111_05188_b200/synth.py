"""Seeded synthetic inputs shared by the CUDA path, the oracle and the bench.

This module holds NO arithmetic of the method (no env step, no observation,
no actor, no sampling, no GAE, no selection).  It only draws the inputs both
sides consume, so that the GPU path and the oracle see byte-identical data:

* correlated GBM close prices shaped like Dow-30 daily / NASDAQ-100 minute data
  ("the data volume varies with ... the length of
  data period, the time granularity, the number of stocks"),
* three technical-indicator channels (MACD, RSI, CCI) computed
  once on the host, z-scored per channel (input preprocessing, out of the hot
  path per SURVEY.md §2.1 A17),
* per-agent actor weights (bf16-representable), tile start rows, injected-action
  sets and GAE inputs.

All generators are numpy ``Generator(PCG64(seed))`` based and deterministic.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np
from scipy.signal import lfilter

ENV_TILE = 32  # envs per tile (one warp); tiles share a start row


# ---------------------------------------------------------------------------
# Market data
# ---------------------------------------------------------------------------
def _ema(x: np.ndarray, period: int) -> np.ndarray:
    """EMA along the last axis (time), seeded with the first value."""
    a = 2.0 / (period + 1.0)
    zi = ((1.0 - a) * x[:, :1])
    y, _ = lfilter([a], [1.0, -(1.0 - a)], x, axis=-1, zi=zi)
    return y


def _wilder(x: np.ndarray, period: int) -> np.ndarray:
    a = 1.0 / period
    zi = ((1.0 - a) * x[:, :1])
    y, _ = lfilter([a], [1.0, -(1.0 - a)], x, axis=-1, zi=zi)
    return y


def _macd(close: np.ndarray) -> np.ndarray:
    """close [n, T] -> MACD line EMA12 - EMA26 [n, T]."""
    return _ema(close, 12) - _ema(close, 26)


def _rsi(close: np.ndarray, period: int = 14) -> np.ndarray:
    """Wilder RSI [n, T]; flat series -> 50 (S:L90 convention)."""
    d = np.diff(close, axis=-1, prepend=close[:, :1])
    g = _wilder(np.maximum(d, 0.0), period)
    l = _wilder(np.maximum(-d, 0.0), period)
    with np.errstate(divide="ignore", invalid="ignore"):
        rsi = 100.0 - 100.0 / (1.0 + g / l)
    return np.where(l == 0.0, np.where(g == 0.0, 50.0, 100.0), rsi)


def _cci(high: np.ndarray, low: np.ndarray, close: np.ndarray, period: int = 20) -> np.ndarray:
    """CCI [n, T] = (tp - SMA(tp)) / (0.015 * mean |tp - SMA|) over the trailing window
    (shorter during warm-up); zero deviation -> 0."""
    tp = (high + low + close) / 3.0
    n, T = tp.shape
    cs = np.concatenate([np.zeros((n, 1)), np.cumsum(tp, axis=-1)], axis=-1)
    idx = np.arange(T)
    lo = np.maximum(idx - period + 1, 0)
    cnt = (idx - lo + 1).astype(np.float64)
    sma = (cs[:, idx + 1] - cs[:, lo]) / cnt
    # trailing-window sum of |tp_j - sma_t|; torch (multi-threaded CPU) over time blocks
    import torch

    tpt = torch.from_numpy(tp)
    smat = torch.from_numpy(sma)
    md_t = torch.zeros_like(tpt)
    for t in range(min(period - 1, T)):  # warm-up: windows [0, t]
        md_t[:, t] = (tpt[:, : t + 1] - smat[:, t : t + 1]).abs().sum(-1)
    blk = 32768
    for t0 in range(period - 1, T, blk):  # full windows [t - period + 1, t]
        t1 = min(T, t0 + blk)
        win = tpt[:, t0 - period + 1 : t1].unfold(1, period, 1)       # [n, t1 - t0, period]
        md_t[:, t0:t1] = (win - smat[:, t0:t1, None]).abs().sum(-1)
    md = md_t.numpy()
    md /= cnt
    with np.errstate(divide="ignore", invalid="ignore"):
        c = (tp - sma) / (0.015 * md)
    return np.where(md == 0.0, 0.0, c)


@dataclass
class Market:
    close: np.ndarray  # [T_data, n] float32, > 0
    feat: np.ndarray   # [T_data, f, n] float32, channel-major, z-scored per channel
    dt: float

    @property
    def T_data(self) -> int:
        return int(self.close.shape[0])

    @property
    def n(self) -> int:
        return int(self.close.shape[1])

    @property
    def f(self) -> int:
        return int(self.feat.shape[1])


def make_market(n: int, T_data: int, dt: float, seed: int, n_feat: int = 3,
                beta: float = 0.5, chunk: int = 1 << 17) -> Market:
    """Correlated GBM:
    ln S_{t+1,i} = ln S_{t,i} + (mu_i - sigma_i^2/2) dt
                   + sigma_i sqrt(dt) (beta z_m,t + sqrt(1-beta^2) z_i,t),
    mu_i ~ U[-0.05, 0.25]/yr, sigma_i ~ U[0.15, 0.50]/yr, S_0 = exp(U[ln 10, ln 500]).
    Synthetic high/low for CCI: close (1 +- |N(0, 0.25 sigma sqrt(dt))|).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    mu = rng.uniform(-0.05, 0.25, n)
    sig = rng.uniform(0.15, 0.50, n)
    s0 = np.exp(rng.uniform(math.log(10.0), math.log(500.0), n))
    drift = (mu - 0.5 * sig * sig) * dt
    vol = sig * math.sqrt(dt)
    logp = np.empty((T_data, n), dtype=np.float64)
    cur = np.log(s0)
    logp[0] = cur
    t = 1
    while t < T_data:
        m = min(chunk, T_data - t)
        zm = rng.standard_normal((m, 1))
        zi = rng.standard_normal((m, n))
        inc = drift + vol * (beta * zm + math.sqrt(1.0 - beta * beta) * zi)
        blk = cur + np.cumsum(inc, axis=0)
        logp[t : t + m] = blk
        cur = blk[-1]
        t += m
    close64 = np.exp(logp)
    del logp
    close = close64.astype(np.float32)
    del close64
    cT = np.ascontiguousarray(close.T, dtype=np.float64)  # [n, T]: indicators see exactly the stored prices
    feat = np.empty((T_data, n_feat, n), dtype=np.float32)

    def put(ch, x):
        m, s = float(x.mean()), float(x.std())
        feat[:, ch, :] = ((x - m) / (s if s > 0 else 1.0)).T.astype(np.float32)

    if n_feat >= 1:
        put(0, _macd(cT))
    if n_feat >= 2:
        put(1, _rsi(cT))
    if n_feat >= 3:
        spread = np.abs(rng.standard_normal((n, T_data))) * (0.25 * vol)[:, None]
        spread2 = np.abs(rng.standard_normal((n, T_data))) * (0.25 * vol)[:, None]
        put(2, _cci(cT * (1.0 + spread), cT * (1.0 - spread2), cT))
        del spread, spread2
    for extra in range(3, n_feat):
        put(extra, _ema(cT, 5 + 5 * extra) / cT - 1.0)
    return Market(close=np.ascontiguousarray(close), feat=feat, dt=dt)


def make_flat_market(n: int, T_data: int, prices, n_feat: int = 0) -> Market:
    """Hand-specified price rows (for worked examples): prices[T_data][n]."""
    close = np.asarray(prices, dtype=np.float32).reshape(T_data, n)
    feat = np.zeros((T_data, n_feat, n), dtype=np.float32)
    return Market(close=close, feat=feat, dt=1.0)


# ---------------------------------------------------------------------------
# Actor weights (N(0, 1/fan_in) rounded to bf16, log-std = ln 0.5)
# ---------------------------------------------------------------------------
def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (RNE) and return them as float32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


@dataclass
class ActorWeights:
    """One agent's actor: layers W[l] [out, in] (bf16-representable float32),
    b[l] [out] float32, log_std [n] float32.  Layer 0 has in = obs_dim, the
    hidden layers in = hidden, the head out = n.  Critic (R#22): V(s) =
    w_v . h_L(s) + b_v on the same trunk (w_v [hidden] bf16-representable)."""
    W: list
    b: list
    log_std: np.ndarray
    w_v: Optional[np.ndarray] = None
    b_v: float = 0.0


def make_actor(obs_dim: int, n_hidden: int, hidden: int, n: int, seed: int,
               bias_scale: float = 0.05, log_std: float = math.log(0.5)) -> ActorWeights:
    rng = np.random.Generator(np.random.PCG64(seed))
    dims = [obs_dim] + [hidden] * n_hidden + [n]
    Ws, bs = [], []
    for l in range(n_hidden + 1):
        fan_in, fan_out = dims[l], dims[l + 1]
        W = rng.standard_normal((fan_out, fan_in)) / math.sqrt(fan_in)
        Ws.append(bf16_round(W.astype(np.float32)))
        bs.append((rng.standard_normal(fan_out) * bias_scale).astype(np.float32))
    ls = np.full(n, log_std, dtype=np.float32)
    # critic row, drawn after the actor's so the actor weights do not depend on it
    w_v = bf16_round((rng.standard_normal(dims[-2]) / math.sqrt(dims[-2])).astype(np.float32))
    b_v = float(np.float32(rng.standard_normal() * bias_scale))
    return ActorWeights(W=Ws, b=bs, log_std=ls, w_v=w_v, b_v=b_v)


# ---------------------------------------------------------------------------
# Env layout inputs
# ---------------------------------------------------------------------------
def tile_starts(n_tiles: int, T_data: int, horizon: int, seed: int) -> np.ndarray:
    """Episode start row per tile, uniform in [0, T_data - H - 1] (so a full
    episode fits: start + H <= T_data - 1)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    hi = T_data - horizon - 1
    if hi < 0:
        raise ValueError("horizon too long for the market data")
    return rng.integers(0, hi + 1, size=n_tiles, dtype=np.int64)


def injected_u(kind: str, T: int, N: int, n: int, seed: int) -> np.ndarray:
    """Injected squashed actions u in [-1, 1] (float32), SURVEY §8(d) parity sets."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if kind == "uniform":
        u = rng.uniform(-1.0, 1.0, (T, N, n))
    elif kind == "all_buy":
        u = np.ones((T, N, n))
    elif kind == "all_sell":
        u = -np.ones((T, N, n))
    elif kind == "sparse":
        u = rng.uniform(-1.0, 1.0, (T, N, n)) * (rng.uniform(0, 1, (T, N, n)) < 0.1)
    elif kind == "buy_then_sell":
        u = rng.uniform(0.0, 1.0, (T, N, n))
        u[T // 2 :] = -u[T // 2 :]
    else:
        raise ValueError(kind)
    return np.ascontiguousarray(u.astype(np.float32))


def gae_inputs(T: int, N: int, seed: int, p_done: float = 1.0 / 64.0):
    """GAE standalone inputs: r, V, boot ~ N(0,1); d ~ Bernoulli."""
    rng = np.random.Generator(np.random.PCG64(seed))
    r = rng.standard_normal((T, N)).astype(np.float32)
    v = rng.standard_normal((T, N)).astype(np.float32)
    boot = rng.standard_normal(N).astype(np.float32)
    d = (rng.uniform(0, 1, (T, N)) < p_done).astype(np.uint8)
    return r, v, d, boot
