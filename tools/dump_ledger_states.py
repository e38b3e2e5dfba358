# steady-state pre-buy ledger states for the ledger probe: 8 steps x 32 envs after the sell pass
import numpy as np, sys, math
sys.path.insert(0,'.')
import oracle
from paper_2111_05188_b200 import synth, configs
oracle.build()
w = configs.preset("C3")
m = synth.make_market(100, 60000, w.dt, w.seed, n_feat=3)
aw = synth.make_actor(w.obs_dim, 3, 512, 100, w.seed*1000)
wf = oracle.actor_flat(aw.W, aw.b, aw.log_std)
N, T = 32, 120
env = oracle.Env(m.close, m.feat, N, horizon=8192, seed=w.seed)
st = np.repeat(synth.tile_starts(1, 60000, 8192, 3), 32)
env.reset(st)
out = env.rollout(T, "sample", weights=wf[None,:], n_hidden=3, hidden=512, nthreads=8, want=("a_int","hold","cash"))
a = out["a_int"]; hold = out["hold"]; cash = out["cash"]
close = m.close.astype(np.float64); c = 0.002
recs = []
for t in range(T-8, T):
    row = st[0] + t; p = close[row]
    unit = p*(1+c); 
    A = np.zeros((100, 32), np.int16); Hh = np.zeros((100, 32), np.int32); B = np.zeros(32)
    for e in range(32):
        h = hold[t-1, e].astype(np.int64).copy(); b = cash[t-1, e]; ai = a[t, e]
        for i in range(100):
            q = min(h[i], -ai[i]) if ai[i] < 0 else 0
            b = b + (p[i]*q)*(1-c)
        A[:, e] = ai; Hh[:, e] = hold[t-1, e]; B[e] = b
    recs.append((unit, A, Hh, B, p, cash[t-1, :32].copy()))
with open("exp/ledger_states.bin", "wb") as f:
    for unit, A, Hh, B, p, c0 in recs:
        unit.astype(np.float64).tofile(f); A.tofile(f); Hh.tofile(f); B.astype(np.float64).tofile(f)
        p.astype(np.float64).tofile(f); c0.astype(np.float64).tofile(f)
print("wrote", len(recs))
