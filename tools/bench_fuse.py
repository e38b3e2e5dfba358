"""Throughput of K-pod ensemble fusion (pod_fuse_pods, R#24) on one GPU: K_local pods x A agents of the
C3 actor (3x512, n = 100).  Algorithmic bytes per call: every slab read once by the sum and written K
times by the blend, the float32 work vector written then read, prev read + written (tau < 1)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2111_05188_b200 import api, configs, synth  # noqa: E402

w = configs.preset("C3")
cfg = api.config_from_workload(w)
K, A = 8, 1
L = api.actor_layout(cfg, w.n_hidden, w.hidden)
obs_dim = int(L.obs_dim)
aws = [synth.make_actor(obs_dim, w.n_hidden, w.hidden, w.n_stocks, 7 + s) for s in range(K * A)]
params = api.pack_actor_params(cfg, aws, w.n_hidden, w.hidden)
E = int(L.n_elems)
prev = torch.zeros((A, E), dtype=torch.float32, device="cuda")
work = torch.empty((A, E), dtype=torch.float32, device="cuda")
for _ in range(3):
    api.fuse_pods(cfg, w.n_hidden, w.hidden, params, K, tau=0.5, prev=prev, work=work)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 50
e0.record()
for _ in range(reps):
    api.fuse_pods(cfg, w.n_hidden, w.hidden, params, K, tau=0.5, prev=prev, work=work)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
slab = int(L.param_bytes)
nbytes = K * A * slab * 2 + A * E * 4 * 2 + A * E * 4 * 2
print(json.dumps({"op": "pod_fuse_pods", "K_local": K, "agents": A, "n_elems": E, "us": ms * 1e3,
                  "alg_bytes": nbytes, "GBps": nbytes / (ms / 1e3) / 1e9}))
