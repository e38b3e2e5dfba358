"""Throughput of the PPO update (pod_ppo_update, R#26) at the C3 actor shape (3x512, n = 100) on one GPU:
minibatches of 1024 rows drawn from a synthetic rollout buffer.  Reports samples/s and the float32 GEMM
rate (forward 2 sum d_in d_out + backward 4 sum d_in d_out per sample, padded dims; the first layer's
input gradient is not computed)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_05188_b200 import api, configs, synth  # noqa: E402

w = configs.preset("C3")
cfg = api.config_from_workload(w)
L = api.actor_layout(cfg, w.n_hidden, w.hidden)
aw = synth.make_actor(int(L.obs_dim), w.n_hidden, w.hidden, w.n_stocks, 11)
params = api.pack_actor_params(cfg, [aw], w.n_hidden, w.hidden)
B, M, n_mb = 1024, 65536, 32
g = torch.Generator(device="cuda")
g.manual_seed(0)
obs = (torch.randn((M, int(L.k_pad)), generator=g, device="cuda") * 0.5).to(torch.bfloat16)
act = torch.randn((M, w.n_stocks), generator=g, device="cuda")
lpo = torch.randn(M, generator=g, device="cuda") - 100.0
adv = torch.randn(M, generator=g, device="cuda")
ret = torch.randn(M, generator=g, device="cuda")
learner = api.PPOLearner(cfg, w.n_hidden, w.hidden, params, batch=B)
perm = torch.from_numpy(np.random.default_rng(1).permutation(M)[: n_mb * B].astype(np.int32)).cuda()
for _ in range(2):
    learner.update(obs, act, lpo, adv, ret, perm)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 5
for _ in range(reps):
    learner.update(obs, act, lpo, adv, ret, perm)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
sizes = [(L.w_rows[l], L.w_cols[l]) for l in range(L.n_layers)]
flop = sum(2 * r * c for r, c in sizes) + sum(4 * r * c for r, c in sizes) - 2 * sizes[0][0] * sizes[0][1]
samples = n_mb * B
print(json.dumps({"op": "pod_ppo_update", "batch": B, "minibatches": n_mb, "ms": ms,
                  "samples_per_s": samples / (ms / 1e3), "gemm_tflops": samples * flop / (ms / 1e3) / 1e12}))
