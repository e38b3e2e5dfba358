"""Throughput of the PPO update (pod_ppo_update, R#26) at the C3 actor shape (3x512, n = 100) on one GPU:
minibatches of 1024 rows drawn from a synthetic rollout buffer.  Reports samples/s and the GEMM rate
(forward 2 sum d_in d_out + backward 4 sum d_in d_out per sample, padded dims; the first layer's input
gradient is not computed).  --pods P runs P independent learners (the K pods of an agent, each with its
own master/moments/workspace) concurrently on P CUDA streams: the per-minibatch chain is latency bound,
so concurrent pods fill the GPU."""
import argparse
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_05188_b200 import api, configs, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pods", type=int, default=1)
ap.add_argument("--mb", type=int, default=32, help="minibatches per update call")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--fp32", action="store_true", help="the float32 reference mode")
args = ap.parse_args()
w = configs.preset("C3")
cfg = api.config_from_workload(w)
L = api.actor_layout(cfg, w.n_hidden, w.hidden)
P = args.pods
aws = [synth.make_actor(int(L.obs_dim), w.n_hidden, w.hidden, w.n_stocks, 11 + p) for p in range(P)]
B, M, n_mb = 1024, 65536, args.mb
g = torch.Generator(device="cuda")
g.manual_seed(0)
obs = (torch.randn((M, int(L.k_pad)), generator=g, device="cuda") * 0.5).to(torch.bfloat16)
act = torch.randn((M, w.n_stocks), generator=g, device="cuda")
lpo = torch.randn(M, generator=g, device="cuda") - 100.0
adv = torch.randn(M, generator=g, device="cuda")
ret = torch.randn(M, generator=g, device="cuda")
params = [api.pack_actor_params(cfg, [aws[p]], w.n_hidden, w.hidden) for p in range(P)]
learners = [api.PPOLearner(cfg, w.n_hidden, w.hidden, params[p], batch=B, fp32=args.fp32) for p in range(P)]
perms = [torch.from_numpy(np.random.default_rng(1 + p).permutation(M)[: n_mb * B].astype(np.int32)).cuda()
         for p in range(P)]
streams = [torch.cuda.Stream() for _ in range(P)]


def run():
    main = torch.cuda.current_stream()
    for p in range(P):
        streams[p].wait_stream(main)
        learners[p].update(obs, act, lpo, adv, ret, perms[p], stream=streams[p])
    for p in range(P):
        main.wait_stream(streams[p])


for _ in range(2):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = args.reps
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
sizes = [(L.w_rows[l], L.w_cols[l]) for l in range(L.n_layers)]
flop = sum(2 * r * c for r, c in sizes) + sum(4 * r * c for r, c in sizes) - 2 * sizes[0][0] * sizes[0][1]
samples = P * n_mb * B
print(json.dumps({"op": "pod_ppo_update", "pods": P, "batch": B, "minibatches": n_mb, "ms": ms,
                  "samples_per_s": samples / (ms / 1e3), "gemm_tflops": samples * flop / (ms / 1e3) / 1e12}))
