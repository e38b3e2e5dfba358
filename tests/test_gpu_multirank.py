"""Two ranks, one GPU each, over NCCL: the generation's exchange (P:L322–324 selector, P:L372 parameters,
not gradients) and the K-pod fusion across ranks, through the C ABI, against the float64 oracle.

Skipped unless two GPUs are visible (the round-end boxes have one; the routing itself is covered on CPU
by tests/test_lib_cpu.py with gloo, world size 2).
"""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _slab_bytes(params):
    return params.cpu().numpy().copy()


def _worker(rank, port, out_dir):
    import torch.distributed as dist

    import oracle
    from paper_2111_05188_b200 import api, synth

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(WORLD))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=WORLD, device_id=dev)
    api.load()
    n, f, nh, hid = 30, 3, 2, 128
    cfg = api.make_config(64, n, f, 20, 4, 100, rank * 64, 1e6, 0.002, 1.0, 0.99, 91)
    obs_dim = 1 + 2 * n + n * f
    P_local = 4
    comm = api.Comm(WORLD, rank, P_local)
    res = {}
    # ---- selection: k = 1 (the paper's experiment) and k = P/2, slabs byte-equal to the plan's sources
    for k in (1, WORLD * P_local // 2):
        aws = [synth.make_actor(obs_dim, nh, hid, n, 500 + g) for g in range(WORLD * P_local)]
        all_slabs = api.pack_actor_params(cfg, aws, nh, hid, device=dev)
        params = all_slabs[rank * P_local : (rank + 1) * P_local].clone()
        J = np.random.default_rng(7 + k).normal(size=WORLD * P_local)
        fit = torch.from_numpy(J[rank * P_local : (rank + 1) * P_local].copy()).to(dev)
        plan = comm.select_elite(fit, k, params)
        torch.cuda.synchronize()
        ref = oracle.select_elite(J, k)
        res[f"plan{k}"] = plan
        res[f"ref{k}"] = ref
        exp = all_slabs.cpu().numpy()[ref[rank * P_local : (rank + 1) * P_local]]
        res[f"slabs_equal{k}"] = bool(np.array_equal(params.cpu().numpy(), exp))
    # ---- K-pod fusion across ranks: K_local = 2 pods of each of 2 agents per rank, K = 4
    K_local, A = 2, 2
    aws = [synth.make_actor(obs_dim, nh, hid, n, 900 + r * 10 + s) for r in range(WORLD) for s in range(K_local * A)]
    L = api.actor_layout(cfg, nh, hid)
    for tau in (1.0, 0.3):
        all_slabs = api.pack_actor_params(cfg, aws, nh, hid, device=dev)   # [WORLD * P_local]
        params = all_slabs[rank * P_local : (rank + 1) * P_local].clone()
        prev0 = torch.from_numpy(np.random.default_rng(3).normal(size=(A, int(L.n_elems))).astype(np.float32)).to(dev)
        prev = prev0.clone() if tau != 1.0 else None
        api.fuse_pods(cfg, nh, hid, params, K_local, tau=tau, prev=prev, comm=comm)
        torch.cuda.synchronize()
        np.save(os.path.join(out_dir, f"fuse_{tau}_{rank}.npy"), params.cpu().numpy())
        if prev is not None:
            np.save(os.path.join(out_dir, f"prev_{tau}_{rank}.npy"), prev.cpu().numpy())
        if rank == 0:
            np.save(os.path.join(out_dir, f"before_{tau}.npy"), all_slabs.cpu().numpy())
            np.save(os.path.join(out_dir, f"prev0_{tau}.npy"), prev0.cpu().numpy())
    np.save(os.path.join(out_dir, f"sel_{rank}.npy"), np.array([res], dtype=object), allow_pickle=True)
    comm.destroy()
    dist.destroy_process_group()


def test_two_rank_select_elite_and_fuse(tmp_path):
    if torch.cuda.device_count() < WORLD:
        pytest.skip("needs two GPUs")
    import torch.multiprocessing as mp

    import oracle
    from paper_2111_05188_b200 import api
    from test_gpu_parity import _slab_flat

    mp.spawn(_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True)
    for rank in range(WORLD):
        res = np.load(tmp_path / f"sel_{rank}.npy", allow_pickle=True)[0]
        for k in (1, 4):
            np.testing.assert_array_equal(res[f"plan{k}"], res[f"ref{k}"])
            assert res[f"slabs_equal{k}"], (rank, k)
    cfg = api.make_config(64, 30, 3, 20, 4, 100, 0, 1e6, 0.002, 1.0, 0.99, 91)
    L = api.actor_layout(cfg, 2, 128)
    nw = sum(L.w_rows[l] * L.w_cols[l] for l in range(L.n_layers))
    K_local, A = 2, 2
    for tau in (1.0, 0.3):
        before = np.load(tmp_path / f"before_{tau}.npy")
        prev0 = np.load(tmp_path / f"prev0_{tau}.npy").astype(np.float64)
        after = [np.load(tmp_path / f"fuse_{tau}_{r}.npy") for r in range(WORLD)]
        for a in range(A):
            pods = [r * 4 + a * K_local + k for r in range(WORLD) for k in range(K_local)]
            flats = np.stack([_slab_flat(before[p], L) for p in pods])
            exp = oracle.fuse(flats, prev0[a], tau)
            ref = after[0][a * K_local]
            for r in range(WORLD):
                for k in range(K_local):
                    assert np.array_equal(after[r][a * K_local + k], ref), (tau, a, r, k)   # every pod identical
            got = _slab_flat(ref, L)
            mag = tau * np.abs(flats).mean(axis=0) + (1.0 - tau) * np.abs(prev0[a])
            tol32 = 8.0 * 2.0 ** -24 * mag
            assert np.all(np.abs(got[:nw] - exp[:nw]) <= np.abs(exp[:nw]) * 2.0 ** -8 + 2.0 * tol32[:nw])
            assert np.all(np.abs(got[nw:] - exp[nw:]) <= tol32[nw:])
            if tau != 1.0:
                for r in range(WORLD):
                    pv = np.load(tmp_path / f"prev_{tau}_{r}.npy")[a].astype(np.float64)
                    assert np.all(np.abs(pv - exp) <= tol32)
