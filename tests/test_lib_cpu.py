"""CPU-only checks of the C ABI library: it loads without a GPU, exports every
symbol include/pod.h declares, and its host-only entry points (layout,
workspace sizing, argument validation, elite plan and transfer routing)
behave as specified.  The multi-rank routing is exercised with a gloo
world_size-2 process group (one process per rank, as on the GPU box)."""
import os
import re

import numpy as np
import pytest
import torch

import oracle
from paper_2111_05188_b200 import _lib, api, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2111_05188_b200 import _build
    _build.build()


def test_exports_match_header():
    hdr = open(os.path.join(ROOT, "include", "pod.h")).read()
    declared = set(re.findall(r"^\s*(?:pod_status|const char\*|int|unsigned long long)\s+(pod_\w+)\s*\(", hdr, re.M))
    assert declared == set(_lib.EXPORTS)
    L = _lib.load()
    for name in declared:
        assert hasattr(L, name), name
    assert L.pod_abi_version() == 3
    assert isinstance(L.pod_kernel_launches(), int)
    assert L.pod_status_string(3) == b"POD_ERR_RANGE"


def test_layout_and_workspace():
    cfg = api.make_config(8192, 100, 3, 8192)
    L = api.actor_layout(cfg, 3, 512)
    assert (L.obs_dim, L.k_pad, L.n_out_pad, L.n_layers) == (501, 512, 128, 4)
    assert [L.w_rows[i] for i in range(4)] == [512, 512, 512, 128]
    assert [L.w_cols[i] for i in range(4)] == [512, 512, 512, 512]
    assert L.param_bytes % 1024 == 0 and L.w_offset[0] == 0
    assert L.b_offset[0] >= L.w_offset[3] + 128 * 512 * 2
    cfg30 = api.make_config(16, 30, 3, 64)
    L30 = api.actor_layout(cfg30, 2, 128)
    assert (L30.obs_dim, L30.k_pad, L30.n_out_pad) == (151, 192, 32)
    ws = api.pod_env_workspace_size(cfg)
    assert ws >= 8192 * 100 * 6 + 8192 * 32
    with pytest.raises(_lib.PodError) as ei:
        api.actor_layout(cfg, 3, 300)
    assert ei.value.name == "POD_ERR_UNSUPPORTED"
    for bad in (dict(cost_rate=1.0), dict(initial_capital=0.0), dict(gamma=0.0), dict(h_max=0), dict(n_agents=3)):
        kw = dict(n_envs=64, n_stocks=30, n_feat=3, horizon=10)
        kw.update(bad)
        with pytest.raises(_lib.PodError) as ei:
            api.pod_env_workspace_size(api.make_config(**kw))
        assert ei.value.name == "POD_ERR_ARG", bad


def test_pack_actor_params_roundtrip():
    cfg = api.make_config(32, 30, 3, 64)
    aw = synth.make_actor(151, 2, 128, 30, seed=1)
    slab = api.pack_actor_params(cfg, [aw], 2, 128, device="cpu")[0].numpy()
    L = api.actor_layout(cfg, 2, 128)
    for l in range(3):
        rows, cols = L.w_rows[l], L.w_cols[l]
        raw = slab[L.w_offset[l] : L.w_offset[l] + rows * cols * 2].view(np.uint16).astype(np.uint32) << 16
        W = raw.view(np.float32).reshape(rows, cols)
        np.testing.assert_array_equal(W[: aw.W[l].shape[0], : aw.W[l].shape[1]], aw.W[l])
        b = slab[L.b_offset[l] : L.b_offset[l] + rows * 4].view(np.float32)
        np.testing.assert_array_equal(b[: aw.b[l].size], aw.b[l])
        r0 = aw.W[l].shape[0]
        if l == 2:   # head row n = the critic (R#22)
            np.testing.assert_array_equal(W[r0, : aw.w_v.size], aw.w_v)
            assert b[r0] == np.float32(aw.b_v)
            r0 += 1
        assert not W[r0:].any() and not W[:, aw.W[l].shape[1]:].any() and not b[r0:].any()
    ls = slab[L.log_std_offset : L.log_std_offset + 32 * 4].view(np.float32)
    np.testing.assert_array_equal(ls[:30], aw.log_std)


def test_layout_n_elems():
    """pod_actor_layout.n_elems (the float32 vector of pod_fuse_pods) counts every slab entry once."""
    for n, nh, hid in ((30, 2, 128), (100, 3, 512), (32, 1, 256)):
        cfg = api.make_config(64, n, 3, 10)
        L = api.actor_layout(cfg, nh, hid)
        ne = sum(L.w_rows[l] * L.w_cols[l] + L.w_rows[l] for l in range(L.n_layers)) + L.n_out_pad
        assert L.n_elems == ne
        assert L.n_out_pad >= n + 1 and L.n_out_pad % 32 == 0   # row n is the critic (R#22)


def test_early_stop_matches_oracle():
    """pod_early_stop (host) vs the oracle rule (R#25) on the S:L446–448 examples and random histories."""
    assert api.early_stop([1.0, 2.0, 1.5, 1.4, 1.3], 3) == (True, 1)
    assert api.early_stop([1.0, 2.0, 3.0, 4.0], 2) == (False, 3)
    assert api.early_stop([2.0, 2.0], 1)[1] == 0
    rng = np.random.default_rng(4)
    for _ in range(300):
        h = rng.integers(0, 6, size=int(rng.integers(1, 12))).astype(float)
        p = int(rng.integers(0, 5))
        assert api.early_stop(h, p) == oracle.early_stop(h, p)
    with pytest.raises(_lib.PodError) as ei:
        api.early_stop([], 1)
    assert ei.value.name == "POD_ERR_ARG"


def test_elite_plan_matches_oracle():
    rng = np.random.default_rng(0)
    for _ in range(200):
        P = int(rng.integers(1, 40))
        J = rng.integers(-4, 5, P).astype(float)
        k = int(rng.integers(1, P + 1))
        np.testing.assert_array_equal(api.pod_elite_plan(J, k), oracle.select_elite(J, k))
    with pytest.raises(_lib.PodError) as ei:
        api.pod_elite_plan(np.array([1.0, np.inf]), 1)
    assert ei.value.name == "POD_ERR_NONFINITE"
    with pytest.raises(_lib.PodError):
        api.pod_elite_plan(np.array([1.0, 2.0]), 3)


def _apply_transfers(slabs_per_rank, plan, P_local):
    """Reference semantics of the routing: every rank's slabs after the moves (kind 0 local copies, then the
    sends/receives matched in order per rank pair, then kind 3 fan-out copies of received slabs)."""
    out = [s.copy() for s in slabs_per_rank]
    R = len(slabs_per_rank)
    ops = [api.pod_elite_transfers(plan, P_local, r) for r in range(R)]
    for r in range(R):
        kinds = [k for k, _, _, _ in ops[r]]
        assert kinds == sorted(kinds, key=lambda k: {0: 0, 1: 1, 2: 1, 3: 2}[k])   # execution order
        for kind, peer, src, dst in ops[r]:
            if kind == 0:
                out[r][dst] = slabs_per_rank[r][src]
    for r in range(R):
        recvs = [(p, d) for k, p, s, d in ops[r] if k == 2]
        for peer in range(R):
            sends = [s for k, p, s, d in ops[peer] if k == 1 and p == r]
            mine = [d for p, d in recvs if p == peer]
            assert len(sends) == len(mine)
            for s, d in zip(sends, mine):
                out[r][d] = slabs_per_rank[peer][s]
    for r in range(R):
        for kind, peer, src, dst in ops[r]:
            if kind == 3:
                out[r][dst] = out[r][src]
    return out


def test_elite_slab_crosses_once_per_rank():
    """k = 1 (the paper's experiment): the elite's slab leaves its rank once per other rank (a
    broadcast), not once per eliminated slot; the other slots of each rank are filled by local copies."""
    R, P_local = 8, 8
    J = np.arange(R * P_local, dtype=float)   # agent 63 (rank 7) is the elite
    plan = api.pod_elite_plan(J, 1)
    sends = [op for op in api.pod_elite_transfers(plan, P_local, 7) if op[0] == 1]
    assert sorted(p for _, p, _, _ in sends) == list(range(7))
    for r in range(7):
        ops = api.pod_elite_transfers(plan, P_local, r)
        assert [k for k, _, _, _ in ops].count(2) == 1 and [k for k, _, _, _ in ops].count(3) == P_local - 1
    # k = P/2 with every rank needing elites from every other rank: at most one receive per (elite, rank)
    J = np.random.default_rng(5).normal(size=R * P_local)
    plan = api.pod_elite_plan(J, R * P_local // 2)
    for r in range(R):
        rec = [(p, d) for k, p, s, d in api.pod_elite_transfers(plan, P_local, r) if k == 2]
        srcs = [plan[r * P_local + d] for _, d in rec]
        assert len(srcs) == len(set(srcs))


def test_transfers_realise_the_plan():
    rng = np.random.default_rng(1)
    for _ in range(100):
        R = int(rng.integers(1, 9))
        P_local = int(rng.integers(1, 9))
        P = R * P_local
        J = rng.normal(size=P)
        k = int(rng.integers(1, P + 1))
        plan = api.pod_elite_plan(J, k)
        slabs = [np.arange(r * P_local, (r + 1) * P_local) for r in range(R)]
        out = _apply_transfers(slabs, plan, P_local)
        got = np.concatenate(out)
        np.testing.assert_array_equal(got, plan)   # slot g now holds agent plan[g]


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P_local, k, W = 3, 2, 16
        rng = np.random.default_rng(100 + rank)
        fit = torch.from_numpy(rng.normal(size=P_local))
        gathered = [torch.zeros(P_local, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, fit)
        J = torch.cat(gathered).numpy()
        plan = api.pod_elite_plan(J, k)
        slabs = torch.stack([torch.full((W,), float(rank * P_local + i)) for i in range(P_local)])
        new = slabs.clone()
        ops = api.pod_elite_transfers(plan, P_local, rank)
        for kind, peer, src, dst in ops:   # same order on both sides
            if kind == 0:
                new[dst] = slabs[src]
            elif kind == 1:
                dist.send(slabs[src].contiguous(), peer)
            elif kind == 2:
                buf = torch.empty(W)
                dist.recv(buf, peer)
                new[dst] = buf
            else:
                new[dst] = new[src]
        allp = [torch.zeros(1, dtype=torch.int32) for _ in range(world)]
        q.put((rank, plan.tolist(), new[:, 0].tolist(), J.tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_select_routing():
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(2)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, plan0, slab0, J0), (r1, plan1, slab1, J1) = res
    assert plan0 == plan1 and J0 == J1                      # identical plan on every rank
    ref = oracle.select_elite(np.array(J0), 2)
    assert plan0 == list(ref)
    np.testing.assert_array_equal(np.array(slab0 + slab1), ref.astype(float))  # slot g holds agent plan[g]
