"""Host logic of the sharded build, no GPU: the plan helpers of the C ABI
(h2_shard_cut_level, h2_shard_split) and the world-size-2 path over torch.distributed (gloo), where
each process plans its own share and the ranks check they agree and tile the cut level."""
import os
import socket

import numpy as np
import pytest


@pytest.fixture(scope="module")
def P():
    import paper_2206_01885_b200 as P
    from paper_2206_01885_b200 import build
    build.build()
    return P


def test_cut_level_rule(P):
    # shallowest level with >= 64 nodes per rank
    assert P.shard_cut_level([1, 8, 64, 512, 4096], 2) == 3
    assert P.shard_cut_level([1, 8, 64, 512, 4096], 1) == 2
    assert P.shard_cut_level([1, 8, 64, 512, 4096], 8) == 3
    assert P.shard_cut_level([1, 8, 64, 512, 4096], 64) == 4
    # none reaches 64 per rank: the most populous level, shallowest on ties
    assert P.shard_cut_level([1, 4, 30, 30, 12], 8) == 2
    assert P.shard_cut_level([1], 4) == 0


def brute_split(w, R):
    """first[q] = smallest t with prefix(t) * R >= q * total, written out directly."""
    pre = np.concatenate([[0], np.cumsum(w)])
    tot = pre[-1]
    first = [0]
    for q in range(1, R):
        first.append(int(np.flatnonzero(pre * R >= q * tot)[0]))
    return np.array(first + [len(w)])


@pytest.mark.parametrize("seed", range(6))
def test_split_matches_definition_and_balances(P, seed):
    rng = np.random.default_rng(seed)
    for R in (1, 2, 3, 4, 8):
        ncut = int(rng.integers(1, 300))
        w = rng.integers(0, 10 ** rng.integers(1, 12), ncut).astype(np.int64)
        if seed == 0:
            w[:] = 7  # uniform
        first = P.shard_split(w, R)
        assert np.array_equal(first, brute_split(w, R))
        assert first[0] == 0 and first[-1] == ncut and np.all(np.diff(first) >= 0)
        tot = int(w.sum())
        for q in range(R):  # every share within one node's weight of the ideal
            share = int(w[first[q]:first[q + 1]].sum())
            assert share * R <= tot + R * int(w.max(initial=0)) or share == 0


def test_split_edge_cases(P):
    assert np.array_equal(P.shard_split([5], 4), [0, 1, 1, 1, 1])
    assert np.array_equal(P.shard_split([0, 0, 0], 2), [0, 0, 3])
    assert np.array_equal(P.shard_split([], 3), [0, 0, 0, 0])
    with pytest.raises(P.H2Error):
        P.shard_split([1, -1], 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2206_01885_b200 as P
        # rank 0 draws the per-level counts and cut weights; everyone receives them (the build
        # derives them from the redundant tree, identical on every rank)
        obj = [None]
        if rank == 0:
            rng = np.random.default_rng(123)
            counts = np.array([1, 4, 16, 64, 256, 1024], np.int64)
            obj = [(counts, rng.integers(1, 10 ** 6, 4096).astype(np.int64))]
        dist.broadcast_object_list(obj, src=0)
        counts, w_all = obj[0]
        cut = P.shard_cut_level(counts, world)
        w = w_all[: counts[cut]]
        first = P.shard_split(w, world)
        mine = torch.tensor([cut, first[rank], first[rank + 1], int(w[first[rank]:first[rank + 1]].sum())])
        got = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(got, mine)
        q.put((rank, [g.tolist() for g in got], first.tolist()))
    finally:
        dist.destroy_process_group()


def test_world_size_2_gloo_plan_agrees_and_tiles():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    (_, got0, first0), (_, got1, first1) = res
    assert got0 == got1 and first0 == first1  # both ranks hold the same plan
    cuts = {g[0] for g in got0}
    assert cuts == {4}  # 256 >= 64 * 2
    assert got0[0][1] == 0 and got0[0][2] == got0[1][1] and got0[1][2] == 256  # contiguous tiling
    tot = got0[0][3] + got0[1][3]
    assert abs(got0[0][3] - got0[1][3]) <= 10 ** 6 and tot > 0
