"""N > 1 host logic on CPU: whole-group sharding (paper_2503_18929_b200.dist) + one
all-reduce of the partials, run as world_size 2 and 3 gloo process groups. The per-shard
head is the fp64 oracle standing in for the kernels (which need a GPU); what is tested is
that the shards and the single collective compose exactly to the unsharded Eq. 5."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_18929_b200.dist import allreduce_partial_async, group_range, token_balanced_ranges


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _instance(B, K, T, V, seed=0):
    rng = np.random.default_rng(seed)
    N = B * K
    logits = rng.normal(0, 2, size=(N, T, V))
    tokens = rng.integers(0, V, size=(N, T))
    mask = (rng.random((N, T)) < 0.8).astype(np.uint8)
    ref = rng.normal(-5, 1, N)
    rew = rng.normal(0, 1, N)
    return logits, tokens, mask, ref, rew


def _worker(rank, world, port, B, K, out_q):
    from oracle import tba_oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    logits, tokens, mask, ref, rew = _instance(B, K, 3, 7)
    N = B * K
    g0, g1 = group_range(B, world, rank)
    sl = slice(g0 * K, g1 * K)
    if g1 > g0:
        h = O.vargrad_head(logits[sl], tokens[sl], mask[sl], ref[sl], rew[sl], 0.3, K, n_global=N)
        part, d = h["partial"], h["dlogits"]
    else:  # a rank with zero groups contributes zero partials
        part, d = np.zeros(3), np.zeros((0, 3, 7))
    t = torch.tensor(part, dtype=torch.float64)
    pend = allreduce_partial_async(t, dist.group.WORLD)  # the side-stream form (CPU: in place)
    dist.all_reduce(t)  # the path's only collective
    assert torch.equal(pend.wait(), t)
    out_q.put((rank, g0, g1, t.numpy().copy(), d))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,B", [(2, 6), (3, 2)])
def test_sharded_partials_allreduce_to_unsharded_loss(world, B):
    from oracle import tba_oracle as O
    K = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    logits, tokens, mask, ref, rew = _instance(B, K, 3, 7)
    full = O.vargrad_head(logits, tokens, mask, ref, rew, 0.3, K)
    for rank, g0, g1, tot, d in res:
        assert abs(tot[0] - full["loss"]) <= 1e-12 * max(1.0, full["loss"])
        assert tot[1] == B * K and tot[2] == B
        np.testing.assert_allclose(d, full["dlogits"][g0 * K:g1 * K], rtol=1e-12, atol=1e-18)
    covered = sorted((g0, g1) for _, g0, g1, _, _ in res)
    assert covered[0][0] == 0 and covered[-1][1] == B
    assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))


def test_group_range_partition():
    for B in range(0, 20):
        for world in range(1, 9):
            spans = [group_range(B, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        group_range(4, 2, 2)


def test_token_balanced_ranges():
    rng = np.random.default_rng(0)
    toks = list(rng.integers(64 * 20, 512 * 20, size=32))
    for world in (1, 2, 4, 8):
        r = token_balanced_ranges(toks, world)
        assert r[0][0] == 0 and r[-1][1] == 32 and len(r) == world
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
        loads = [sum(toks[a:b]) for a, b in r]
        assert max(loads) <= sum(toks) / world + max(toks)
