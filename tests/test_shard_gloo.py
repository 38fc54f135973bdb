"""Host side of the column-sharded path with world_size 2 and 4 on CPU.

Each rank owns a column block and its slices of x and g, computes its shard values with the
oracle's canonical trees, and the ranks exchange them over torch.distributed (gloo) as the
engine's allgathers do: the K d values are joined with shard.rank_tree; the packets [x | g |
subtree values of s'z, s's, z'z] give the full x, g and, joined with the same rank tree, the
full canonical dots.  The NCCL unique-id broadcast is the same code the GPU path uses (with
a stand-in id).  (The product itself runs multi-process in tests/test_gpu_shard_mp.py.)
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cases, out):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_0902_4424_b200 import shard as S
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    import torch
    res = {}
    try:
        for (n, p, seed) in cases:
            K = O.gaussian_matrix(seed, n, p)
            rng = np.random.default_rng(seed)
            x = rng.normal(size=p) * (rng.random(p) < 0.1)  # a sparse direction, like d
            r = rng.normal(size=n)
            sh = S.shard_plan(p, world)[rank]
            Ks = np.ascontiguousarray(K[:, sh.cols])
            kd_part = torch.from_numpy(O.apply(Ks, np.ascontiguousarray(x[sh.cols])))
            g_part = torch.from_numpy(O.apply_adjoint(Ks, r))
            # secant dots of this rank's slices (s = x' - x, z = g' - g), subtree values
            sv, zv = x[sh.cols] * 0.5 - x[sh.cols], g_part.numpy() * 1.5 - g_part.numpy()
            dots = torch.tensor([O.dot(sv, zv), O.dot(sv, sv), O.dot(zv, zv)], dtype=torch.float64)
            dots_all = [torch.empty_like(dots) for _ in range(world)]
            dist.all_gather(dots_all, dots)
            kd_all = [torch.empty_like(kd_part) for _ in range(world)]
            g_all = [torch.empty_like(g_part) for _ in range(world)]
            dist.all_gather(kd_all, kd_part)
            dist.all_gather(g_all, g_part)
            kd = S.rank_tree(np.stack([t.numpy() for t in kd_all]))
            g = np.concatenate([t.numpy() for t in g_all])
            sd = S.rank_tree(np.stack([t.numpy() for t in dots_all]))
            s_full, z_full = x * 0.5 - x, g * 1.5 - g
            full_dots = [O.dot(s_full, z_full), O.dot(s_full, s_full), O.dot(z_full, z_full)]
            res[(n, p)] = dict(
                kd_exact=bool(np.array_equal(kd, O.apply(K, x))),
                kd_close=bool(np.allclose(kd, O.apply(K, x), rtol=1e-12, atol=1e-12)),
                g_exact=bool(np.array_equal(g, O.apply_adjoint(K, r))),
                dots_exact=bool(list(sd) == full_dots),
                bit_exact_expected=S.bit_exact(p, world))
        uid = S.exchange_id(dist, rank, make_id=lambda: bytes(range(128)))
        res["uid"] = uid == bytes(range(128))
        dist.barrier()
    finally:
        dist.destroy_process_group()
    out.put((rank, res))


def _run(world, cases):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    return out


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_exchange_matches_unsharded(world):
    cases = [(64, 2048, 3), (33, 4096, 4), (16, 3072, 5)]
    cases = [(n, p, s) for (n, p, s) in cases if p % world == 0 and (p // world) % 256 == 0]
    cases.append((40, 768 * world, 6))  # 768 columns per rank: not a power of two
    out = _run(world, cases)
    for rank, res in out.items():
        assert res["uid"], rank
        for (n, p, _) in cases:
            r = res[(n, p)]
            assert r["g_exact"], (rank, n, p)  # column trees are per column: always exact
            assert r["kd_close"], (rank, n, p)
            if r["bit_exact_expected"]:
                assert r["kd_exact"], (rank, n, p)
                assert r["dots_exact"], (rank, n, p)


def test_shard_plan_rules():
    from paper_0902_4424_b200 import shard as S
    plan = S.shard_plan(32768, 8)
    assert [s.col0 for s in plan] == [r * 4096 for r in range(8)]
    assert all(s.p_local == 4096 for s in plan)
    assert S.bit_exact(32768, 8) and S.bit_exact(262144, 4) and not S.bit_exact(1536, 2)
    assert S.shard_plan(300, 1)[0].p_local == 300  # one rank: no alignment needed
    with pytest.raises(ValueError):
        S.shard_plan(1000, 3)
    with pytest.raises(ValueError):
        S.shard_plan(2 * 300, 2)
    t = np.array([[1.0], [1e16], [-1e16], [1.0]])
    # (a + b) + (c + d): the rank tree order, not a left fold
    assert S.rank_tree(t)[0] == (1.0 + 1e16) + (-1e16 + 1.0) == 0.0
    assert ((1.0 + 1e16) + -1e16) + 1.0 == 1.0
