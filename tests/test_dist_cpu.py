"""Multi-process view-parallel logic on CPU (gloo, world_size 2).

The CUDA kernels need a GPU; here the per-view gradients come from the fp64
oracle, so what is tested is the host-side data-parallel plumbing of
paper_2503_10148_b200.dist: the round-robin view shard, the flat-buffer sum
all-reduce, the identical replicated sampler step (same Philox counters) and
the replica checksum.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from sss_synth import make_custom_scene, make_targets, sghmc_params_for


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from oracle import oracle as O
    from paper_2503_10148_b200 import dist as D

    D.init(backend="gloo")
    sc = make_custom_scene(250, 1, 40, 32, n_views=4, seed=17, p_negative=0.3)
    tg = make_targets(sc)
    mine = D.shard_views(sc.n_views, rank, world)
    g = np.zeros(sc.params.shape)
    for v in mine:
        fr = O.render(sc.params, 1, sc.cameras[v], mode="tiled")
        _, dl = O.l1_loss_and_grad(fr.rgb, tg[v])
        g += O.backward(sc.params, 1, sc.cameras[v], dl, mode="tiled")[0]
    flat = torch.from_numpy(g.copy())
    D.allreduce_sum_(flat)
    # reference: every view on this rank alone
    ref = np.zeros_like(g)
    for v in range(sc.n_views):
        fr = O.render(sc.params, 1, sc.cameras[v], mode="tiled")
        _, dl = O.l1_loss_and_grad(fr.rgb, tg[v])
        ref += O.backward(sc.params, 1, sc.cameras[v], dl, mode="tiled")[0]
    ok_sum = bool(np.allclose(flat.numpy(), ref, rtol=1e-12, atol=1e-15))
    # the replicated sampler step keeps replicas bit-identical
    P, n = sc.params.shape
    hp = sghmc_params_for(sc, step=3, seed=11)
    p2, _, _, _ = O.sghmc_step(sc.params, 1, flat.numpy(), np.zeros((P, n)), np.zeros((P, n)),
                               np.zeros((3, n)), hp)
    same = D.replicas_identical(torch.from_numpy(p2))
    # a rank that diverges is detected
    bad = torch.from_numpy(p2.copy())
    if rank == 1:
        bad[0, 0] += 1e-9
    diverged = not D.replicas_identical(bad)
    mx = D.allreduce_max(float(rank) + 0.5)
    out_q.put((rank, mine, ok_sum, same, diverged, mx))
    dist.destroy_process_group()


def test_view_parallel_gradient_sum_and_replicas():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [[0, 2], [1, 3]]
    for _, _, ok_sum, same, diverged, mx in res:
        assert ok_sum and same and diverged
        assert mx == 1.5


def test_shard_views_partitions():
    from paper_2503_10148_b200 import dist as D

    for V in (1, 8, 64, 7):
        for R in (1, 2, 4, 8):
            parts = [D.shard_views(V, r, R) for r in range(R)]
            flat = sorted(v for p in parts for v in p)
            assert flat == list(range(V))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_checksum_is_bitwise():
    from paper_2503_10148_b200 import dist as D

    a = torch.randn(1000)
    b = a.clone()
    assert D.replica_checksum(a) == D.replica_checksum(b)
    b[17] = torch.nextafter(b[17], torch.tensor(10.0))
    assert D.replica_checksum(a) != D.replica_checksum(b)
