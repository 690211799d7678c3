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


def _shard_worker(rank, world, port, out_q):
    """ZeRO-1 plane-sharded step on gloo: reduce-scatter of the padded
    gradient planes, each rank keeps the sampler update of its own planes
    (computed here with the fp64 oracle, which updates every plane from the
    pre-update state), all-gather of the parameter planes; the result must
    equal the replicated full step on every rank, bit for bit."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from oracle import oracle as O
    from paper_2503_10148_b200 import dist as D

    D.init(backend="gloo")
    sc = make_custom_scene(300, 2, 16, 16, seed=23)
    P, n = sc.params.shape
    rng = np.random.default_rng(100 + rank)
    g_local = rng.normal(size=(P, n))  # this rank's partial gradient
    pr, (p0, p1) = D.plane_shard(P, rank, world)
    gpad = torch.zeros((pr * world, n), dtype=torch.float64)
    gpad[:P] = torch.from_numpy(g_local)
    scratch = torch.empty((pr, n), dtype=torch.float64)
    mine = D.reduce_scatter_planes_(gpad, scratch)
    # reference gradient: the sum of every rank's partial
    g_all = sum(np.random.default_rng(100 + r).normal(size=(P, n)) for r in range(world))
    ok_rs = bool(np.allclose(mine.numpy()[:p1 - p0], g_all[p0:p1], rtol=1e-14, atol=1e-14))
    hp = sghmc_params_for(sc, step=2, seed=9, eps_o=0.01, eps_sigma=0.01)
    full, *_ = O.sghmc_step(sc.params, 2, g_all, np.zeros((P, n)), np.zeros((P, n)), np.zeros((3, n)), hp)
    ppad = torch.zeros((pr * world, n), dtype=torch.float64)
    ppad[:P] = torch.from_numpy(sc.params.astype(np.float64))
    ppad[p0:p1] = torch.from_numpy(full[p0:p1])  # this rank's planes of the step
    D.all_gather_planes_(ppad, scratch)
    ok_ag = bool(np.array_equal(ppad[:P].numpy(), full))
    out_q.put((rank, (p0, p1), ok_rs, ok_ag))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_plane_sharded_step(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spans = [r[1] for r in res]
    assert spans[0][0] == 0 and all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    for _, _, ok_rs, ok_ag in res:
        assert ok_rs and ok_ag


def test_plane_shard_partition():
    from paper_2503_10148_b200 import dist as D

    for P in (15, 24, 39, 60):
        for R in (1, 2, 3, 4, 8):
            spans = [D.plane_shard(P, r, R)[1] for r in range(R)]
            covered = [p for a, b in spans for p in range(a, b)]
            assert covered == list(range(P))


def _blocked_worker(rank, world, port, out_q):
    """Overlapped exchange on gloo: the gradient in the component-blocked
    layout (api.BlockedParams, sss.h sss_params.block), one reduce-scatter per
    block issued as each block is finished, this rank's planes of every block
    then hold the global sum -- the same values as the plain plane-sharded
    reduce-scatter of the [P][n] buffer; the layout maps back exactly."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from paper_2503_10148_b200 import api as A
    from paper_2503_10148_b200 import dist as D

    D.init(backend="gloo")
    sh, n = 1, 1003  # ragged: the last block is partial
    P = A.n_planes(sh)
    pr, (p0, p1) = D.plane_shard(P, rank, world)
    rng = np.random.default_rng(200 + rank)
    g_local = rng.normal(size=(P, n))
    g_all = sum(np.random.default_rng(200 + r).normal(size=(P, n)) for r in range(world))
    ok = True
    for n_blocks in (1, 3, 8):
        blk = A.BlockedParams.zeros(n, sh, n_blocks, pr * world, "cpu")
        blk.buf = blk.buf.double()
        B = blk.block
        for k in range(n_blocks):  # fill block k as the projection backward would, then exchange it
            i0, i1 = blk.block_range(k)
            blk.buf[k, :P, :i1 - i0] = torch.from_numpy(g_local[:, i0:i1])
            D.reduce_scatter_block_(blk.buf[k])
        got = blk.buf[:, p0:p1, :].permute(1, 0, 2).reshape(p1 - p0, -1)[:, :n].numpy()
        ok = ok and bool(np.allclose(got, g_all[p0:p1], rtol=1e-14, atol=1e-14))
        # to_planes() is the inverse of the block layout on the local data
        fresh = A.BlockedParams.zeros(n, sh, n_blocks, pr * world, "cpu")
        for k in range(n_blocks):
            i0, i1 = fresh.block_range(k)
            fresh.buf[k, :P, :i1 - i0] = torch.from_numpy(g_local[:, i0:i1]).float()
        ok = ok and bool(np.array_equal(fresh.to_planes().numpy(), g_local.astype(np.float32)))
        ok = ok and B * n_blocks >= n
    out_q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_blocked_overlapped_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_blocked_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res)
