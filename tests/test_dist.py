"""The N > 1 data-parallel plumbing on CPU: world_size 2 over gloo (no GPU)."""
import os
import socket

import numpy as np
import pytest

from paper_2306_17486_b200 import dist as hdist
from paper_2306_17486_b200 import problems


def test_shard_range_covers_everything_once():
    for n in (0, 1, 7, 128, 129):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                a, b = hdist.shard_range(n, world, r)
                seen.extend(range(a, b))
            assert seen == list(range(n))
    with pytest.raises(ValueError):
        hdist.shard_range(4, 2, 2)


def test_rank_instances_are_distinct_and_same_shaped():
    a = problems.make_config("C1", seed_offset=0)
    b = problems.make_config("C1", seed_offset=1)
    assert a.rhs.shape == b.rhs.shape and a.shape == b.shape
    assert not np.array_equal(a.models[0].kappa_sq, b.models[0].kappa_sq)
    # seed offset 0 reproduces the fixtures' inputs
    c = problems.make_config("C1")
    assert np.array_equal(a.models[0].kappa_sq, c.models[0].kappa_sq)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # each rank owns an independent instance and a shard of its RHS (no data-path collective)
        cfg = problems.make_config("C1", seed_offset=rank)
        lo, hi = hdist.shard_range(cfg.rhs.shape[0], world, rank)
        local = [(rank, i, float(np.abs(cfg.rhs[i]).sum())) for i in range(lo, hi)]
        t = hdist.reduce_scalar(1.5 + rank, "max")
        s = hdist.reduce_scalar(len(local), "sum")
        allr = hdist.gather_reports(local)
        q.put((rank, t, s, allr))
    finally:
        dist.destroy_process_group()


def test_gloo_world_size_two():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t, s, allr in res:
        assert t == 2.5  # max over ranks
        assert s == 4  # C1 has 4 RHS: 2 per rank
        assert [r for r, _, _ in allr] == [0, 0, 1, 1]
    assert res[0][3] == res[1][3]


def _train_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from oracle import train_oracle as to
    from paper_2306_17486_b200 import netparams
    from paper_2306_17486_b200 import train as tr
    from conftest import golden

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # data-parallel training step: each rank's gradient of ITS shard, averaged by the all-reduce
        g = golden("train.npz")
        ch = tuple(int(c) for c in g["channels_a"])
        names = [n for n, *_ in netparams.param_spec(ch)]
        params = {n: g[f"p_a_{n}"].copy() for n in names}
        sl = slice(rank, rank + 1)  # ranks 0 and 1 take samples 0 and 1
        loss, grads, _ = to.loss_and_grads(params, int(g["levels_a"]), g["media_a"][sl], g["r_a"][sl], g["e_a"][sl],
                                           float(g["h_a"]))
        vec = torch.from_numpy(tr.flatten({**params, **grads}, ch).astype(np.float32))
        hdist.allreduce_mean(vec)
        mean_loss = hdist.reduce_scalar(loss, "sum") / hdist.world_size()
        q.put((rank, vec.numpy(), mean_loss))
    finally:
        dist.destroy_process_group()


def test_gloo_data_parallel_gradient_average():
    import multiprocessing as mp

    from conftest import golden
    from oracle import train_oracle as to
    from paper_2306_17486_b200 import netparams
    from paper_2306_17486_b200 import train as tr

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_train_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # serial reference: the mean of the two per-sample gradients
    g = golden("train.npz")
    ch = tuple(int(c) for c in g["channels_a"])
    names = [n for n, *_ in netparams.param_spec(ch)]
    vecs, losses = [], []
    for r in range(2):
        params = {n: g[f"p_a_{n}"].copy() for n in names}
        sl = slice(r, r + 1)
        loss, grads, _ = to.loss_and_grads(params, int(g["levels_a"]), g["media_a"][sl], g["r_a"][sl], g["e_a"][sl],
                                           float(g["h_a"]))
        vecs.append(tr.flatten({**params, **grads}, ch).astype(np.float32))
        losses.append(loss)
    want = (vecs[0] + vecs[1]) / 2
    for rank, vec, mean_loss in res:
        assert np.allclose(vec, want, rtol=1e-6, atol=1e-7)
        assert mean_loss == pytest.approx(np.mean(losses), rel=1e-12)
    assert np.array_equal(res[0][1], res[1][1])  # every rank holds the same averaged vector
