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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_problem():
    """A small two-model batch of 5 RHS at 33^2 (the oracle stands in for the device solver on CPU)."""
    from oracle import helm_oracle as ho

    rng = np.random.default_rng(7)
    models = [ho.make_model(problems.smooth_random_kappa_sq((33, 33), 3.0, s), layer_width=4) for s in (1, 2)]
    rhs = rng.standard_normal((5, 33, 33)) + 1j * rng.standard_normal((5, 33, 33))
    owner = np.array([0, 1, 1, 0, 1])
    return models, rhs, owner


def _oracle_solve_fn(models):
    from oracle import helm_oracle as ho
    from paper_2306_17486_b200.krylov import SolveReport

    def solve(rhs, owner):
        xs, reps = [], []
        for b, o in zip(rhs, owner):
            x, r = ho.solve_vcycle(models[int(o)], b, None, 1e-6, 200, 10)
            xs.append(x)
            reps.append(SolveReport(r.iterations, list(r.history), r.converged))
        return np.array(xs), reps

    return solve


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # the bench's exact shard-and-gather path: this rank solves its share of ONE batch, the per-RHS
        # reports are all-gathered in batch order; the max-over-ranks timing reduction
        models, rhs, owner = _oracle_problem()
        rows, x, (lo, hi) = hdist.sharded_solve(_oracle_solve_fn(models), rhs, owner)
        t = hdist.reduce_scalar(1.5 + rank, "max")
        s = hdist.reduce_scalar(hi - lo, "sum")
        q.put((rank, t, s, rows, (lo, hi), x))
    finally:
        dist.destroy_process_group()


def test_gloo_sharded_solve_equals_one_rank():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    models, rhs, owner = _oracle_problem()
    rows1, x1, span1 = hdist.sharded_solve(_oracle_solve_fn(models), rhs, owner)  # no process group: one rank
    assert span1 == (0, 5)
    for rank, t, s, rows, (lo, hi), x in res:
        assert t == 2.5  # max over ranks
        assert s == 5  # every RHS solved exactly once
        assert (lo, hi) == hdist.shard_range(5, 2, rank)
        assert rows == rows1  # gathered reports == the one-rank run, in batch order
        assert np.array_equal(x, x1[lo:hi])
    assert [r[4] for r in res] == [(0, 3), (3, 5)]


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


def test_bench_gpus_relaunches_under_torchrun(monkeypatch):
    # `python bench.py --gpus N` without a torchrun environment re-launches itself with N ranks
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2", "--warmup", "3"])
    assert bench.main() == 0
    cmd = calls[0]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-6:] == ["--gpus", "4", "--steps", "2", "--warmup", "3"]
