"""CLI end to end on the GPU (SPEC.md bench_cli examples)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import helm_oracle as ho  # noqa: E402
from paper_2306_17486_b200 import cli, formats  # noqa: E402
from paper_2306_17486_b200 import train as tr  # noqa: E402


def test_solve_writes_solution_and_report(tmp_path):
    out = str(tmp_path / "run")
    assert cli.main(["solve", "--synthetic", "65", "--tol", "1e-7", "--out", out]) == 0
    x, h = formats.read_field(out + ".field")
    rep = formats.read_json(out + ".report.json", "report")
    formats.read_json(out + ".manifest.json", "manifest")
    assert rep["converged"] and rep["iterations"] == len(rep["relative_residual_history"]) - 1
    # the written solution solves the written problem (oracle operator, fp64)
    m = cli._synthetic_model(65, 0, 0.01)
    b = np.zeros(m.shape, dtype=complex)
    b[32, 32] = 1.0 / (m.h * m.h)
    res = np.linalg.norm(b - ho.helmholtz(x, ho.Model(m.kappa_sq, m.gamma, m.omega, m.h))) / np.linalg.norm(b)
    assert res <= 1e-7 * 1.001 and res == pytest.approx(rep["relative_residual_history"][-1], rel=1e-6)
    # a model file and an RHS file give the same answer
    formats.write_field(str(tmp_path / "k2.field"), m.kappa_sq, m.h)
    formats.write_field(str(tmp_path / "b.field"), b, m.h)
    out2 = str(tmp_path / "run2")
    assert cli.main(["solve", "--model", str(tmp_path / "k2.field"), "--rhs", str(tmp_path / "b.field"),
                     "--out", out2]) == 0
    x2, _ = formats.read_field(out2 + ".field")
    assert np.array_equal(x, x2)


def test_solve_tol_one_needs_no_iterations(tmp_path):
    out = str(tmp_path / "t1")
    assert cli.main(["solve", "--synthetic", "33", "--tol", "1", "--out", out]) == 0
    assert formats.read_json(out + ".report.json", "report")["iterations"] == 0


def test_bench_table(tmp_path):
    out = str(tmp_path / "bench.csv")
    assert cli.main(["bench", "--sizes", "33,65", "--num-rhs", "3", "--out", out]) == 0
    rows = formats.read_bench_csv(out)
    assert [(r[0], r[1]) for r in rows] == [(33, "v_cycle"), (65, "v_cycle")]
    assert all(0 < r[2] < 250 and r[3] == 1.0 for r in rows)
    assert cli.main(["bench", "--sizes", "33", "--num-rhs", "3", "--out", out + "2"]) == 0
    assert formats.read_bench_csv(out + "2")[0] == rows[0]  # deterministic


def test_datagen_manifest_regenerates(tmp_path):
    a, b = str(tmp_path / "a"), str(tmp_path / "b")
    assert cli.main(["datagen", "--size", "33", "--models", "2", "--samples", "6", "--seed", "4", "--out", a]) == 0
    assert cli.main(["datagen", "--from-manifest", os.path.join(a, "manifest.json"), "--out", b]) == 0
    pa, pb = np.load(os.path.join(a, "pairs.npz")), np.load(os.path.join(b, "pairs.npz"))
    for k in ("r", "e", "k", "model_of"):
        assert np.array_equal(pa[k], pb[k]), k
    assert pa["r"].shape == (6, 33, 33) and set(pa["k"]) <= set(range(2, 21))


def test_train_lr_zero_checkpoint_equals_init(tmp_path):
    out = str(tmp_path / "t")
    rc = cli.main(["train", "--sizes", "33", "--samples-per-epoch", "8", "--batch-size", "4", "--max-epochs", "3",
                   "--lr", "0", "--channels", "8,16", "--models", "1", "--out", out])
    assert rc == 0
    ck = tr.load_checkpoint(os.path.join(out, "checkpoint.ckpt"))
    from paper_2306_17486_b200 import netparams

    p0 = tr.flatten(netparams.init_params((8, 16), 0), (8, 16))
    got = tr.unflatten(ck["params"], (8, 16))
    ref = tr.unflatten(p0, (8, 16))
    for k in ref:
        if not (k.endswith(".bn.mean") or k.endswith(".bn.var")):
            assert np.array_equal(got[k], ref[k]), k
    lines = open(os.path.join(out, "loss.csv")).read().strip().splitlines()
    assert lines[0] == "epoch,size,train_mse,val_mse,lr" and len(lines) == 1 + 3  # one row per epoch
    formats.read_json(os.path.join(out, "manifest.json"), "manifest")


def test_retrain_runs(tmp_path):
    out = str(tmp_path / "t")
    assert cli.main(["train", "--sizes", "33", "--samples-per-epoch", "8", "--batch-size", "4", "--max-epochs", "1",
                     "--channels", "8,16", "--models", "1", "--out", out]) == 0
    ck = os.path.join(out, "checkpoint.ckpt")
    out2 = str(tmp_path / "r")
    assert cli.main(["retrain", "--checkpoint", ck, "--synthetic", "33", "--seed", "5", "--pairs", "8",
                     "--epochs", "2", "--batch-size", "4", "--out", out2]) == 0
    assert os.path.exists(os.path.join(out2, "checkpoint.ckpt"))
    # the retrained network drives a learned solve through the CLI
    out3 = str(tmp_path / "s")
    assert cli.main(["solve", "--synthetic", "33", "--preconditioner", "implicit_net", "--checkpoint",
                     os.path.join(out2, "checkpoint.ckpt"), "--tol", "1e-6", "--out", out3]) == 0
    rep = formats.read_json(out3 + ".report.json", "report")
    assert rep["converged"]
