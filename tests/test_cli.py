"""CLI and on-disk formats, CPU side (SPEC.md bench_cli)."""
import json

import numpy as np
import pytest

from paper_2306_17486_b200 import cli, formats
from paper_2306_17486_b200.errors import ConfigurationError, DimensionError


@pytest.mark.parametrize("dtype", ["complex128", "complex64", "float64", "float32"])
def test_field_file_round_trip(tmp_path, rng, dtype):
    a = rng.standard_normal((5, 7))
    if dtype.startswith("complex"):
        a = a + 1j * rng.standard_normal((5, 7))
    a = a.astype(dtype)
    p = str(tmp_path / "f.field")
    formats.write_field(p, a, 0.125)
    b, h = formats.read_field(p)
    assert h == 0.125 and b.dtype == a.dtype and np.array_equal(a, b)
    head = open(p, "rb").read().split(b"\n\n")[0].decode()
    assert head.splitlines() == [formats.MAGIC, "nx 5", "ny 7", "h 0.125", f"dtype {dtype}"]


def test_field_file_errors(tmp_path):
    p = str(tmp_path / "bad.field")
    open(p, "wb").write(b"not a field\n\n")
    with pytest.raises(ConfigurationError):
        formats.read_field(p)
    formats.write_field(p, np.zeros((3, 3)), 1.0)
    blob = open(p, "rb").read()
    open(p, "wb").write(blob[:-8])  # truncated grid
    with pytest.raises(DimensionError):
        formats.read_field(p)
    with pytest.raises(DimensionError):
        formats.write_field(p, np.zeros(3), 1.0)


class Rep:
    iterations, converged, relative_residual_history, wall_time = 2, True, [1.0, 0.1, 1e-8], 0.5


CFG = {"nx": 33, "ny": 33, "h": 1 / 32, "preconditioner": "v_cycle", "tol": 1e-7, "max_iter": 250, "restart": 10}


def test_report_schema(tmp_path):
    doc = formats.solve_report(Rep(), dict(CFG))
    p = str(tmp_path / "r.json")
    formats.write_json(p, doc, "report")
    assert formats.read_json(p, "report") == json.loads(json.dumps(doc))
    bad = dict(doc, relative_residual_history=[])
    with pytest.raises(ConfigurationError):
        formats.validate(bad, "report")
    bad = dict(doc, config=dict(CFG, preconditioner="explicit"))
    with pytest.raises(ConfigurationError):
        formats.validate(bad, "report")


def test_manifest_schema():
    formats.validate(cli._manifest("datagen", 3, {"size": 65}), "manifest")
    with pytest.raises(ConfigurationError):
        formats.validate(cli._manifest("plot", 3, {}), "manifest")


def test_bench_csv_round_trip(tmp_path):
    p = str(tmp_path / "t.csv")
    rows = [(129, "v_cycle", 112.9, 1.0), (257, "implicit_net", 250.0, 0.85)]
    formats.write_bench_csv(p, rows)
    assert open(p).readline().strip() == "size,preconditioner,mean_iters,converged_fraction"
    assert formats.read_bench_csv(p) == rows


def test_kv_config(tmp_path):
    p = tmp_path / "train.cfg"
    p.write_text("# desk scale\nsizes = 65,129\nsamples_per_epoch = 2000,500\nlr = 0.001\nmax_epochs = 30\n")
    args = cli.parser().parse_args(["train", "--config", str(p), "--out", str(tmp_path)])
    cfg = cli._train_config(args)
    assert cfg.sizes == (65, 129) and cfg.samples_per_epoch == (2000, 500) and cfg.max_epochs == 30


def test_errors_are_machine_readable(capsys, tmp_path):
    # a net preconditioner without a checkpoint is a configuration error (exit 2), before any device work
    rc = cli.main(["solve", "--preconditioner", "implicit_net", "--out", str(tmp_path / "x")])
    assert rc == 2
    err = json.loads(capsys.readouterr().err.strip())
    assert err["error"] == "ConfigurationError" and "checkpoint" in err["message"]
    rc = cli.main(["datagen", "--samples", "0", "--out", str(tmp_path / "d")])
    assert rc == 2
    rc = cli.main(["solve", "--tol", "0", "--out", str(tmp_path / "x")])
    assert rc == 2


def test_checkpoint_manifest_and_blob(tmp_path):
    # text manifest (names, shapes, dtypes, architecture hash, training metadata) + a flat
    # little-endian float32 blob in manifest order; atomic; round-1 .npz checkpoints still load
    from paper_2306_17486_b200 import netparams
    from paper_2306_17486_b200 import train as tr

    ch = (4, 8, 8)
    params = tr.flatten(netparams.init_params(ch, seed=3), ch)
    rng = np.random.default_rng(0)
    state = {"params": params, "m": rng.standard_normal(params.size).astype(np.float32),
             "v": rng.random(params.size).astype(np.float32), "step": 7, "lr": 1e-3}
    path = str(tmp_path / "ck.ckpt")
    tr.save_checkpoint(path, state, ch)
    text = open(path).read()
    assert text.startswith("format: helmsolve-checkpoint v1")
    assert "tensor: param sol.implicit.w shape=4x3x3 dtype=complex64 as (re, im) float32 pairs" in text
    blob = np.fromfile(path + ".bin", dtype="<f4")
    assert blob.size == 3 * params.size and np.array_equal(blob[: params.size], params)
    back = tr.load_checkpoint(path)
    assert back["channels"] == ch and back["step"] == 7 and back["lr"] == 1e-3
    for k in ("params", "m", "v"):
        assert np.array_equal(back[k], state[k])
    with pytest.raises(Exception):
        tr.save_checkpoint(path, {**state, "params": params[:-1]}, ch)
    old = str(tmp_path / "old.npz")
    np.savez(old, params=params, m=state["m"], v=state["v"], step=3, lr=0.5, channels=np.asarray(ch))
    assert np.array_equal(tr.load_checkpoint(old)["params"], params)
