"""``helmsolve`` command line (SPEC.md ``[MODULE] bench_cli``).

The reference declares ``helmsolve = "helmsolve.cli:main"`` (``pyproject.toml:15-16``) but ships no
``cli`` module; this implements the SPEC's subcommands over the B200 package:

  solve    one model, one RHS (a point source at the centre by default) -> solution field + JSON report
  bench    sizes x preconditioners, mean FGMRES iterations over num_rhs RHS on an unseen model -> CSV
  datagen  (r, e) training pairs -> pairs.npz + manifest (``--from-manifest`` regenerates a run)
  train    SPEC multiscale training -> checkpoint + loss CSV + manifest
  retrain  out-of-distribution fine-tuning (300 pairs, 30 epochs, lr / 10; PAPER §5.1)

Every run writes a manifest (``schemas/manifest.schema.json``).  Errors exit non-zero with one JSON
object on stderr: {"error": <class>, "message": ...}; configuration errors exit 2, others 1.

Run as ``python -m paper_2306_17486_b200.cli <command> ...``.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

from . import errors, formats

VERSION = "b200-1"


def _manifest(command: str, seed: int, config: dict, outputs: dict | None = None) -> dict:
    return {"kind": "manifest", "command": command, "seed": int(seed), "version": VERSION, "config": config,
            "outputs": outputs or {}}


def _synthetic_model(n: int, seed: int, gamma0: float):
    from . import fields, problems

    k2 = problems.smooth_random_kappa_sq((n, n), max(2.0, n / 21.0), seed)
    return fields.slowness_model(k2, gamma0=gamma0)


def _model(args):
    from . import fields

    if getattr(args, "model", None):
        k2, _ = formats.read_field(args.model)
        return fields.slowness_model(np.real(k2), gamma0=args.gamma0)
    return _synthetic_model(args.synthetic, args.seed, args.gamma0)


def _load_net(path: str):
    from . import network
    from . import train as tr

    if not path:
        raise errors.ConfigurationError("the implicit_net preconditioner needs --checkpoint")
    if not os.path.exists(path):
        raise errors.ConfigurationError(f"checkpoint {path} not found")
    ck = tr.load_checkpoint(path)
    return network.EncoderSolverNet(tr.unflatten(ck["params"], ck["channels"]), ck["channels"])


def _levels_for(net):
    return net.levels if net is not None else 3


# ---------------------------------------------------------------- solve


def cmd_solve(args) -> int:
    from . import krylov

    if not 0 < args.tol <= 1:
        raise errors.ConfigurationError("tol must be in (0, 1]")
    net = _load_net(args.checkpoint) if args.preconditioner == "implicit_net" else None
    model = _model(args)
    nx, ny = model.shape
    if args.rhs:
        b, _ = formats.read_field(args.rhs)
        b = b.astype(np.complex128)
    else:
        b = np.zeros((nx, ny), dtype=np.complex128)
        b[nx // 2, ny // 2] = 1.0 / (model.h * model.h)
    xs, reps = krylov.solve_batch([model], b[None], net=net, tol=args.tol, max_iter=args.max_iter,
                                  restart=args.restart, num_levels=_levels_for(net))
    config = {"nx": nx, "ny": ny, "h": model.h, "preconditioner": args.preconditioner, "tol": args.tol,
              "max_iter": args.max_iter, "restart": args.restart, "seed": args.seed,
              "model": args.model or f"synthetic:{args.synthetic}", "checkpoint": args.checkpoint or None}
    formats.write_field(args.out + ".field", xs[0], model.h)
    formats.write_json(args.out + ".report.json", formats.solve_report(reps[0], config), "report")
    formats.write_json(args.out + ".manifest.json",
                       _manifest("solve", args.seed, config, {"solution": args.out + ".field",
                                                               "report": args.out + ".report.json"}), "manifest")
    print(json.dumps({"iterations": reps[0].iterations, "converged": reps[0].converged}))
    return 0


# ---------------------------------------------------------------- bench


def cmd_bench(args) -> int:
    from . import krylov, problems

    sizes = [int(s) for s in args.sizes.split(",")]
    pres = args.preconditioners.split(",")
    if args.num_rhs < 1:
        raise errors.ConfigurationError("num_rhs must be >= 1")
    net = _load_net(args.checkpoint) if "implicit_net" in pres else None
    rows = []
    for n in sizes:
        model = _synthetic_model(n, 10_000 + args.seed, args.gamma0)  # a model unseen in training
        rhs = problems.complex_gaussian_rhs(model.shape, args.num_rhs, args.seed)
        for pre in pres:
            if pre not in ("v_cycle", "implicit_net"):
                raise errors.ConfigurationError(f"unknown preconditioner {pre}")
            use = net if pre == "implicit_net" else None
            _, reps = krylov.solve_batch([model], rhs, net=use, tol=args.tol, max_iter=args.max_iter,
                                         restart=args.restart, num_levels=_levels_for(use))
            its = [r.iterations if r.converged else args.max_iter for r in reps]
            rows.append((n, pre, float(np.mean(its)), float(np.mean([r.converged for r in reps]))))
    formats.write_bench_csv(args.out, rows)
    config = {"sizes": sizes, "preconditioners": pres, "num_rhs": args.num_rhs, "tol": args.tol,
              "max_iter": args.max_iter, "restart": args.restart, "gamma0": args.gamma0,
              "checkpoint": args.checkpoint or None}
    formats.write_json(args.out + ".manifest.json", _manifest("bench", args.seed, config, {"table": args.out}),
                       "manifest")
    return 0


# ---------------------------------------------------------------- datagen


def _datagen_models(cfg: dict):
    from . import corpus, datagen

    if cfg.get("corpus"):
        return corpus.load_slowness_corpus(cfg["corpus"], target_n=cfg["size"] - 1, gamma0=datagen.TRAINING_GAMMA0)
    return [_synthetic_model(cfg["size"], cfg["seed"] + i, datagen.TRAINING_GAMMA0) for i in range(cfg["models"])]


def generate(cfg: dict):
    """Deterministic (r, e, k, model_of) from a datagen config (the manifest's ``config``)."""
    from . import datagen

    models = _datagen_models(cfg)
    ds = datagen.build_dataset(models, cfg["samples"], cfg["seed"])
    r = np.stack([p.residual.data for p in ds])
    e = np.stack([p.true_error.data for p in ds])
    return models, r, e, np.array([p.iterations for p in ds]), np.array([p.model_id for p in ds])


def cmd_datagen(args) -> int:
    if args.from_manifest:
        cfg = formats.read_json(args.from_manifest, "manifest")["config"]
    else:
        cfg = {"size": args.size, "models": args.models, "samples": args.samples, "seed": args.seed,
               "corpus": args.corpus or None, "k_range": [2, 20], "gamma0": 0.05}
    if cfg["samples"] <= 0:
        raise errors.ConfigurationError("samples_per_epoch must be positive")
    _, r, e, k, owner = generate(cfg)
    os.makedirs(args.out, exist_ok=True)
    data = os.path.join(args.out, "pairs.npz")
    np.savez(data, r=r, e=e, k=k, model_of=owner)
    formats.write_json(os.path.join(args.out, "manifest.json"),
                       _manifest("datagen", cfg["seed"], cfg, {"pairs": data}), "manifest")
    return 0


# ---------------------------------------------------------------- train / retrain


def _read_kv(path: str) -> dict:
    """Flat ``key = value`` config file (SPEC trainer External Interfaces)."""
    out = {}
    with open(path) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            k, _, v = line.partition("=")
            out[k.strip()] = v.strip()
    return out


def _train_config(args):
    from . import train as tr

    kv = _read_kv(args.config) if args.config else {}
    ints = lambda s: tuple(int(x) for x in str(s).split(","))  # noqa: E731
    return tr.TrainConfig(
        sizes=ints(kv.get("sizes", args.sizes)),
        samples_per_epoch=ints(kv.get("samples_per_epoch", args.samples_per_epoch)),
        epochs_per_size_block=int(kv.get("epochs_per_size_block", args.epochs_per_size_block)),
        max_epochs=int(kv.get("max_epochs", args.max_epochs)),
        lr=float(kv.get("lr", args.lr)),
        lr_decay_epochs=int(kv.get("lr_decay_epochs", args.lr_decay_epochs)),
        batch_size=int(kv.get("batch_size", args.batch_size)),
        seed=int(kv.get("seed", args.seed)))


def _corpora(config, models_per_size: int):
    corpora = {}
    for i, n in enumerate(config.sizes):
        cfg = {"size": n, "models": models_per_size, "samples": config.samples_per_epoch[i],
               "seed": config.seed + 97 * i, "corpus": None}
        models, r, e, _, owner = generate(cfg)
        corpora[n] = (models, r, e, owner)
    return corpora


def cmd_train(args) -> int:
    from dataclasses import asdict

    from . import network
    from . import train as tr

    config = _train_config(args)
    channels = tuple(int(c) for c in args.channels.split(","))
    net = _load_net(args.init) if args.init else network.EncoderSolverNet.seeded(channels, seed=config.seed)
    corpora = _corpora(config, args.models)
    os.makedirs(args.out, exist_ok=True)
    ck = os.path.join(args.out, "checkpoint.ckpt")
    trained, hist = tr.train(net, config, corpora, checkpoint=ck)
    tr.save_checkpoint(ck, hist.state, trained.channels)
    with open(os.path.join(args.out, "loss.csv"), "w") as f:
        f.write(hist.csv())
    cfg = asdict(config)
    cfg.update({"channels": list(channels), "models_per_size": args.models, "init": args.init or None})
    formats.write_json(os.path.join(args.out, "manifest.json"),
                       _manifest("train", config.seed, cfg, {"checkpoint": ck, "loss": os.path.join(args.out, "loss.csv")}),
                       "manifest")
    return 0


def cmd_retrain(args) -> int:
    """PAPER §5.1: 300 pairs on the OOD model (prepared at half resolution), 30 epochs at lr / 10."""
    from . import datagen, fields
    from . import train as tr

    net = _load_net(args.checkpoint)
    model = _model(args)
    model = fields.slowness_model(model.kappa_sq, gamma0=datagen.TRAINING_GAMMA0)
    gen = datagen.PairGenerator([model], num_levels=net.levels)
    rng = np.random.default_rng(args.seed)
    draws = [datagen._draw(rng, model.shape) for _ in range(args.pairs)]
    r, e = gen.pairs(np.stack([d[0] for d in draws]), [d[1] for d in draws], [0] * args.pairs)
    config = tr.TrainConfig(sizes=(model.shape[0],), samples_per_epoch=(args.pairs,), epochs_per_size_block=args.epochs,
                            max_epochs=args.epochs, lr=args.lr, lr_decay_epochs=10 ** 9,
                            batch_size=min(args.batch_size, args.pairs), seed=args.seed)
    trained, hist = tr.train(net, config, {model.shape[0]: ([model], r, e, np.zeros(args.pairs, dtype=int))})
    os.makedirs(args.out, exist_ok=True)
    ck = os.path.join(args.out, "checkpoint.ckpt")
    tr.save_checkpoint(ck, hist.state, trained.channels)
    with open(os.path.join(args.out, "loss.csv"), "w") as f:
        f.write(hist.csv())
    formats.write_json(os.path.join(args.out, "manifest.json"),
                       _manifest("retrain", args.seed, {"base": args.checkpoint, "pairs": args.pairs, "epochs": args.epochs,
                                                        "lr": args.lr, "model": args.model or f"synthetic:{args.synthetic}"},
                                 {"checkpoint": ck}), "manifest")
    return 0


# ---------------------------------------------------------------- entry point


def parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="helmsolve", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="command", required=True)

    def model_args(p):
        p.add_argument("--model", help="kappa^2 field file (formats.write_field)")
        p.add_argument("--synthetic", type=int, default=129, help="node count of a seeded synthetic model")
        p.add_argument("--gamma0", type=float, default=0.01)
        p.add_argument("--seed", type=int, default=0)

    p = sub.add_parser("solve")
    model_args(p)
    p.add_argument("--preconditioner", default="v_cycle", choices=["v_cycle", "implicit_net"])
    p.add_argument("--checkpoint")
    p.add_argument("--rhs", help="complex RHS field file (default: a point source at the centre)")
    p.add_argument("--tol", type=float, default=1e-7)
    p.add_argument("--max-iter", type=int, default=250)
    p.add_argument("--restart", type=int, default=10)
    p.add_argument("--out", required=True, help="output prefix")
    p.set_defaults(fn=cmd_solve)

    p = sub.add_parser("bench")
    p.add_argument("--sizes", default="129")
    p.add_argument("--preconditioners", default="v_cycle")
    p.add_argument("--checkpoint")
    p.add_argument("--num-rhs", type=int, default=20)
    p.add_argument("--tol", type=float, default=1e-7)
    p.add_argument("--max-iter", type=int, default=250)
    p.add_argument("--restart", type=int, default=10)
    p.add_argument("--gamma0", type=float, default=0.01)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", required=True, help="CSV path")
    p.set_defaults(fn=cmd_bench)

    p = sub.add_parser("datagen")
    p.add_argument("--size", type=int, default=65)
    p.add_argument("--models", type=int, default=2)
    p.add_argument("--samples", type=int, default=64)
    p.add_argument("--corpus")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--from-manifest")
    p.add_argument("--out", required=True, help="output directory")
    p.set_defaults(fn=cmd_datagen)

    p = sub.add_parser("train")
    p.add_argument("--config", help="flat key = value TrainConfig file")
    p.add_argument("--sizes", default="65")
    p.add_argument("--samples-per-epoch", default="64")
    p.add_argument("--epochs-per-size-block", type=int, default=20)
    p.add_argument("--max-epochs", type=int, default=2)
    p.add_argument("--lr", type=float, default=1e-3)
    p.add_argument("--lr-decay-epochs", type=int, default=100)
    p.add_argument("--batch-size", type=int, default=16)
    p.add_argument("--channels", default="16,32,64")
    p.add_argument("--models", type=int, default=2)
    p.add_argument("--init", help="start from this checkpoint")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", required=True, help="output directory")
    p.set_defaults(fn=cmd_train)

    p = sub.add_parser("retrain")
    model_args(p)
    p.add_argument("--checkpoint", required=True)
    p.add_argument("--pairs", type=int, default=300)
    p.add_argument("--epochs", type=int, default=30)
    p.add_argument("--lr", type=float, default=1e-4)
    p.add_argument("--batch-size", type=int, default=16)
    p.add_argument("--out", required=True)
    p.set_defaults(fn=cmd_retrain)
    return ap


def main(argv=None) -> int:
    args = parser().parse_args(argv)
    try:
        return int(args.fn(args) or 0)
    except errors.ConfigurationError as exc:
        print(json.dumps({"error": type(exc).__name__, "message": str(exc)}), file=sys.stderr)
        return 2
    except Exception as exc:  # noqa: BLE001 - the CLI contract: machine-readable error, non-zero exit
        print(json.dumps({"error": type(exc).__name__, "message": str(exc)}), file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
