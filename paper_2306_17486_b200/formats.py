"""On-disk formats around the solve path (SPEC.md ``[MODULE] bench_cli``).

The reference declares a ``helmsolve`` console script and ``schemas/*.json`` package data
(``pyproject.toml:15-22``) but ships neither; the formats here follow SPEC.md's External Interfaces:

* field file: a text header (``nx``, ``ny``, ``h``, ``dtype``), a blank line, then the raw
  little-endian grid in C order (``data[ix, iy]``, fields.py:5-12);
* solve report: JSON (iterations, converged, relative-residual history, config echo),
  validated against ``schemas/report.schema.json``;
* run manifest: JSON capturing the full config and seed of a datagen / train / bench run
  (``schemas/manifest.schema.json``), enough to regenerate the run;
* bench table: CSV ``size,preconditioner,mean_iters,converged_fraction``; loss history CSV
  ``epoch,size,train_mse,val_mse,lr``.
"""
from __future__ import annotations

import json
import os

import numpy as np

from .errors import ConfigurationError, DimensionError

MAGIC = "helmsolve-field v1"
SCHEMA_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "schemas")
_DTYPES = {"complex128": "<c16", "complex64": "<c8", "float64": "<f8", "float32": "<f4"}
BENCH_COLUMNS = ("size", "preconditioner", "mean_iters", "converged_fraction")


def write_field(path: str, values, h: float):
    """Text header + raw little-endian grid; written atomically (temp file, rename)."""
    a = np.asarray(values)
    if a.ndim != 2:
        raise DimensionError(f"a field is 2-D, got shape {a.shape}")
    name = a.dtype.name
    if name not in _DTYPES:
        raise ConfigurationError(f"unsupported field dtype {name}")
    head = f"{MAGIC}\nnx {a.shape[0]}\nny {a.shape[1]}\nh {float(h)!r}\ndtype {name}\n\n".encode()
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(head)
        f.write(np.ascontiguousarray(a, dtype=_DTYPES[name]).tobytes())
    os.replace(tmp, path)


def read_field(path: str):
    """-> (array, h)."""
    with open(path, "rb") as f:
        blob = f.read()
    sep = blob.find(b"\n\n")
    if sep < 0 or not blob.startswith(MAGIC.encode()):
        raise ConfigurationError(f"{path}: not a {MAGIC} file")
    meta = {}
    for line in blob[:sep].decode().splitlines()[1:]:
        k, _, v = line.partition(" ")
        meta[k] = v
    try:
        nx, ny, h, dtype = int(meta["nx"]), int(meta["ny"]), float(meta["h"]), meta["dtype"]
    except (KeyError, ValueError) as exc:
        raise ConfigurationError(f"{path}: bad header ({exc})") from None
    if dtype not in _DTYPES:
        raise ConfigurationError(f"{path}: unsupported dtype {dtype}")
    raw = blob[sep + 2:]
    a = np.frombuffer(raw, dtype=_DTYPES[dtype])
    if a.size != nx * ny:
        raise DimensionError(f"{path}: {a.size} values for a {nx}x{ny} header")
    return a.reshape(nx, ny).astype(dtype), h


def load_schema(name: str) -> dict:
    with open(os.path.join(SCHEMA_DIR, f"{name}.schema.json")) as f:
        return json.load(f)


def validate(doc: dict, name: str):
    """Validate against schemas/<name>.schema.json (jsonschema when installed, else the subset used)."""
    schema = load_schema(name)
    try:
        import jsonschema
    except ImportError:  # pragma: no cover - jsonschema is in the image
        _validate_subset(doc, schema, name)
        return
    try:
        jsonschema.validate(doc, schema)
    except jsonschema.ValidationError as exc:
        raise ConfigurationError(f"{name}: {exc.message}") from None


def _validate_subset(doc, schema, where):
    types = {"object": dict, "array": list, "string": str, "integer": int, "number": (int, float), "boolean": bool}
    t = schema.get("type")
    if t and not isinstance(doc, types[t]):
        raise ConfigurationError(f"{where}: expected {t}")
    if t == "object":
        for k in schema.get("required", []):
            if k not in doc:
                raise ConfigurationError(f"{where}: missing {k}")
        for k, sub in schema.get("properties", {}).items():
            if k in doc:
                _validate_subset(doc[k], sub, f"{where}.{k}")
    if t == "array" and "items" in schema:
        for i, v in enumerate(doc):
            _validate_subset(v, schema["items"], f"{where}[{i}]")


def write_json(path: str, doc: dict, schema: str | None = None):
    if schema:
        validate(doc, schema)
    tmp = path + ".tmp"
    with open(tmp, "w") as f:
        json.dump(doc, f, indent=1, sort_keys=True)
        f.write("\n")
    os.replace(tmp, path)


def read_json(path: str, schema: str | None = None) -> dict:
    with open(path) as f:
        doc = json.load(f)
    if schema:
        validate(doc, schema)
    return doc


def solve_report(report, config: dict) -> dict:
    """SolveReport (krylov.py:19-26) + config echo as the report document."""
    return {"kind": "solve_report", "iterations": int(report.iterations), "converged": bool(report.converged),
            "relative_residual_history": [float(v) for v in report.relative_residual_history],
            "wall_time": float(getattr(report, "wall_time", 0.0)), "config": config}


def write_bench_csv(path: str, rows):
    lines = [",".join(BENCH_COLUMNS)]
    for size, pre, mean_iters, frac in rows:
        lines.append(f"{int(size)},{pre},{float(mean_iters):.4f},{float(frac):.4f}")
    tmp = path + ".tmp"
    with open(tmp, "w") as f:
        f.write("\n".join(lines) + "\n")
    os.replace(tmp, path)


def read_bench_csv(path: str):
    with open(path) as f:
        head, *body = [ln.strip() for ln in f if ln.strip()]
    if tuple(head.split(",")) != BENCH_COLUMNS:
        raise ConfigurationError(f"{path}: columns {head} != {','.join(BENCH_COLUMNS)}")
    out = []
    for ln in body:
        s, p, m, c = ln.split(",")
        out.append((int(s), p, float(m), float(c)))
    return out
