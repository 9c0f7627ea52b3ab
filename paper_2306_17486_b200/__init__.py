"""B200-native Helmholtz FGMRES hot path of arXiv 2306.17486 (drop-in for ``helmsolve``).

Submodules mirror the reference package: ``errors``, ``fields``, ``multigrid``,
``krylov``, ``green``, ``network`` (the module the reference imports but never
shipped), plus ``engine`` (batched device solve), ``problems`` (seeded BASELINE
inputs) and ``dist`` (data-parallel plumbing).  Compute runs in the in-tree
C-ABI library ``libhelmsolve_b200.so`` (sm_100a); there is no CPU fallback.
"""
import importlib
import sys

__all__ = ["errors", "fields", "multigrid", "krylov", "green", "network", "engine", "problems", "netparams",
           "dist", "datagen", "train", "corpus", "formats", "cli", "install_as_helmsolve"]

# the reference's modules plus the ones its SPEC / pyproject name but it never shipped
# (network: krylov.py:201; cli: pyproject.toml:15-16; datagen / trainer: SPEC.md:395-507)
_MIRRORED = ("errors", "fields", "multigrid", "krylov", "green", "network", "cli", "datagen", "train")


def install_as_helmsolve() -> None:
    """Register this package as ``helmsolve`` (and ``helmsolve.<module>``) in sys.modules.

    Code written against the reference (``from helmsolve.krylov import ...``)
    then runs on the B200 path unchanged.
    """
    pkg = sys.modules[__name__]
    sys.modules["helmsolve"] = pkg
    for name in _MIRRORED:
        sys.modules[f"helmsolve.{name}"] = importlib.import_module(f"{__name__}.{name}")
