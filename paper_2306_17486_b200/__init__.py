"""B200-native Helmholtz FGMRES hot path of arXiv 2306.17486 (drop-in for ``helmsolve``).

Submodules mirror the reference package: ``errors``, ``fields``, ``multigrid``,
``krylov``, ``green``, ``network`` (the module the reference imports but never
shipped), plus ``engine`` (batched device solve) and ``problems`` (seeded
BASELINE inputs).  Compute runs in the in-tree C-ABI library
``libhelmsolve_b200.so`` (sm_100a); there is no CPU fallback.
"""
__all__ = ["errors", "fields", "multigrid", "krylov", "green", "network", "engine", "problems", "netparams"]
