"""Host-side logic (no GPU): problem generators, parameter layout, hierarchy setup, drop-in shim."""
import numpy as np
import pytest

from paper_2306_17486_b200 import fields, multigrid, netparams, problems
from paper_2306_17486_b200.errors import ConfigurationError, DimensionError, SingularityError


def test_config_shapes_match_baseline():
    c1 = problems.make_config("C1")
    assert c1.shape == (129, 129) and c1.rhs.shape == (4, 129, 129)
    assert c1.models[0].omega == pytest.approx(80.384)  # test_fields.py:86-91 style KAT
    c2 = problems.make_config("C2", rhs_per_model=2)
    assert c2.shape == (257, 257) and len(c2.models) == 4 and c2.rhs.shape[0] == 8
    assert list(c2.model_of_rhs) == [0, 0, 1, 1, 2, 2, 3, 3]
    for m in c2.models:
        assert m.kappa_sq.min() == pytest.approx(0.25) and m.kappa_sq.max() == pytest.approx(1.0)


def test_generators_are_seeded():
    a = problems.smooth_random_kappa_sq((33, 40), 3.0, 5)
    b = problems.smooth_random_kappa_sq((33, 40), 3.0, 5)
    assert np.array_equal(a, b)
    assert problems.gaussian_smooth(np.full((9, 9), 2.0), 1.5) == pytest.approx(2.0)
    src = problems.point_sources((33, 33), 3, 1, 4)
    assert np.all(np.abs(src).sum(axis=(1, 2)) == 1.0)


def test_param_spec_and_init():
    spec = netparams.param_spec((16, 32, 64))
    names = [s[0] for s in spec]
    assert len(names) == len(set(names))
    p = netparams.init_params((16, 32, 64), seed=0)
    q = netparams.init_params((16, 32, 64), seed=0)
    assert all(np.array_equal(p[k], q[k]) for k in p)
    assert p["sol.up2.w"].shape == (64, 32, 3, 3)  # transposed conv layout (c_in, c_out, 3, 3)
    assert p["sol.implicit.w"].shape == (32, 3, 3) and p["sol.implicit.w"][0, 1, 1] == 4 + 1j
    bound = 1 / np.sqrt(9 * 16)
    assert np.abs(p["sol.res0.a.w"]).max() <= bound
    with pytest.raises(ValueError):
        netparams.param_spec((16,))


def test_hierarchy_setup_matches_reference_structure():
    # test_multigrid.py:118-125, :146-162
    m = fields.slowness_model(np.random.default_rng(0).uniform(0.25, 1, (129, 129)), layer_width=16)
    H = multigrid.build_hierarchy(m)
    assert [lv.model.shape for lv in H.levels] == [(129, 129), (64, 64), (32, 32)]
    assert H.levels[0].wall is None and H.levels[1].wall is None
    wall = H.levels[2].wall
    assert wall is not None and np.all(wall[:-1, :-1] == 0) and np.all(wall[-1, :] > 0)
    assert H.levels[2].wall_edges[0] == wall[-1, 0]


def test_validation_errors():
    with pytest.raises(ConfigurationError):
        fields.build_abl(10, 10, 0, 0.01)
    with pytest.raises(DimensionError):
        fields.build_abl(10, 10, 5, 0.01)
    with pytest.raises(ConfigurationError):
        fields.SlownessModel(-np.ones((4, 4)), np.zeros((4, 4)), 1.0, 0.1)
    with pytest.raises(DimensionError):
        multigrid.build_hierarchy(fields.slowness_model(np.ones((6, 6)), layer_width=1), num_levels=3)
    m = fields.SlownessModel(np.ones((5, 5)), np.zeros((5, 5)), 0.0, 0.25)
    with pytest.raises(SingularityError):
        multigrid.Level(m, fields.TRUE_SHIFT, diag=np.zeros((5, 5)))


def test_install_as_helmsolve():
    import sys

    import paper_2306_17486_b200 as hs

    saved = {k: v for k, v in sys.modules.items() if k == "helmsolve" or k.startswith("helmsolve.")}
    try:
        hs.install_as_helmsolve()
        from helmsolve.krylov import SolveReport, solve_helmholtz  # noqa: F401
        from helmsolve.network import precompute_encodings  # noqa: F401

        assert sys.modules["helmsolve.fields"] is fields
    finally:
        for k in [k for k in sys.modules if k == "helmsolve" or k.startswith("helmsolve.")]:
            del sys.modules[k]
        sys.modules.update(saved)
