"""CPU checks of the slowness-model preparation oracle against the SPEC's own examples
(the reference has no code for it) and the corpus file formats."""
import numpy as np

from oracle import corpus_oracle as co


def test_smoothing_examples():
    rng = np.random.default_rng(0)
    a = rng.uniform(size=(20, 30))
    assert np.array_equal(co.gaussian_smooth(a, 0.0), a)                      # sigma = 0 is the identity
    c = np.full((17, 9), 0.6)
    assert np.allclose(co.gaussian_smooth(c, 2.0), c, rtol=0, atol=1e-15)    # constant -> constant
    d = np.zeros((41, 41))
    d[20, 20] = 1.0
    s = 2.0
    out = co.gaussian_smooth(d, s)
    # the analytic kernel: exp(-t^2 / (2 sigma^2)) on |t| <= ceil(3 sigma), normalised, outer product
    r = int(np.ceil(3 * s))
    t = np.arange(-r, r + 1)
    g = np.exp(-0.5 * (t / s) ** 2)
    g /= g.sum()
    ref = np.zeros_like(d)
    ref[20 - r:21 + r, 20 - r:21 + r] = np.outer(g, g)
    assert np.max(np.abs(out - ref)) < 1e-6                                   # delta -> discrete Gaussian
    chk = np.indices((24, 24)).sum(axis=0) % 2 * 1.0
    sm = co.gaussian_smooth(chk, 1.0)
    assert np.max(np.abs(np.diff(sm, axis=1))) < np.max(np.abs(np.diff(chk, axis=1)))


def test_normalisation_examples():
    rng = np.random.default_rng(1)
    a = rng.normal(size=(33, 33)) * 7 + 3
    n = co.normalise(a)
    assert n.min() == 0.25 and n.max() == 1.0
    assert np.max(np.abs(co.normalise(n) - n)) <= 1e-12                      # idempotent
    assert np.all(co.normalise(np.full((5, 5), 3.0)) == 0.25)               # degenerate rule


def test_resize_corners_and_linearity():
    rng = np.random.default_rng(2)
    a = rng.uniform(size=(13, 21))
    r = co.resize_bilinear(a, (49, 33))
    for (i, j), (ii, jj) in (((0, 0), (0, 0)), ((0, 32), (0, 20)), ((48, 0), (12, 0)), ((48, 32), (12, 20))):
        assert r[i, j] == a[ii, jj]
    ramp = np.add.outer(np.arange(13) * 0.5, np.arange(21) * 0.25)
    rr = co.resize_bilinear(ramp, (25, 41))
    assert np.allclose(rr, np.add.outer(np.linspace(0, 6, 25), np.linspace(0, 5, 41)), atol=1e-12)


def test_corpus_files_round_trip(tmp_path):
    img = (np.arange(6 * 4) * 10 % 256).astype(np.uint8).reshape(6, 4)
    (tmp_path / "a.pgm").write_bytes(b"P5\n# a comment\n4 6\n255\n" + img.tobytes())
    f = np.random.default_rng(3).uniform(size=(5, 7))
    f.astype("<f8").tofile(tmp_path / "b.f64")
    (tmp_path / "b.hdr").write_text("5 7\n")
    assert np.array_equal(co.read_pgm(str(tmp_path / "a.pgm")), img.astype(np.float64))
    assert np.array_equal(co.read_f64(str(tmp_path / "b.f64")), f)
    k2 = co.prepare(f, 32)
    assert k2.shape == (33, 33) and k2.min() == 0.25 and k2.max() == 1.0
