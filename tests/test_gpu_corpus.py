"""GPU slowness-model preparation (paper_2306_17486_b200/corpus.py, csrc/prep.cu) against the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2306_17486_b200 import corpus  # noqa: E402
from oracle import corpus_oracle as co  # noqa: E402


def test_resize_smooth_normalise_match_oracle():
    rng = np.random.default_rng(0)
    a = rng.uniform(size=(3, 37, 53)) * 255
    r = corpus.resize_bilinear(a, (65, 65))
    for b in range(3):
        assert np.array_equal(r[b], co.resize_bilinear(a[b], (65, 65)))      # bit-exact
    for sigma in (0.0, 0.5, 1.0, 2.5):
        s = corpus.gaussian_smooth(r, sigma)
        for b in range(3):
            ref = co.gaussian_smooth(r[b], sigma)
            assert np.max(np.abs(s[b] - ref)) <= 1e-13 * np.max(np.abs(ref))
    n = corpus.normalise(s)
    for b in range(3):
        assert n[b].min() == 0.25 and n[b].max() == 1.0
        assert np.max(np.abs(n[b] - co.normalise(s[b]))) <= 1e-15
    assert np.all(corpus.normalise(np.full((2, 9, 9), 4.0)) == 0.25)


def test_load_slowness_corpus(tmp_path):
    rng = np.random.default_rng(1)
    img = rng.integers(0, 256, size=(40, 60), dtype=np.uint8)
    (tmp_path / "m0.pgm").write_bytes(b"P5\n60 40\n255\n" + img.tobytes())
    f = rng.uniform(size=(50, 50))
    f.astype("<f8").tofile(tmp_path / "m1.f64")
    (tmp_path / "m1.hdr").write_text("50 50\n")
    models = corpus.load_slowness_corpus(str(tmp_path), 64, layer_width=8)
    assert [m.shape for m in models] == [(65, 65), (65, 65)]
    for m, src in zip(models, (img.astype(np.float64), f)):
        ref = co.prepare(src, 64)
        assert np.max(np.abs(m.kappa_sq - ref)) <= 1e-13
        assert m.kappa_sq.min() == 0.25 and m.kappa_sq.max() == 1.0
    with pytest.raises(ValueError):
        corpus.load_slowness_corpus(str(tmp_path / "missing"), 64)
