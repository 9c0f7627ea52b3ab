"""Run the REFERENCE's own test files against this package (drop-in proof, SURVEY.md §4 "Reuse").

    python tools/ref_suite.py stage      # here (the container that has /root/reference): copy the reference's
                                         # conftest.py, test_fields.py, test_multigrid.py, test_krylov.py into
                                         # oracle/_ref/ref_tests/ -- git-ignored, never committed, but it travels
                                         # to the GPU box with the gpurun snapshot
    python tools/ref_suite.py run [pytest args]   # on the GPU box: helmsolve -> paper_2306_17486_b200, run them

The reference's test_green.py and test_autodiff.py import ``helmsolve.autodiff``, the reference's generic
reverse-mode engine; that engine is out of scope (training, not the solve path), so
those two files are not run.  The Green's-function layer they pin is covered by tests/test_gpu_network.py
against fixtures generated from the reference's own green.py (tests/golden/cnn_primitives.npz).
"""
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEST = os.path.join(ROOT, "oracle", "_ref", "ref_tests")
FILES = ("conftest.py", "test_fields.py", "test_multigrid.py", "test_krylov.py")


def stage():
    src = "/root/reference/pkg/tests"
    os.makedirs(DEST, exist_ok=True)
    for f in FILES:
        shutil.copyfile(os.path.join(src, f), os.path.join(DEST, f))
    print(f"staged {len(FILES)} reference test files in {DEST} (git-ignored)")


def run(extra):
    sys.path.insert(0, ROOT)
    import paper_2306_17486_b200 as pkg

    pkg.install_as_helmsolve()
    import pytest

    return pytest.main(["-q", "-p", "no:cacheprovider", "--rootdir", DEST, DEST] + list(extra))


if __name__ == "__main__":
    if sys.argv[1:2] == ["stage"]:
        stage()
    else:
        sys.exit(run(sys.argv[2:]))
