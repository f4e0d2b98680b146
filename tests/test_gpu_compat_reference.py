"""Compat mode: the reference's OWN hot-path unit tests -- pkg/tests/test_tensor.py,
test_autodiff.py and test_nn.py, unmodified -- run against this device backend.

``nsk_backend.install_compat()`` (loaded as a pytest plugin before collection) rebinds the reference modules
``nsk.tensor`` / ``nsk.autodiff`` / ``nsk.nn`` / ``nsk.gradcheck`` to this package, so every ``Pool``, ``Tensor``,
``matmul_t``, ``rec_*``, ``backward``, ``sgd_step`` ... those tests touch is the device implementation (libnskb
kernels, device arena, device GradCache). The reference tests were installed next to the package by
tools/install_reference.sh (baseline/_ref/ref_tests).
"""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "ref_tests")
# test counts of each file on the reference's own CPU path (pkg/tests): all of them must pass here
FILES = {"test_tensor.py": 33, "test_autodiff.py": 25, "test_nn.py": 27}


def _run(files, plugin=True):
    if not all(os.path.exists(os.path.join(REF_TESTS, f)) for f in files):
        raise AssertionError("the reference and its tests are not installed: run tools/install_reference.sh "
                             "(baseline/_ref travels to the GPU box with the working tree)")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, os.path.join(ROOT, "tests"), REF]))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", REF_TESTS]
    if plugin:
        cmd += ["-p", "compat_plugin"]
    cmd += [os.path.join(REF_TESTS, f) for f in files]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=REF_TESTS, timeout=900)
    return r


@pytest.mark.parametrize("name", sorted(FILES))
def test_reference_unit_tests_pass_on_device(name):
    r = _run([name])
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    last = r.stdout.strip().splitlines()[-1]
    m = re.search(r"(\d+) passed", last)
    assert m and int(m.group(1)) == FILES[name], tail  # every reference test ran and passed (none skipped)
    assert "failed" not in last and "skipped" not in last and "error" not in last, tail


def test_compat_mode_really_binds_the_device_backend():
    """The rebinding is what the reference tests see: their Pool / matmul_t / backward are this package's."""
    probe = (
        "from paper_2409_11600_b200.nsk_backend import install_compat; install_compat()\n"
        "import nsk.tensor as T, nsk.autodiff as A, nsk.nn as N\n"
        "import paper_2409_11600_b200.tensor as DT, paper_2409_11600_b200.autodiff as DA\n"
        "assert T.Pool is DT.Pool and T.matmul_t is DT.matmul_t and A.backward is DA.backward\n"
        "p = T.Pool(); t = T.tensor_from_array(p, [[1.0, 2.0]])\n"
        "assert t.buffer.ptr != 0 and type(t.buffer).__module__ == 'paper_2409_11600_b200.tensor'\n"
        "print('bound')\n"
    )
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, REF]))
    r = subprocess.run([sys.executable, "-c", probe], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0 and "bound" in r.stdout, r.stderr[-2000:]
