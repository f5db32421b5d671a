"""The reference's own test suite (pkg/tests, 88 tests) run against this
package imported as ``fieldtess`` (tests/ref_shim).  The suite is copied as
fixtures into oracle/_ref/tests by ``make -C oracle ref`` (it travels to the
GPU box; /root/reference does not).  Deselected: test_mirror_symmetry,
whose mirror map is not a symmetry of the sheared lattice (a test bug in
the reference, SURVEY.md finding 2: it fails against the reference too)."""

import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
SUITE = os.path.join(REPO, "oracle", "_ref", "tests")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.isdir(SUITE), reason="reference suite not copied (make -C oracle ref)")
def test_reference_suite_passes():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(HERE, "ref_shim"), REPO, SUITE,
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", SUITE, SUITE,
           "--deselect", "test_field.py::TestStepProperties::test_mirror_symmetry"]
    r = subprocess.run(cmd, cwd=SUITE, env=env, capture_output=True, text=True, timeout=900)
    tail = "\n".join((r.stdout + r.stderr).splitlines()[-40:])
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and "failed" not in r.stdout, tail
