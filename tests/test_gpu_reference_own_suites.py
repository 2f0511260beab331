"""The reference's OWN test modules (pkg/tests, staged unmodified into oracle/_ref/tests by
build()) run against this package's data plane: tests/pl_shim_plugin.py applies the
maintainer shim of INTEGRATION.md §2 before they import anything, so every KvStore they
build and every migration they run is this package's GPU implementation, while their
assertions, helpers, scenarios and the rest of pipeshift (engine, coordinator, fabric,
weights, cli) are the reference's.  The same modules are also run on the unmodified
reference in the same test: the two runs must fail exactly the same tests (the reference
fails one of its own, acceptance criterion 4, a test artefact -- SURVEY Appendix B.1)."""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
REF_TESTS = ROOT / "oracle" / "_ref" / "tests"
MODULES = ["test_kvstore.py", "test_migrator.py", "test_coordinator.py", "test_engine.py",
           "test_acceptance.py", "test_cluster.py", "test_fabric.py", "test_weights.py",
           "test_cli.py"]


def _run(shim: bool) -> tuple[int, set[str], str]:
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join(
        [str(ROOT / "tests"), str(ROOT / "oracle" / "_ref"), env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-rf",
           "--timeout=900", *MODULES]
    if shim:
        cmd[3:3] = ["-p", "pl_shim_plugin"]
    out = subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True,
                         timeout=1800)
    text = out.stdout + out.stderr
    m = re.search(r"(\d+) passed", text)
    failed = set(re.findall(r"^FAILED (\S+)", text, re.M))
    return (int(m.group(1)) if m else 0), failed, text[-3000:]


@pytest.mark.skipif(not REF_TESTS.is_dir(),
                    reason="oracle/_ref/tests not staged (build() stages it in the dev container)")
def test_reference_suites_pass_on_the_gpu_data_plane():
    passed, failed, tail = _run(shim=True)
    ref_passed, ref_failed, ref_tail = _run(shim=False)
    assert passed > 100, tail
    # same verdict as the unmodified reference, test by test
    assert failed == ref_failed, (failed, ref_failed, tail)
    assert passed == ref_passed, (passed, ref_passed)
    assert failed <= {"test_acceptance.py::test_criterion_4_migration_consistency"}, failed
