"""The reference's OWN unit tests, run against this repo's drop-in modules.

tests/refshim/lmmsim_shim.py assembles an ``lmmsim`` package whose image-path symbols are the
product's (core entirely; generator + trace I/O; split/route/schedule; WorkItem/encode_shard/
form_batch) and whose out-of-scope machinery (event loop, autoscaler, placement, latency
model) stays the reference's, so the reference simulator itself runs on the product code.

Needs the read-only reference tree (authoring container only); skipped where it is absent.
Run in a subprocess so the shim's ``lmmsim`` never leaks into this session's modules, from a
scratch cwd with bytecode and cache writes off (the reference tree is read-only).
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

REF_TESTS = Path("/root/reference/pkg/tests")
SHIM = Path(__file__).resolve().parent / "refshim"
ROOT = Path(__file__).resolve().parent.parent

pytestmark = pytest.mark.skipif(not REF_TESTS.is_dir(), reason="reference tree not present")


def _run_reference(args, tmp_path, timeout=900):
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1",
               PYTHONPATH=os.pathsep.join([str(SHIM), str(ROOT), os.environ.get("PYTHONPATH", "")]))
    cmd = [sys.executable, "-m", "pytest", "-p", "lmmsim_shim", "-p", "no:cacheprovider", "-q",
           "--rootdir", str(REF_TESTS), *args]
    r = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout + r.stderr


def test_reference_unit_suites_on_product(tmp_path):
    """reference test_core.py, test_workload.py, test_policies.py, test_engine.py: all 110 pass
    (incl. TestLoadTrace on TraceLoadResult, the preset count, split/route/form_batch goldens)."""
    files = [str(REF_TESTS / f) for f in ("test_core.py", "test_workload.py", "test_policies.py",
                                          "test_engine.py")]
    rc, out = _run_reference(files, tmp_path)
    assert rc == 0, out[-4000:]
    assert "110 passed" in out, out[-2000:]
    assert "lmmsim shim:" in out  # the shim was active


def test_reference_property_acceptance_on_product(tmp_path):
    """reference test_acceptance.py criterion 9 (shard makespan = 1/4, partition [4,4,4,4],
    starvation bound, ...: test_acceptance.py:445-550) with the product's batch objects."""
    rc, out = _run_reference([str(REF_TESTS / "test_acceptance.py") + "::test_criterion_9_property_suites",
                              "-s"], tmp_path)
    assert rc == 0, out[-4000:]
    assert "ACCEPTANCE 9" in out and "PASS" in out, out[-2000:]
