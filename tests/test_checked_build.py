"""Bounds evidence without compute-sanitizer (closed on this pool): the parity workloads re-run
against the test-only "checked" build (build.py VARIANTS, -DDGDS_CHECKED), whose kernels check
every slot id, stream row, token-extent range, history range and event-queue index they use
(DGDS_CHECK, csrc/trie.cuh) and flag a violation in the device error word. The runs set
DGDS_ASSERT_CLEAN, so every server closed in them fails unless the flags are clear.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _env():
    return dict(os.environ, DGDS_LIB_VARIANT="checked", DGDS_ASSERT_CLEAN="1")


def test_checked_build_sanitize_workload():
    """Every kernel of the library (append, walks, query modes, decode step, rebuild, blobs,
    compaction, peer exchange) on a small workload that forces rebuilds and extent moves."""
    r = subprocess.run([sys.executable, "tools/sanitize_workload.py"], env=_env(), cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "sanitize workload ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


def test_checked_build_parity_suite():
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        "tests/test_gpu_parity.py", "tests/test_scale_parity.py::test_c2_scale_parity",
                        "tests/test_replica_sync.py"],
                       env=_env(), cwd=ROOT, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    print(r.stdout[-400:])
