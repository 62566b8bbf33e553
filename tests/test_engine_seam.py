"""The reference engine driving the B200 draft server through the SpeculationSource seam
(INTEGRATION.md §3): oracle/_ref/engine_seam runs the reference Instance::decode_step replay
(proj/src/engine.cpp:69-167) once over the reference's DraftClient / LocalTransport /
DraftServer and once over DgdsSource -> dgds_b200::GpuSpeculationSource -> DraftClient(DraftTransport&)
-> the GPU server, and requires every StepReport to be identical. The "replicas" run puts a
non-local transport in between, so the client serves from GPU replicas synced by GDX1 blobs.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "engine_seam")


@pytest.mark.parametrize("k,mode", [(1, "server"), (4, "server"), (1, "replicas")])
def test_reference_engine_through_the_seam(k, mode):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/engine_seam not built (reference sources absent at build time)")
    r = subprocess.run([BIN, str(k), mode], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "engine seam ok" in r.stdout
    print(r.stdout)
