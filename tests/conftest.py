import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFSIM = os.path.join(ROOT, "oracle", "_ref", "refsim")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")


def refsim(spec: str):
    """Run the compiled reference simulator (oracle/_ref/refsim) on a spec."""
    if not os.path.exists(REFSIM):
        pytest.skip("oracle/_ref/refsim not built (needs /root/reference at build time)")
    p = subprocess.run([REFSIM, spec], capture_output=True, text=True)
    return p.returncode, p.stdout, p.stderr


@pytest.fixture(scope="session")
def swlib():
    import paper_2505_03763_b200 as sw

    sw.lib()
    return sw
