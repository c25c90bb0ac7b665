import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    return {name: dict(np.load(os.path.join(GOLDEN, name + ".npz")))
            for name in ("fit", "closed", "mc", "rng", "semi", "comb", "io", "cases", "synth")}

# small host-path chunks so the GPU tests exercise cpb_run_host's chunked
# upload and chunk views (the library reads this once, at first use)
os.environ.setdefault("CPB_HOST_CHUNK_BYTES", str(64 * 1024))
