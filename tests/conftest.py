import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "reference: needs the reference source tree at /root/reference")


def pytest_collection_modifyitems(config, items):
    have_ref = Path("/root/reference/pkg/src/fragserve").exists()
    skip_ref = pytest.mark.skip(reason="reference tree not present (GPU box)")
    for item in items:
        if "reference" in item.keywords and not have_ref:
            item.add_marker(skip_ref)
