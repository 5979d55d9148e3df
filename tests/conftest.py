import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run on the GPU box)")
    config.addinivalue_line("markers", "slow: long CPU test (full-size configs)")
    # build the C/CUDA artefacts once (idempotent; make only rebuilds what changed)
    subprocess.run(["make", "-C", ROOT, "-s", "gen", "oracle", "spchol"], check=False)
