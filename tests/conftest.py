import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def golden(name):
    import numpy as np

    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def lib():
    from paper_2006_04391_b200 import _lib

    return _lib.load()


@pytest.fixture(scope="session")
def parity_log():
    """parity_log(what, **errors): append measured parity errors as a JSON
    line to $AM_PARITY_LOG (if set), so the numbers behind DESIGN.md's
    parity table come from the GPU test run itself."""
    import json

    path = os.environ.get("AM_PARITY_LOG")

    def log(what, **errs):
        if path:
            with open(path, "a", encoding="utf-8") as fh:
                fh.write(json.dumps({"what": what, **errs}) + "\n")

    return log
