import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: long CPU test (oracle at paper scale)")


def pytest_sessionfinish(session, exitstatus):
    # parity-floor report of tests/test_gpu_parity.py (how many queries only the 2e-6·S floor admits)
    mod = sys.modules.get("test_gpu_parity") or sys.modules.get("tests.test_gpu_parity")
    rep = getattr(mod, "FLOOR_REPORT", None)
    out = os.environ.get("WN_PARITY_REPORT")
    if rep and out:
        import json

        with open(out, "w") as f:
            json.dump(rep, f, indent=1)
