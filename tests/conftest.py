import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    # GPU tests are NOT auto-skipped: on a GPU box a missing device or a missing libfb.so
    # must fail loudly.  On the CPU dev box run with -m "not gpu".
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libfb.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")
