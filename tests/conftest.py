import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# The tests target the general tree engine at every width; the small-state tree kernel
# (n <= 10, options.small_tree) is exercised by explicit small_tree = 1 / auto cases in
# tests/test_gpu_small.py.  "0" only stops the automatic choice.
os.environ.setdefault("TQSIM_SMALL", "0")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running (minutes)")
