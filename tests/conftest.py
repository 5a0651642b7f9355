"""Shared test configuration.

Markers:
  gpu  -- needs a B200 (sm_100a) and the built CUDA library; run with -m gpu.
Everything unmarked runs on the CPU-only build container.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

try:
    from hypothesis import settings
    settings.register_profile("repo", deadline=None, max_examples=50)
    settings.load_profile("repo")
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a B200 GPU and the built CUDA library")


GOLDEN = os.path.join(ROOT, "tests", "golden")
