import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libtetsplat_b200.so")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


RENDER_CASES = sorted(os.path.basename(p)[len("render_"):-4]
                      for p in glob.glob(os.path.join(GOLDEN, "render_*.npz")))


def rel_err(a, b):
    """max|a-b| / max|b| — the normalisation of gradcheck.py:136-137."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.abs(b).max(initial=0.0)
    num = np.abs(a - b).max(initial=0.0)
    return num / den if den > 0 else num
