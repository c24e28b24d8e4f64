"""Shared helpers for the test-suite (golden loading, error metrics, GPU probe)."""
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))


def rel_err(a, b):
    """max|a-b| / max|b| (the reference tests' relative-to-scale metric)."""
    a = np.asarray(a)
    b = np.asarray(b)
    scale = np.abs(b).max()
    return float(np.abs(a - b).max() / (scale if scale > 0 else 1.0))


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
