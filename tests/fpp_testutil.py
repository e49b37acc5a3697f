"""Shared helpers for the test suite (imported as a top-level module from tests/)."""
import numpy as np


def gpu_available() -> bool:
    try:
        import paper_2206_01382_b200 as fpp
        return fpp.device_count() > 0
    except Exception:
        return False


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
