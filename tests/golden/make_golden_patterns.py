"""Deterministic inputs shared by the golden generator and the tests (no reference import)."""
import numpy as np


def fresh_pattern(step, layer, k, n, h):
    """Exactly representable stand-in for fresh expert rows [k, n, h]."""
    s = np.arange(k)[:, None, None]
    t = np.arange(n)[None, :, None]
    c = np.arange(h)[None, None, :]
    return (step * 16 + layer * 4 + s + 1) + t / 64.0 + c / 4096.0
