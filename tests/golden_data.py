"""Loader for tests/golden/reference_golden.npz (made by tests/golden/make_golden.py)."""
import os

import numpy as np

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz")
_G = None


def golden():
    global _G
    if _G is None:
        _G = dict(np.load(PATH))
    return _G


def rows_of(prefix, ears, dirs):
    g = golden()
    return [(g["%s_idx_%d_%d" % (prefix, e, d)], g["%s_vals_%d_%d" % (prefix, e, d)])
            for e in range(ears) for d in range(dirs)]
