"""Shipped gradient tables (30/60/90 directions), as in the reference's directions.py:21-233.

The tables are package data exported from the reference by tests/golden/make_golden.py.
"""

from __future__ import annotations

import os
from functools import lru_cache

import numpy as np

_TABLES = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "gradient_tables.npz")


@lru_cache(maxsize=None)
def _load() -> dict:
    with np.load(_TABLES) as z:
        return {k: z[k] for k in z.files}


def unit_sphere_directions(n: int) -> np.ndarray:
    """Copy of the shipped n-direction table (n in 30, 60, 90); rows are unit vectors as exported."""
    t = _load().get(f"dirs{n}")
    if t is None:
        raise ValueError(f"no shipped direction table for n={n}; available: [30, 60, 90]")
    return t.copy()
