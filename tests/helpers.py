"""Shared test helpers."""
import numpy as np


def rel_l2(x, ref):
    """||x - ref||_2 / ||ref||_2 over the whole array in canonical order."""
    x = np.asarray(x, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    nr = np.linalg.norm(ref)
    if nr == 0.0:
        return float(np.linalg.norm(x))
    return float(np.linalg.norm(x - ref) / nr)


