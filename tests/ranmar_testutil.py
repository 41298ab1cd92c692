"""Helpers shared by the test modules (kept out of conftest.py so they can be imported)."""
import numpy as np

from oracle.bind import STATE_DTYPE


def state_from_json(d):
    s = np.zeros(1, STATE_DTYPE)
    s["lane"][0] = d["lane"]
    s["i"], s["j"], s["v"] = d["i"], d["j"], d["v"]
    return s
