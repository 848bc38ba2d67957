"""Readers for the golden fixtures produced by tests/golden/make_golden.py."""

import json
import os

import numpy as np

import workloads as W

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sweep(algo):
    """Yield (recipe, x, y, want) for the committed reference sweep."""
    d = np.load(os.path.join(GOLDEN, f"sweep_{algo}.npz"))
    recs = json.loads(str(d["recipes"]))
    off = d["offsets"]
    out = d["out"]
    for i, rec in enumerate(recs):
        x, y = W.materialize(rec)
        yield rec, x, y, out[off[i] : off[i + 1]], int(d["input_hash"][i])


def cases():
    with open(os.path.join(GOLDEN, "cases.json")) as f:
        c = json.load(f)
    arrays = np.load(os.path.join(GOLDEN, "cases.npz"))
    return c, arrays


def configs():
    p = os.path.join(GOLDEN, "configs.npz")
    if not os.path.exists(p):
        return None
    return np.load(p)
