"""Load the reference-generated golden fixtures (tests/golden/make_golden.py)."""
import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def cases():
    return sorted(glob.glob(os.path.join(GOLDEN, "case_*.npz")))


def tw_cases():
    return sorted(glob.glob(os.path.join(GOLDEN, "tw_*.npz")))


def load(path):
    g = dict(np.load(path))
    d = int(g["dims"].size - 1)
    g["d"] = d
    g["p"] = int(g["p"])
    g["trial"] = "final" if int(g.get("trial", 0)) == 1 else "initial"
    g["dims"] = [int(v) for v in g["dims"]]
    g["U"] = [g[f"U{l}"] for l in range(d)]
    g["lam"] = [g[f"lam{l}"] for l in range(d)]
    for k in "MLGV":
        g[k] = [g[f"{k}{l}"] for l in range(d)]
    return g


def ids(paths):
    return [os.path.basename(p)[:-4] for p in paths]
