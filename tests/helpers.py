"""Shared test helpers (fixture paths, golden-case enumeration)."""
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def fold_cases(folds):
    """(key, dtype, n, shape) for every case in folds.npz."""
    out = []
    for k in folds.files:
        if k.endswith("_sum"):
            key = k[: -len("_sum")]
            dtype, nstr, shp = key.split("_", 2)
            n = int(nstr[1:])
            shape = () if shp == "scalar" else tuple(int(s) for s in shp.split("x"))
            out.append((key, dtype, n, shape))
    return sorted(out)
