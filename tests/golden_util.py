"""Shared loader for the reference-generated golden fixtures (tests/golden/)."""
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=1)
def arrays():
    with np.load(GOLDEN / "golden.npz") as z:
        return {k: z[k] for k in z.files}


@lru_cache(maxsize=1)
def meta():
    with open(GOLDEN / "golden.json") as f:
        return json.load(f)
