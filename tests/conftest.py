import gzip
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libskygpu.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def golden_names(prefixes=None, exclude=()):
    names = sorted(f[: -len(".json.gz")] for f in os.listdir(GOLDEN) if f.endswith(".json.gz"))
    if prefixes:
        names = [n for n in names if n.startswith(tuple(prefixes))]
    return [n for n in names if not n.startswith(tuple(exclude))]


def load_golden(name):
    with gzip.open(os.path.join(GOLDEN, name + ".json.gz"), "rt") as f:
        return json.load(f)


def golden_input(g, generate):
    """(values, ids) of a golden case; `generate(kind, n, d, seed)` builds seeded inputs."""
    sp = g["spec"]
    if sp["kind"] == "literal":
        v = np.asarray(sp["values"], dtype=np.float64).reshape(sp["n"], sp["d"])
    else:
        v = generate(sp["gen"], sp["n"], sp["d"], sp["seed"])
    return v, np.arange(v.shape[0], dtype=np.int64)


def spec_cap(g):
    c = g["spec"]["cap"]
    return None if c == 0 else c
