"""The device CSV parser (csv.cu) against the reference's read_dataset_csv
(proj/src/harness.cpp:93-134): every golden case made by
tests/golden/make_csv_golden.py from the unmodified reference — values bit
for bit, ids, and the exact error texts.  The CPU test cross-checks the
goldens themselves against Python's correctly rounded float()."""
import gzip
import json
import os
import struct

import pytest

from conftest import ROOT

CSV = os.path.join(ROOT, "tests", "golden", "csv")
CASES = json.load(open(os.path.join(CSV, "INDEX.json"))) if os.path.exists(
    os.path.join(CSV, "INDEX.json")) else []


def load(name):
    with gzip.open(os.path.join(CSV, name + ".json.gz"), "rt") as f:
        g = json.load(f)
    with open(os.path.join(ROOT, g["path"]), "rb") as f:
        data = f.read()
    return g, data


def test_goldens_agree_with_python_float():
    """For every accepted file the reference's bits are Python's
    correctly rounded float() of the same field text."""
    checked = 0
    for name in CASES:
        g, data = load(name)
        e = g["expect"]
        if "csv_error" in e:
            continue
        lines = data.decode().split("\n")
        fields = []
        for line in lines[1:]:
            if line == "":
                continue
            fields += [f.replace("\r", "") for f in line.split(",")]
        bits = ["%016x" % struct.unpack("<Q", struct.pack("<d", float(f)))[0] for f in fields]
        assert bits == e["bits"], name
        checked += len(bits)
    assert checked > 8000


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_csv_parser_matches_reference(name):
    import numpy as np

    import paper_2412_02274_b200 as sk

    g, data = load(name)
    e = g["expect"]
    if "csv_error" in e:
        with pytest.raises(RuntimeError) as ei:
            sk.read_csv_bytes(data, g["path"])
        assert str(ei.value) == e["csv_error"]
        return
    vals, ids = sk.read_csv_bytes(data, g["path"])
    assert vals.shape == (e["rows"], e["dims"])
    assert ids.tolist() == e["ids"]
    got = ["%016x" % b for b in vals.reshape(-1).view(np.uint64).tolist()]
    assert got == e["bits"]


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [11, 12])
def test_device_csv_parser_random_stress(seed):
    """50k generated number texts (random doubles in several formats, exact
    midpoints and their neighbours, random digit strings) against Python's
    correctly rounded float() — which equals the reference's from_chars on
    every golden value (test above)."""
    import random
    import sys

    import numpy as np

    import paper_2412_02274_b200 as sk

    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    import make_csv_golden as mk

    rng = random.Random(seed)
    nums = [t for t in mk.number_cases(rng, 60000) if mk.in_range(t)][:50000]
    data = ("v\n" + "\n".join(nums) + "\n").encode()
    vals, _ = sk.read_csv_bytes(data, "stress.csv")
    want = np.array([float(t) for t in nums])
    assert vals.reshape(-1).view(np.uint64).tolist() == want.view(np.uint64).tolist()


@pytest.mark.gpu
@pytest.mark.parametrize("normalize,strategy", [(False, "none"), (True, "grid"), (False, "angular")])
def test_pipeline_from_csv_on_device(normalize, strategy):
    """run_experiment --dataset [--normalize] on the device: same skyline and
    map as parsing first and running the pipeline on the values."""
    import numpy as np

    import paper_2412_02274_b200 as sk

    v = sk.generate("ant", 30000, 3, 5) * [2.0, 1.0, 0.5]
    if strategy == "grid" and not normalize:
        v = v / v.max(axis=0)
    text = "x1,x2,x3\n" + "\n".join(",".join(repr(float(x)) for x in row) for row in v) + "\n"
    data = text.encode()
    res, shape = sk.pipeline_csv(data, "gen.csv", strategy, 16, cap=25, normalize=normalize)
    assert shape == (30000, 3)
    vals, ids = sk.read_csv_bytes(data, "gen.csv")
    assert vals.tobytes() == v.tobytes()  # repr round-trips exactly
    plan = sk.make_plan(strategy, 16, 3)
    ref = sk.pipeline(vals, ids, plan, cap=25, normalize=normalize)
    assert res.positions.tolist() == ref.positions.tolist()
    assert res.g_max == ref.g_max and res.den.tolist() == ref.den.tolist()
