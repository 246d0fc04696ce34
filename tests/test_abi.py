"""CPU checks of the C-ABI boundary: the library builds/loads, exports every
symbol include/skygpu.h declares, host logic works, and compute entry points
fail loudly (no CPU fallback) when no GPU is present."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2412_02274_b200 as sk
from paper_2412_02274_b200 import skypar
from conftest import ROOT
from oracle import pyoracle as po

HEADER = os.path.join(ROOT, "include", "skygpu.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void)\s+(skygpu_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = skypar.lib()
    names = declared_functions()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n
    nm = subprocess.run(["nm", "-D", "--defined-only", skypar.LIB_PATH], capture_output=True, text=True)
    exported = set(re.findall(r" T (skygpu_\w+)", nm.stdout))
    assert set(names) <= exported
    assert set(skypar.EXPORTED_SYMBOLS) == set(names)


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", skypar.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_make_plan_matches_oracle():
    for strat in ("none", "grid", "angular", "sliced"):
        for target in (1, 2, 4, 16, 32, 64, 100, 1000):
            for dims in (2, 3, 5, 7):
                p = sk.make_plan(strat, target, dims)
                assert (p.slices, p.partitions) == po.make_plan(strat, target, dims)
    with pytest.raises(ValueError, match="angular partitioning needs dims >= 2"):
        sk.make_plan("angular", 4, 1)
    with pytest.raises(ValueError, match="target partition count"):
        sk.make_plan("grid", 0, 3)
    with pytest.raises(ValueError, match="unknown strategy"):
        sk.make_plan("bogus", 4, 3)


@pytest.mark.parametrize("kind", ["uni", "ant", "corr", "lattice"])
@pytest.mark.parametrize("d", [1, 3, 7])
def test_product_generator_matches_oracle(kind, d):
    a = sk.generate(kind, 3000, d, 17)
    b = po.generate(kind, 3000, d, 17)
    assert (a.view(np.uint64) == b.view(np.uint64)).all()


@pytest.mark.skipif(skypar.device_count() > 0, reason="a GPU is present")
def test_no_cpu_fallback_without_gpu():
    v = sk.generate("uni", 100, 3, 1)
    with pytest.raises(sk.SkyGpuError, match="no CPU fallback"):
        sk.parallel_skyline(v)
    with pytest.raises(sk.SkyGpuError):
        sk.pipeline(v)
