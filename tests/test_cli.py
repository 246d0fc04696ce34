"""The skypar CLI — the reference's UNMODIFIED proj/tools/skypar_main.cpp
compiled against the original CLI11-subset header
(adapter/cli11_subset/CLI11.hpp) — argument handling, on CPU: the binary
built over the unmodified reference library (skypar_ref) shares the parser
with the GPU build, and --help / usage errors never touch a device."""
import os
import subprocess

import pytest

from conftest import ROOT

REF = os.path.join(ROOT, "oracle", "_ref")
CLI_REF = os.path.join(REF, "skypar_ref")
CLI_GPU = os.path.join(REF, "skypar_gpu")

pytestmark = pytest.mark.skipif(not os.path.exists(CLI_REF),
                                reason="CLI binaries not built (needs /root/reference)")


def run(exe, *args):
    return subprocess.run([exe, *args], capture_output=True, text=True, timeout=120)


@pytest.mark.parametrize("exe", [CLI_REF, CLI_GPU])
def test_help(exe):
    if not os.path.exists(exe):
        pytest.skip("not built")
    r = run(exe, "--help")
    assert r.returncode == 0 and "--strategy" in r.stdout and "--oracle" in r.stdout


@pytest.mark.parametrize("args,needle", [
    (["--gen", "zipf"], "not in {uni,ant}"),
    (["--gen", "uni", "--dataset", "x.csv"], "excludes"),
    (["--gen", "uni", "--cap", "1"], "not in range"),
    (["--gen", "uni", "--d", "0"], "not positive"),
    (["--gen", "uni", "--reps", "-1"], "negative"),
    (["--gen", "uni", "--strategy", "ring"], "not in {none,grid,angular,sliced}"),
    (["--gen", "uni", "--format", "xml"], "not in {csv,jsonl}"),
    (["--gen", "uni", "--n", "abc"], "not a valid number"),
    (["--bogus"], "unknown option"),
])
def test_usage_errors(args, needle):
    r = run(CLI_REF, *args)
    assert r.returncode == 2 and needle in r.stderr


def test_missing_source_is_a_runtime_error():
    r = run(CLI_REF, "--n", "10")
    assert r.returncode == 1 and "one of --dataset and --gen is required" in r.stderr


def test_list_sweeps_cross_product(tmp_path):
    out = tmp_path / "r.csv"
    r = run(CLI_REF, "--gen", "uni", "--n", "300,400", "--d", "2", "--strategy", "none,sliced",
            "--partitions=4", "--mode", "skyline", "--out", str(out))
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    assert len(lines) == 1 + 4  # header + one skyline row per combination
    assert {l.split(",")[2] for l in lines[1:]} == {"300", "400"}
    assert {l.split(",")[4] for l in lines[1:]} == {"none", "sliced"}
