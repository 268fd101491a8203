"""The C++ facade (include/spotsim_b200/planner.hpp) over the C ABI: compiles on
CPU; its parity suite (tests/cpp/test_planner.cpp) runs on the GPU."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_2403_14097_b200" / "lib"
BIN = ROOT / "tests" / "cpp" / "test_planner"


def build():
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", str(ROOT / "tests" / "cpp" / "test_planner.cpp"),
           f"-I{ROOT / 'include'}", f"-L{LIBDIR}", "-lliveput", f"-Wl,-rpath,{LIBDIR}", "-o", str(BIN)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_facade_compiles_and_links():
    build()
    assert BIN.exists()


@pytest.mark.gpu
def test_facade_parity_suite_on_gpu():
    build()
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
    assert " 0 failed" in r.stdout
