"""The drop-in proven with the reference's own code.

adapter/ builds the reference's UNMODIFIED unit suite (proj/tests/*.cpp, 73
test cases, including the 200-instance DP-vs-exhaustive-search test,
test_optimizer.cpp:107-131) and its simulator (simulator.cpp:119-340) against
adapter/optimizer.cpp — a spotsim::Planner with the reference's public
interface that forwards to libliveput.so.  Built in the dev container (the
sources live under /root/reference), the binary travels to the GPU box.

  * CPU: the control build (same suite, the reference's own optimizer.cpp)
    passes 73/73 under the doctest stand-in, which pins the stand-in.
  * GPU: the adapter build passes 73/73 with every Planner call on the B200.
"""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BUILD = ROOT / "adapter" / "_build"
REF = Path("/root/reference/proj")


def _binary(name):
    b = BUILD / name
    if not b.exists() and REF.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "adapter"), "all", "control"], check=True,
                       capture_output=True)
    if not b.exists():
        pytest.skip(f"{b} not built (needs /root/reference in the dev container)")
    return b


def _run(b, timeout):
    r = subprocess.run([str(b)], capture_output=True, text=True, timeout=timeout)
    print(r.stdout[-2000:], r.stderr[-4000:])
    return r


def test_control_suite_with_reference_optimizer_cpu():
    r = _run(_binary("ref_unit_tests_cpu"), 600)
    assert r.returncode == 0
    assert "test cases: 73 | 73 passed | 0 failed" in r.stdout


def test_adapter_links_liveput():
    b = _binary("ref_unit_tests")
    out = subprocess.run(["ldd", str(b)], capture_output=True, text=True).stdout
    assert "libliveput.so" in out and "not found" not in out.split("libliveput.so")[1].split("\n")[0]


@pytest.mark.gpu
def test_reference_unit_suite_through_liveput_on_gpu():
    r = _run(_binary("ref_unit_tests"), 1200)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "test cases: 73 | 73 passed | 0 failed" in r.stdout
