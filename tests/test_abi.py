"""CPU: the C-ABI library loads, exports every symbol include/liveput.h declares,
and its host table producers (perf_model stays on the host) are bit-identical
to the oracle.  No kernel is launched here."""
import ctypes as C
import re
from pathlib import Path

import pytest

from conftest import ROOT, load_golden, profile_by_name
from paper_2403_14097_b200 import _abi
from paper_2403_14097_b200.model import ParallelConfig, PlannerOptions, lm_1p5b

HEADER = ROOT / "include" / "liveput.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(lp_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _abi.lib()
    declared = declared_symbols()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_abi.exported_symbols()) == declared


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_abi.LIB_PATH)], capture_output=True, text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2403_14097_b200.planner import Planner
    with pytest.raises(_abi.LiveputError):
        Planner(lm_1p5b(), None, PlannerOptions())


def test_host_tables_match_golden():
    from paper_2403_14097_b200.planner import enumerate_configs, reactive_plan, scenario_count, throughput, mix_seed
    g = load_golden("tables")
    for c in g["throughput"]:
        assert float.hex(throughput(ParallelConfig(*c["cfg"]), profile_by_name(c["profile"]))) == c["value"]
    for c in g["configs"]:
        got = enumerate_configs(c["n"], profile_by_name(c["profile"]))
        assert [[x.pipelines, x.stages] for x in got] == c["configs"]
    for c in g["reactive"]:
        r = reactive_plan(c["n"], profile_by_name(c["profile"]))
        assert (None if r is None else [r.pipelines, r.stages]) == c["cfg"]
    for n, k, v in load_golden("scenarios")["scenario_count"]:
        assert scenario_count(n, k) == v
    for a, b, v in load_golden("rng")["mix_seed"]:
        assert mix_seed(a, b) == v


def test_struct_layout_matches_header():
    # lp_plan_step: int32 + 2*int32 + pad + 2*double
    assert C.sizeof(_abi.lp_plan_step) == 32
    assert C.sizeof(_abi.lp_liveput_row) == 24
    assert C.sizeof(_abi.lp_options) == 48
