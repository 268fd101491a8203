import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libliveput.so on cuda:0)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    return json.loads((GOLDEN / f"{name}.json").read_text())


def unhex(s):
    return float.fromhex(s)


@pytest.fixture(scope="session")
def golden():
    return load_golden


def profile_by_name(name):
    from paper_2403_14097_b200.model import PROFILES
    return PROFILES[name]()


def profile_from_dict(d):
    from paper_2403_14097_b200.model import WorkloadProfile
    d = dict(d)
    d["pipeline_rates"] = {int(k): v for k, v in d.get("pipeline_rates", {}).items()}
    return WorkloadProfile(**d)
